MOQE_GPU_LIB=ab/half/libmoqe_gpu.so timeout 120 python -m pytest tests/test_gpu_moe.py -q -x -p no:cacheprovider -k "32-1024-4096-3-24 or 32-1024-4096-2-24" 2>&1 | tail -1
bash tools/ab_run.sh "--bits 3 2" cur3 half
for n in trace3 halft; do echo "== $n"; MOQE_GPU_LIB=ab/$n/libmoqe_gpu.so python tools/dec_trace.py 2>&1 | grep -A1 "^router [01] "; done
