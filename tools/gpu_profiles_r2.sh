# Round-2 profile batch (run on the GPU box from the repo root): launch list of the bench
# command, full ncu captures of the decode kernel (k_dec), the prefill GEMM and the
# tensor-core prefill router, DRAM traffic per launch.
set -x
mkdir -p gpurun_out/r2prof
O=gpurun_out/r2prof
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu > $O/launch.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:k_dec -s 16 -c 1 \
    -o $O/k_dec python tools/dec_bench.py --layers 8 --reps 2 --bits 3 > $O/k_dec.log 2>&1; echo "k_dec rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:k_ffn_gemm2 -s 2 -c 1 \
    -o $O/gemm16k python tools/time_layer.py --bits 3 --tokens 16384 --banks 2 > $O/gemm.log 2>&1; echo "gemm rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:k_route_mma_p -s 2 -c 1 \
    -o $O/route16k python tools/time_layer.py --bits 3 --tokens 16384 --banks 2 > $O/route.log 2>&1; echo "route rc=$?"
for r in k_dec gemm16k route16k; do
  ncu -i $O/$r.ncu-rep --page details --csv > $O/${r}_details.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active > $O/${r}_raw.csv 2>/dev/null
done
ls -la $O
