# Round measurement batch (run on the GPU box from the repo root).
set -x
mkdir -p gpurun_out
timeout 500 python -m pytest tests -q -m gpu --timeout 120 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_decode.csv \
    python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gemv -s 16 -c 2 -o gpurun_out/prof_decode_r1b \
    python tools/prof_layer.py --banks 8 --iters 3 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/prof_decode_r1b.ncu-rep --page details --csv > gpurun_out/ncu_decode_details.csv 2>/dev/null
ncu -i gpurun_out/prof_decode_r1b.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/ncu_decode_dram.csv 2>/dev/null
