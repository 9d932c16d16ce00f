python tools/trace_gemv.py --banks 8 --dump gpurun_out/trace_int3_cold.npy
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:"k_route_small|k_ffn_gemv" -c 2 -o gpurun_out/prof_dec_r1d python tools/prof_layer.py > gpurun_out/ncu_dec.log 2>&1; tail -1 gpurun_out/ncu_dec.log
python bench.py --no-sweep --no-cpu --steps 200 --warmup 10 2>&1 | tail -1 > gpurun_out/bench_imma.json
python -c "import json; d=json.loads(open('gpurun_out/bench_imma.json').read()); print(d['value'], d['ms_per_step'], d['detail']['kernel_share'], d['roofline'])"
