K=${K:-k_gemv_fc1}
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:"$K" -c 1 -o gpurun_out/prof_gemv python tools/prof_layer.py "$@" > gpurun_out/ncu_gemv.log 2>&1; tail -1 gpurun_out/ncu_gemv.log
