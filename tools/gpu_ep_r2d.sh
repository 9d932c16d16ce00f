# EP device dispatch/combine on the GPU box: tests, config-4 EP bench line at N=1, launch list.
mkdir -p gpurun_out/ep2
O=gpurun_out/ep2
timeout 900 python -m pytest tests/test_gpu_ep.py "tests/test_gpu_large.py::test_config4_ep_world1" -q --timeout 600 -p no:cacheprovider > $O/gpu_tests_ep.log 2>&1; tail -3 $O/gpu_tests_ep.log
timeout 900 python bench.py --ep --steps 20 --warmup 3 --no-sweep > $O/bench_ep.json 2> $O/bench_ep.err; echo "ep bench rc=$?"; tail -c 1500 $O/bench_ep.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:'k_|nccl|Kernel2|elementwise|index|reduce|cat' -c 400 --csv \
    --log-file $O/launches_ep.csv python bench.py --ep --steps 2 --warmup 1 --no-sweep --no-cpu > $O/launch_ep.log 2>&1; echo "launch rc=$?"
grep -c k_ep_ $O/launches_ep.csv || true
