# Closing check on the GPU box: full -m gpu suite, smoke, config-4 EP bench line, EP launch list.
mkdir -p gpurun_out/fin2
O=gpurun_out/fin2
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py --ep --steps 20 --warmup 3 --no-sweep > $O/bench_ep.json 2> $O/bench_ep.err; echo "ep bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base function \
    -k regex:'^k_|nccl' -c 300 --csv --log-file $O/launches_ep.csv python bench.py --ep --steps 2 --warmup 1 --no-sweep --no-cpu > $O/launch_ep.log 2>&1; echo "launch rc=$?"
