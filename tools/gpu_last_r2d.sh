# Last check of the round on HEAD: full -m gpu suite, smoke, default bench line.
mkdir -p gpurun_out/last
O=gpurun_out/last
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; head -c 400 $O/bench.json
