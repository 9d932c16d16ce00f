# k_route_logits2t (two tokens per lane) parity + A/B timing on config 4's EP step
mkdir -p gpurun_out/r2t
O=gpurun_out/r2t
timeout 900 python -m pytest tests/test_gpu_route.py tests/test_gpu_large.py tests/test_gpu_ep.py -q --timeout 400 -p no:cacheprovider > $O/tests.log 2>&1; tail -3 $O/tests.log
for v in 0 1 0 1; do
  echo -n "2T=$v "; MOQE_ROUTE_LOGITS_2T=$v timeout 600 python bench.py --ep --steps 20 --warmup 3 --no-sweep --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function \
    -k regex:'k_route' -c 20 --csv --log-file $O/route_launches.csv python bench.py --ep --steps 2 --warmup 1 --no-sweep --no-cpu > $O/launch.log 2>&1; echo "launch rc=$?"
