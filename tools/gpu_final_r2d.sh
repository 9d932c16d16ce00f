# Round-2 closing batch (GPU box, repo root): GPU tests, smoke, default bench, reference arm,
# launch list of the bench command, full captures of the headline decode kernel and of the
# mid-size path (T=512 int4, config 1).
mkdir -p gpurun_out/r2d
O=gpurun_out/r2d
timeout 900 python -m pytest tests -q -m gpu --timeout 300 -p no:cacheprovider > $O/gpu_tests.log 2>&1; tail -2 $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"; tail -c 600 $O/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 --csv \
    --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu > $O/launch.log 2>&1; echo "launch list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:k_dec -s 16 -c 1 \
    -o $O/k_dec python tools/dec_bench.py --layers 8 --reps 2 --bits 3 > $O/k_dec.log 2>&1; echo "k_dec rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:k_dec -s 16 -c 1 \
    -o $O/k_dec_mid512 python tools/dec_bench.py --layers 8 --reps 2 --bits 4 --tokens 512 > $O/k_dec_mid.log 2>&1; echo "k_dec mid rc=$?"
for r in k_dec k_dec_mid512; do
  ncu -i $O/$r.ncu-rep --page details --csv > $O/${r}_details.csv 2>/dev/null
  ncu -i $O/$r.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active > $O/${r}_raw.csv 2>/dev/null
done
ls -la $O
ncu -i $O/k_dec.ncu-rep --page source --csv --print-source sass > $O/k_dec_sass.csv 2>/dev/null
python tools/ncu_sass_regions.py $O/k_dec_sass.csv 64 > $O/k_dec_regions.txt 2>&1
rm -f $O/*.ncu-rep $O/k_dec_sass.csv
