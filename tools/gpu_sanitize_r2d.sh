# compute-sanitizer on small forwards through every kernel family (tools/sanitize_small.py)
mkdir -p gpurun_out/san
O=gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 400 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py > $O/$tool.log 2>&1; echo "$tool rc=$?"; tail -4 $O/$tool.log
done
