#!/bin/bash
# tools/ab_run.sh "<dec_bench args>" name1 name2 ...: decode timing of each ab/ variant (interleaved twice)
args=$1; shift
for rep in 1 2; do
  for n in "$@"; do
    echo -n "$n: "
    MOQE_GPU_LIB=ab/$n/libmoqe_gpu.so timeout 300 python tools/dec_bench.py $args 2>&1 | grep "us/forward"
  done
done
