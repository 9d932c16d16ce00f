#!/bin/bash
# usage: tools/ncu_one.sh <kernel-base-name> <out-name> <command...>: one --set full capture (2nd launch)
k=$1; o=$2; shift 2
timeout 600 ncu --set full --warp-sampling-interval 0 --import-source on --clock-control none --kernel-name-base function -k "$k" -s 2 -c 1 \
  -o gpurun_out/$o "$@" > gpurun_out/$o.log 2>&1
tail -2 gpurun_out/$o.log
