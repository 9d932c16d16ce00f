#!/bin/bash
# A/B variant of the decode kernel: tools/ab_build.sh NAME [-DMACRO=V ...]
# SRC=path overrides the source (e.g. a git-show copy of an earlier dec.cu).
# Compiles dec.cu (d_model 1024, int2/int3 instantiations only) with the given macros and links it
# with the regular objects into ab/NAME/libmoqe_gpu.so; select it with MOQE_GPU_LIB=ab/NAME/libmoqe_gpu.so.
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
b=$root/paper_2310_02410_b200/build
out=$root/ab/$name
mkdir -p "$out"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
  -DDEC_AB_ONLY -I"$root/paper_2310_02410_b200/csrc" "$@" -c "${SRC:-$root/paper_2310_02410_b200/csrc/dec.cu}" -o "$out/dec.o"
objs=$(ls $b/*.o | grep -v '/dec.o$')
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libmoqe_gpu.so" $objs "$out/dec.o" -lcudart
echo "$out/libmoqe_gpu.so"
