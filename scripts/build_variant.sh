#!/bin/bash
# Developer A/B: build the library with extra nvcc defines into _lib/variants/<name>/
# (load it with YAS_LIBRARY=<that path>/libyasmin_b200.so).
#   scripts/build_variant.sh nohint -DYAS_NO_L2HINT
set -e
cd "$(dirname "$0")/../paper_1909_01786_b200/csrc"
name=$1; shift
out=../_lib/variants/$name
mkdir -p $out
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC "$@" \
    -c device/engine.cu -o $out/engine.o
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $out/libyasmin_b200.so \
    ../_lib/obj/host/program.o ../_lib/obj/host/compile.o ../_lib/obj/capi.o ../_lib/obj/fleet.o $out/engine.o \
    -Xlinker -soname=libyasmin_b200.so -ldl
echo $out/libyasmin_b200.so
