#!/bin/bash
# Diagnostics: build a trace library with extra -D flags and print the prefix-kernel timeline.
# usage: tools/trace_variant.sh WORKLOAD CTA "-DHTA_SKIP=4 ..."
cd "$(dirname "$0")/.."
W=$1; CTA=$2; FLAGS=$3
d=/tmp/tv; mkdir -p $d
for f in paper_2502_17421_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -DHTA_TRACE $FLAGS -c $f -o $d/$(basename $f).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libhta_trace.so $d/*.o -ldl -lpthread
HTA_LIB=$d/libhta_trace.so python tools/trace_prefix.py $W $CTA
