#!/bin/bash
# Diagnostics: rebuild prefix_tc.cu with extra -D flags and time one workload's prefix kernel.
# usage: tools/variant_sweep.sh WORKLOAD "label1:-DFLAG=..." "label2:-D..."

cd "$(dirname "$0")/.."
W=$1; shift
mkdir -p /tmp/vs_common
for f in paper_2502_17421_b200/csrc/*.cu; do
  [ "$(basename $f)" = prefix_tc.cu ] && continue
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -c $f -o /tmp/vs_common/$(basename $f).o &
done
wait
for spec in "$@"; do
  label=${spec%%:*}; flags=${spec#*:}
  d=/tmp/vs_$label; mkdir -p $d
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Iinclude $flags -c paper_2502_17421_b200/csrc/prefix_tc.cu -o $d/prefix_tc.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libhta.so $d/prefix_tc.o /tmp/vs_common/*.o -ldl -lpthread
  echo "$label [$flags]: $(HTA_LIB=$d/libhta.so python bench.py --workload $W --steps 10 --no-cpu-baseline --no-all-configs | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("prefix_us %.1f  step_us %.1f" % (r["kernel_us"], d["us_per_step"]))')"
done
