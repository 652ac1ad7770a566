#!/bin/bash
# Diagnostics: build libhta variants with the softmax (HTA_SKIP=1) or softmax+MMA (HTA_SKIP=2)
# skipped and time the prefix kernel of a workload with each (tools/, not the product).
set -e
cd "$(dirname "$0")/.."
W=${1:-llama8b_64k}
for k in ${SKIPS:-0 1 2}; do
  mkdir -p /tmp/skip$k
  for f in paper_2502_17421_b200/csrc/*.cu; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Iinclude -DHTA_SKIP=$k -c $f -o /tmp/skip$k/$(basename $f).o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /tmp/skip$k/libhta.so /tmp/skip$k/*.o -ldl -lpthread
  echo "HTA_SKIP=$k: $(HTA_LIB=/tmp/skip$k/libhta.so python bench.py --workload $W --steps 10 --no-cpu-baseline --no-all-configs | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print("prefix_us %.1f  hbm %.0f GB/s" % (r["kernel_us"], r["hbm_gbs_achieved"]))')"
done
