#!/bin/bash
# Diagnostics: build whole-library variants with extra -D flags (optionally replacing prefix_tc.cu
# by another source) and run a command against each.
# usage: tools/lib_variants.sh "CMD" "label1:-DFLAG=...[@path/to/prefix_tc.cu]" ...   (CMD sees HTA_LIB)
cd "$(dirname "$0")/.."
CMD=$1; shift
for spec in "$@"; do
  label=${spec%%:*}; rest=${spec#*:}
  flags=${rest%%@*}; src=""
  [ "$rest" != "$flags" ] && src=${rest#*@}
  d=/tmp/lv_$label; mkdir -p $d
  for f in paper_2502_17421_b200/csrc/*.cu; do
    ff=$f
    if [ -n "$src" ] && [ "$(basename $f)" = prefix_tc.cu ]; then ff=$(dirname $f)/_variant_prefix_tc.cu; cp $src $ff; fi
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Iinclude $flags -c $ff -o $d/$(basename $f).o &
  done
  wait
  rm -f paper_2502_17421_b200/csrc/_variant_prefix_tc.cu
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libhta.so $d/*.o -ldl -lpthread
  echo "== $label [$flags] ${src}"
  HTA_LIB=$d/libhta.so bash -c "$CMD"
done
