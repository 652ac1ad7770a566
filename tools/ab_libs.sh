#!/bin/bash
# A/B of two builds on one box (diagnostics): tools/ab_libs.sh LIB_A LIB_B [workload ...]
A=${1:-paper_2502_17421_b200/libhta_base.so}; B=${2:-paper_2502_17421_b200/libhta.so}; shift 2
for i in 1 2; do for L in $A $B; do HTA_LIB=$L python tools/fuse_probe.py "$@"; done; done
