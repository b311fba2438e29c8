#!/bin/bash
# Experiment build: libtcl with a kernel's phase trace -> exp/libtcl_trace.so
#   KERNEL=inconv (default) | ... ; EXTRA_DEFS: more -D flags
set -e
cd "$(dirname "$0")/.."
python -m paper_2604_12891_b200.build > /dev/null
K=${KERNEL:-inconv}
KU=$(echo $K | tr a-z A-Z)
B=paper_2604_12891_b200/build
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  -DTCL_${KU}_TRACE ${EXTRA_DEFS} -Iinclude -Ipaper_2604_12891_b200/csrc -c paper_2604_12891_b200/csrc/kernels/$K.cu -o /tmp/${K}_trace.o
objs=$(ls $B/*.o | grep -v kernels_$K.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/libtcl_trace.so $objs /tmp/${K}_trace.o -lnccl
echo built exp/libtcl_trace.so
