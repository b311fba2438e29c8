#!/bin/bash
# Experiment A/B build: libtcl with one source compiled with extra -D flags -> exp/libtcl_ab.so
#   SRC=kernels/mixer_split.cu EXTRA_DEFS="-DTCL_SCAN_POLY=1" bash exp/ab_build.sh
set -e
cd "$(dirname "$0")/.."
python -m paper_2604_12891_b200.build > /dev/null
B=paper_2604_12891_b200/build
O=$(echo $SRC | tr '/' '_'); O=${O%.cu}.o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr \
  ${EXTRA_DEFS} -Iinclude -Ipaper_2604_12891_b200/csrc -c paper_2604_12891_b200/csrc/$SRC -o /tmp/ab_$O
objs=$(ls $B/*.o | grep -v "$O")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp/libtcl_ab.so $objs /tmp/ab_$O -lnccl
echo built exp/libtcl_ab.so
