#!/bin/bash
# Build an alternative libtrigraph_b200.so with intersect.cu compiled under
# extra -D flags (kernel-variant experiments); load it with TG_LIB_PATH.
#   tools/build_variant.sh u8b5 -DTG_UNROLL=8 -DTG_WBLOCKS=5
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_1706_05151_b200/csrc
make -s -C "$C"
mkdir -p "$R/variants/$name"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr "$@" -c "$C/intersect.cu" \
  -o "$R/variants/$name/intersect.o" 2> "$R/variants/$name/ptxas.log"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared \
  -o "$R/variants/$name/libtrigraph_b200.so" "$R/variants/$name/intersect.o" \
  "$C/build/prep.o" "$C/build/exchange.o" "$C/build/engine.o" "$C/build/generators.o" -lpthread
grep -A3 "k_intersect_warpILb0ELb0ELb0ELb0ENS0_8RowsApex" "$R/variants/$name/ptxas.log" | grep -E "registers|spill"
