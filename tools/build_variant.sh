#!/bin/bash
# Build an alternative libtrigraph_b200.so with one source (intersect or
# prep) compiled under extra -D flags (kernel-variant experiments); load it
# with TG_LIB_PATH.   tools/build_variant.sh u8b5 intersect -DTG_UNROLL=8 -DTG_WBLOCKS=5
set -e
name=$1; src=$2; shift 2
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_1706_05151_b200/csrc
make -s -C "$C"
D=$R/exp_variants/$name
mkdir -p "$D"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr "$@" -c "$C/$src.cu" \
  -o "$D/$src.o" 2> "$D/ptxas.log"
objs=""
for o in prep intersect exchange engine sparsify analytics order io gen window comm; do
  if [ "$o" = "$src" ]; then objs="$objs $D/$o.o"; else objs="$objs $C/build/$o.o"; fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared \
  -o "$D/libtrigraph_b200.so" $objs "$C/build/generators.o" -lpthread -ldl
grep -A3 -E "k_intersect_warpILb0ELb0ELb0ELb0ENS0_8RowsApex|k_orient_tilesILi2ELb0E" "$D/ptxas.log" | grep -E "registers|spill" || true
