#!/bin/bash
# Build an A/B experiment copy of libaxb.so with extra -D flags into build/exp_<tag>/libaxb.so
# (load it with AXB_LIB_PATH=...; never the product library).
#   bash scripts/build_exp.sh norefill -DAXB_EXP_C64_NOREFILL
set -e
cd "$(dirname "$0")/.."
T=$1; shift
O=build/exp_$T; mkdir -p $O
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -warn-spills -Iinclude $*"
for s in paper_2002_09481_b200/csrc/*.cu; do
  b=$(basename $s .cu)
  if [ "$b" = axb_ftconv ] || [ "$b" = axb_depthwise ] || [ "$b" = axb_quant ] || [ ! -f build/$b.o ]; then nvcc $F -c -o $O/$b.o $s & else cp build/$b.o $O/$b.o; fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $O/libaxb.so $O/*.o
echo built $O/libaxb.so
