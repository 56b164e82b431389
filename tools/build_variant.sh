#!/bin/bash
# build_variant.sh NAME "-DFLAG=.. ..." [SRC]: libott_b200.so variant at tools/variants/NAME.so for
# timing experiments: SRC (default the product ott_attend.cu) compiled with the extra flags, linked
# with the product objects of the other translation units (run `make -C paper_2505_10938_b200/csrc` first).
set -e
cd "$(dirname "$0")/../paper_2505_10938_b200/csrc"
OUT=../../tools/variants; mkdir -p $OUT/obj_$1
SRC=${3:-ott_attend.cu}
ARCH="-gencode arch=compute_100a,code=sm_100a"
F="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include -I. -Xptxas -v $2"
nvcc $F -c $SRC -o $OUT/obj_$1/a.o 2> $OUT/obj_$1/a.ptxas.txt || (cat $OUT/obj_$1/a.ptxas.txt; false)
O=../_lib/obj
nvcc $ARCH -shared -o $OUT/$1.so $O/ott_flush.o $OUT/obj_$1/a.o $O/ott_capi.o $O/ott_model.o $O/ott_api.o -lcudart
grep -A1 "attend_mma_kernelILi8ELi32" $OUT/obj_$1/a.ptxas.txt | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | head -3
