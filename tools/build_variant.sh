#!/bin/bash
# build_variant.sh NAME "-DFLAG=.. ..." : libott_b200.so variant at tools/variants/NAME.so (timing experiments)
set -e
cd "$(dirname "$0")/../paper_2505_10938_b200/csrc"
OUT=../../tools/variants; mkdir -p $OUT/obj_$1
ARCH="-gencode arch=compute_100a,code=sm_100a"
F="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include -Xptxas -v $2"
nvcc $F -fmad=false -c ott_flush.cu -o $OUT/obj_$1/f.o &
nvcc $F -c ott_attend.cu -o $OUT/obj_$1/a.o 2> $OUT/obj_$1/a.ptxas.txt &
nvcc $F -c ott_capi.cu -o $OUT/obj_$1/c.o &
nvcc $F -c ott_model.cu -o $OUT/obj_$1/m.o &
wait
nvcc $ARCH -shared -o $OUT/$1.so $OUT/obj_$1/f.o $OUT/obj_$1/a.o $OUT/obj_$1/c.o $OUT/obj_$1/m.o -lcudart
