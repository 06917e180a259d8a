#!/bin/bash
# Build an A/B variant of libfsil.so with extra nvcc defines: tools/ab_build.sh <tag> [-DX=Y ...]
# -> ab/libfsil_<tag>.so (git-ignored; travels to the GPU box; select with FSIL_LIB_PATH)
set -e
cd "$(dirname "$0")/.."
tag=$1; shift
mkdir -p ab/obj_$tag
C=paper_2303_14102_b200/csrc
objs=()
for f in densify aggregate score_ffma score_tc score_tc2 naive finalize capi; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -O3 \
    -Iinclude -I$C "$@" -c $C/$f.cu -o ab/obj_$tag/$f.o &
  objs+=(ab/obj_$tag/$f.o)
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/libfsil_$tag.so "${objs[@]}" -Xcompiler -fPIC
echo "built ab/libfsil_$tag.so"
