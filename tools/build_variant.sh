#!/bin/bash
# Build libcbp_cuda.so from the in-tree sources with extra nvcc defines into exp/<name>/
# (A/B kernel experiments, loaded with CBP_CUDA_LIB). usage: build_variant.sh name -DX=1 ...
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
obj=/tmp/cbp_variant_$name; rm -rf "$obj"; mkdir -p "$obj" "$root/exp/$name"
cd "$root/paper_1203_4874_b200/csrc"
for f in *.cu; do
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr \
    "$@" -dc -o "$obj/${f%.cu}.o" "$f" &
done
g++ -O2 -std=c++17 -fPIC -Wall -c -o "$obj/enc.o" cbp_encoder_host.cpp
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/exp/$name/libcbp_cuda.so" "$obj"/*.o -cudart static
echo "built exp/$name/libcbp_cuda.so"
