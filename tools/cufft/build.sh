#!/bin/bash
# cuFFT-with-callbacks baseline (static cuFFT: callbacks need it); output stays in tools/cufft/
set -e
cd "$(dirname "$0")"
ARCH="-gencode arch=compute_100a,code=sm_100a"
nvcc -O3 -std=c++17 $ARCH -Xcompiler -fPIC -rdc=true -c cufft_baseline.cu -o cufft_baseline.o
nvcc $ARCH -Xcompiler -fPIC -dlink cufft_baseline.o -o cufft_dlink.o -lcufft_static -lculibos
g++ -shared -o libcufft_baseline.so cufft_baseline.o cufft_dlink.o -L/usr/local/cuda/lib64 -lcufft_static -lculibos -lcudart_static -lpthread -ldl -lrt
echo built tools/cufft/libcufft_baseline.so
