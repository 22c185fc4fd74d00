#!/bin/bash
# Experiments: build the product library with extra -D flags into variants/<name>.so
# (load it with KIFMM_LIB=variants/<name>.so).  usage: tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
cd "$(dirname "$0")/.."
make -s lib >/dev/null
mkdir -p variants build/var
/usr/local/cuda/bin/nvcc -std=c++20 -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -fopenmp -ccbin /usr/bin/g++ \
  -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Iinclude -Ipaper_2303_08394_b200/csrc/host \
  -Ipaper_2303_08394_b200/csrc/cuda -DKIFMM_EXPERIMENTS $2 -c paper_2303_08394_b200/csrc/cuda/plan.cu -o build/var/$1.o
/usr/local/cuda/bin/nvcc -shared -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -o variants/$1.so \
  build/host/*.o build/var/$1.o -cudart static -Xcompiler -fopenmp -ldl -lpthread -lrt
