#!/bin/bash
# instrumented build (per-section k_pcg clocks) → paper_2504_12908_b200/libtaccel_cuda_clk.so
cd "$(dirname "$0")/.." && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -DTAC_CLOCKS -o paper_2504_12908_b200/libtaccel_cuda_clk.so paper_2504_12908_b200/csrc/kernels.cu paper_2504_12908_b200/csrc/api.cu -lcudart
