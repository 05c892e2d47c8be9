#!/bin/bash
# Build + run the block-kernel probe on the GPU box (see zblas_probe.cu).
set -e
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo ${PROBE_FLAGS} -I paper_2306_16778_b200/csrc tools/zblas_probe.cu \
  paper_2306_16778_b200/csrc/*.cu paper_2306_16778_b200/csrc/poles.cpp -o /tmp/zp 2>/dev/null
/tmp/zp
