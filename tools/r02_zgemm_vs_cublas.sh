#!/usr/bin/env bash
# The hand-written 3M DMMA zgemm against cuBLAS ZGEMM (torch.matmul, complex128) on the C4 GEMM shapes.
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2306_16778_b200/csrc -I include \
  tools/zgemm_probe.cu paper_2306_16778_b200/csrc/*.cu paper_2306_16778_b200/csrc/poles.cpp -o /tmp/zgp 2>/dev/null || { echo build failed; exit 1; }
echo "== pfx::zgemm (3M, TMA-staged, batch 12; flops counted as 8mnk, fwd_* triangle-aware)"
/tmp/zgp
echo "== cuBLAS ZGEMM (torch.matmul complex128)"
python tools/zgemm_yardstick.py
