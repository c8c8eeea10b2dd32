#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_svd.py -q -m gpu -k subspace 2>&1 | grep -E "^E  +(Assert|assert)|passed|failed" | head -6
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
echo "== old exit (MPSIM_QUAD=1e-9)"; MPSIM_QUAD=1e-9 timeout 900 python -m pytest tests/test_gpu_svd.py -q -m gpu -k subspace 2>&1 | grep -E "^E  +(Assert|assert)|passed|failed" | head -6
cp /tmp/product.so $L
