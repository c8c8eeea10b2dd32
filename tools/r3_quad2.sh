#!/bin/bash
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for v in "MPSIM_QUAD=1e-12 MPSIM_ORTHO=0" "MPSIM_QUAD=1e-12 MPSIM_ORTHO=1" "MPSIM_QUAD=1e-12 MPSIM_ORTHO=1 MPSIM_QR=0"; do
  echo "== $v"; env $v timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w|Z>"
  env $v timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -k c2 2>&1 | tail -1
done
cp /tmp/product.so $L
