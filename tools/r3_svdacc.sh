#!/bin/bash
# Kept-subspace accuracy of the GPU SVD on the C4 window's truncating thetas, per A/B variant.
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for v in "MPSIM_QUAD=1e-9" "MPSIM_QUAD=0" "MPSIM_QUAD=0 MPSIM_JTOL=1" "MPSIM_QR=0" "MPSIM_QR=0 MPSIM_QUAD=0" "MPSIM_ALT_CROSS=0 MPSIM_CROSS=0 MPSIM_INBLOCK=0 MPSIM_EXACT_CACHE=0"; do
  echo "== $v"; env $v MPSIM_SWEEP_DEBUG=1 timeout 600 python tools/c4_gate_svd.py tools/ab_libs/c4_thetas2.npz 2>&1 | grep -E "theta|sweep [0-9]+:" | cut -c1-200 | tail -30
done
cp /tmp/product.so $L
