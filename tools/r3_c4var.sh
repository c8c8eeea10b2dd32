#!/bin/bash
# C4-window errors under A/B variants (A/B build).
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for v in "MPSIM_JTOL=4" "MPSIM_JTOL=2" "MPSIM_JTOL=8" "MPSIM_QR=0" "MPSIM_QR=1" "MPSIM_EXACT_CACHE=0 MPSIM_INBLOCK=0"; do
  echo "== $v"; env $v timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w|Z>"
done
cp /tmp/product.so $L
