#!/bin/bash
# Quadratic-phase exit threshold: C4-window errors and layer timing (A/B build).
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for v in "MPSIM_QUAD=1e-9" "MPSIM_QUAD=1e-12" "MPSIM_QUAD=0"; do
  echo "== $v"; env $v timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w|Z>"
  env $v timeout 300 python tools/perf_probe.py 512 128 2>&1 | tail -2
done
for v in "MPSIM_QUAD=1e-9" "MPSIM_QUAD=1e-12" "MPSIM_QUAD=0"; do echo "== $v"; env $v timeout 300 python tools/perf_probe.py 512 128 2>&1 | tail -2; done
cp /tmp/product.so $L
