#!/bin/bash
# Sweep-policy knobs on the current build: layer timing (128 gates, chi=512) and C4-window errors (A/B build).
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for v in "MPSIM_JTOL=4" "MPSIM_JTOL=8" "MPSIM_ALT_CROSS=3" "MPSIM_CROSS_SWEEPS=6" "MPSIM_JTOL=4"; do
  echo "== $v $(env $v timeout 300 python tools/perf_probe.py 512 128 2>&1 | tail -2 | awk '{print $4, $6}' | tr '\n' ' ')"
  env $v timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w" | tr '\n' ' '; echo
done
cp /tmp/product.so $L
