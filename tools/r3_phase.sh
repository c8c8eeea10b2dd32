#!/bin/bash
# Phase costs of one (first) persistent sweep over a 128-gate chi=512 layer (A/B build).
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for p in 0 1 2 4; do
  echo "== probe $p"
  MPSIM_SWEEP_CL=0 MPSIM_PHASE_PROBE=$p MPSIM_SWEEP_DEBUG=1 timeout 300 python tools/perf_probe.py 512 128 2>&1 | grep "sweep 0" | tail -1 | cut -c1-200
done
cp /tmp/product.so $L
