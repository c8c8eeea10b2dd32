#!/bin/bash
# One-sweep timing: FP64 EVD vs FP32 EVD + NS polar vs FP32 EVD without NS (profiling only).
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for rep in 1 2; do
for v in "MPSIM_EVD32_MAXOFF=0 MPSIM_PHASE_PROBE=4" "MPSIM_EVD32_MAXOFF=0 MPSIM_PHASE_PROBE=0" "MPSIM_EVD32_MAXOFF=1e-2 MPSIM_PHASE_PROBE=0" "MPSIM_EVD32_MAXOFF=1e-2 MPSIM_PHASE_PROBE=5"; do
  echo "== $v"; env $v MPSIM_SWEEP_DEBUG=1 timeout 300 python tools/perf_probe.py 512 128 2>&1 | grep -E "sweep 0:|per visit" | head -2 | cut -c1-230
done; done
cp /tmp/product.so $L
