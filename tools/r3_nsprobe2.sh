#!/bin/bash
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for rep in 1 2; do
for v in "MPSIM_EVD32_MAXOFF=0" "MPSIM_EVD32_MAXOFF=1e-2"; do
  echo "== $v"; env $v MPSIM_SWEEP_DEBUG=1 timeout 300 python tools/perf_probe.py 512 128 2>&1 | grep -E "sweep 0:|per visit|rep" | sed -n '1,2p;$p' | cut -c1-230
done; done
for v in "MPSIM_EVD32_MAXOFF=1e-2"; do echo "== C2/fullsize with $v"; env $v timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | grep -E "^E |passed|failed" | head; done
cp /tmp/product.so $L
