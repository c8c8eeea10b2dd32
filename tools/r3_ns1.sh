#!/bin/bash
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for v in "MPSIM_EVD32_MAXOFF=1e-2 MPSIM_NS_ITERS=1" "MPSIM_EVD32_MAXOFF=1e-2 MPSIM_NS_ITERS=2"; do
  echo "== $v"; env $v timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w|Z>" | tr '\n' ' '; echo
  env $v timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_golden.py -q -m gpu 2>&1 | tail -1
done
for rep in 1 2 3; do for v in "MPSIM_EVD32_MAXOFF=0" "MPSIM_EVD32_MAXOFF=1e-2 MPSIM_NS_ITERS=1"; do echo "== $v $(env $v timeout 300 python tools/perf_probe.py 512 128 2>&1 | tail -2 | awk '{print $4}' | tr '\n' ' ')"; done; done
cp /tmp/product.so $L
