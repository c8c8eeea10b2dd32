#!/bin/bash
# Four-step QR preconditioning (A/B build): parity subset and layer timing / sweep counts.
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
MPSIM_QR=4 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_svd.py tests/test_gpu_golden.py -q -m gpu -x 2>&1 | grep -E "^E  +(Assert|assert)|passed|failed" | head -4
MPSIM_QR=4 timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w" | tr '\n' ' '; echo
for rep in 1 2 3; do for v in MPSIM_QR=2 MPSIM_QR=4; do echo "== $v $(env $v timeout 300 python tools/perf_probe.py 512 128 2>&1 | tail -2 | awk '{print $4, $7}' | tr '\n' ' ')"; done; done
cp /tmp/product.so $L
