#!/bin/bash
L=paper_2601_04422_b200/libmpsim_gpu.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_svd.py tests/test_gpu_golden.py -q -m gpu 2>&1 | tail -1
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for rep in 1 2 3; do for v in MPSIM_QR_LOOKAHEAD=0 MPSIM_QR_LOOKAHEAD=1; do echo "== $v $(env $v timeout 300 python tools/perf_probe.py 512 128 2>&1 | tail -2 | awk '{print $4}' | tr '\n' ' ')"; done; done
cp /tmp/product.so $L
