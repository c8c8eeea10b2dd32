#!/bin/bash
# Kept-vector orthonormalisation: C4-window errors, parity subset, layer timing with / without (A/B build).
L=paper_2601_04422_b200/libmpsim_gpu.so
timeout 600 python tools/c4_errors.py c4_window 2>&1 | tail -12
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_svd.py tests/test_gpu_golden.py::test_c4_window_reaching_chi1024_against_fixture -q -m gpu -rxX 2>&1 | tail -4
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for rep in 1 2; do for v in MPSIM_ORTHO=0 MPSIM_ORTHO=1; do echo "== $v $(env $v timeout 300 python tools/perf_probe.py 512 128 2>&1 | tail -2 | awk '{print $4}' | tr '\n' ' ')"; done; done
cp /tmp/product.so $L
