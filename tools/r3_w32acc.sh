#!/bin/bash
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
MPSIM_W32=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_golden.py tests/test_gpu_parity.py -q -m gpu 2>&1 | grep -E "^E  +(Assert|assert)|passed|failed|FAILED" | head -8
MPSIM_W32=1 timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w" | tr '\n' ' '; echo
cp /tmp/product.so $L
