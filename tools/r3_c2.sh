#!/bin/bash
# The C2 full-size parity test with its traceback, product build then A/B variants.
L=paper_2601_04422_b200/libmpsim_gpu.so
timeout 600 python -m pytest "tests/test_gpu_fullsize.py::test_c2_full_size" -x -q -m gpu --tb=short 2>&1 | grep -E "^E |passed|failed" | head -20
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for v in ${VARIANTS:-"MPSIM_EVD32_MAXOFF=0"}; do
  echo "== $v"; env $v timeout 600 python -m pytest "tests/test_gpu_fullsize.py::test_c2_full_size" -x -q -m gpu --tb=short 2>&1 | grep -E "^E |passed|failed" | head -20
done
cp /tmp/product.so $L
