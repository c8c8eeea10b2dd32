#!/bin/bash
# C4-window fixture test on the product build and on prebuilt A/B libraries.
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so
echo "== product"; timeout 900 python -m pytest tests/test_gpu_golden.py::test_c4_window_reaching_chi1024_against_fixture -q -m gpu 2>&1 | grep -E "^E  +AssertionError|passed|failed" | head -3
for l in ${LIBS:-tools/ab_libs/base.so}; do
  cp $l $L; echo "== $l $ENVV"; env $ENVV timeout 900 python -m pytest tests/test_gpu_golden.py::test_c4_window_reaching_chi1024_against_fixture -q -m gpu 2>&1 | grep -E "^E  +AssertionError|passed|failed" | head -3
done
cp /tmp/product.so $L
