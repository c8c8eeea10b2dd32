#!/bin/bash
# Alternating A/B of prebuilt libraries on the 128-gate chi=512 layer probe
# (tools/perf_probe.py), optionally the parity subset on the product build first.
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so
if [ -n "$TESTS" ]; then timeout 900 python -m pytest $TESTS -x -q -m gpu 2>&1 | tail -3; fi
for rep in 1 2 3; do
  for l in ${LIBS:-tools/ab_libs/base.so tools/ab_libs/new.so}; do
    cp $l $L
    echo "== $l $(env $ENVV timeout 300 python tools/perf_probe.py 512 128 2>&1 | tail -2 | awk '{print $4}' | tr '\n' ' ')"
  done
done
cp /tmp/product.so $L
