#!/bin/bash
# W = 32 cross-only Gram passes in cross-only EVDs two rounds in three (-DMPSIM_W32_ALT=3, alt3.so) vs the product (base.so) at chi = 1024; then accuracy.
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so
for rep in 1 2 3; do for v in base alt3; do
  cp tools/ab_libs/$v.so $L
  timeout 900 python bench.py --chi 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chi1024 $v', round(d['value'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'])"
done; done
cp tools/ab_libs/alt3.so $L
echo "== accuracy alt3"
timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w" | tr '\n' ' '; echo
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  +(Assert|assert)|passed|failed|FAILED" | head -8
cp /tmp/product.so $L
