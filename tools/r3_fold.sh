#!/bin/bash
# 16-vector-block pair EVD with the Hermitian-folded G update (-DMPSIM_EVD_FOLD=2, fold.so) vs the product (base.so):
# chi = 512 bench alternating on one box, then accuracy with fold.so.
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so
for rep in 1 2 3; do for v in base fold; do
  cp tools/ab_libs/$v.so $L
  timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chi512 $v', round(d['value'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'])"
done; done
cp tools/ab_libs/fold.so $L
echo "== accuracy fold"
timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w" | tr '\n' ' '; echo
timeout 600 python tools/c2_spread.py 2>&1 | tail -2
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  +(Assert|assert)|passed|failed|FAILED" | head -8
cp /tmp/product.so $L
