#!/bin/bash
# Rotation test + maxoff from the cross entries only in pre-asymptotic visits (MPSIM_XTEST=1) vs the full test: bench A/B with clocks, then accuracy (A/B build).
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for rep in 1 2 3; do for v in MPSIM_XTEST=0 MPSIM_XTEST=1; do
  env $v timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'])"
done; done
echo "== accuracy MPSIM_XTEST=1"
MPSIM_XTEST=1 timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w" | tr '\n' ' '; echo
MPSIM_XTEST=1 timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | grep -E "^E  +(Assert|assert)|passed|failed|FAILED" | head -8
cp /tmp/product.so $L
