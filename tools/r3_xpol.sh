#!/bin/bash
# Cross-only EVD policy knobs on the full bench (A/B build), alternating on one box.
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for rep in 1 2; do for v in "MPSIM_ALT_CROSS=2" "MPSIM_ALT_CROSS=3" "MPSIM_CROSS_RMS=0.1" "MPSIM_CROSS_SWEEPS=8 MPSIM_CROSS_RMS=0.05" "MPSIM_ALT_CROSS=0"; do
  env $v timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'])"
done; done
cp /tmp/product.so $L
