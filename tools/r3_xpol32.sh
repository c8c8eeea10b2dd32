#!/bin/bash
# Cross-only EVD policy knobs at chi = 1024 (W = 32 sweeps), A/B build, alternating on one box.
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for rep in 1 2; do for v in "MPSIM_ALT_CROSS=2" "MPSIM_ALT_CROSS=3" "MPSIM_CROSS_RMS=0.1" "MPSIM_CROSS_SWEEPS=6 MPSIM_CROSS_RMS=0.2"; do
  env $v timeout 900 python bench.py --chi 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'])"
done; done
cp /tmp/product.so $L
