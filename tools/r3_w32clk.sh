#!/bin/bash
# W = 16 vs W = 32 sweeps on the full bench: rate and power-capped SM clock (A/B build).
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for rep in 1 2; do for v in MPSIM_W32=0 MPSIM_W32=1; do
  env $v timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'])"
done; done
cp /tmp/product.so $L
