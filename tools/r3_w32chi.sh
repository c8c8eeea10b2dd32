#!/bin/bash
# W = 16 vs W = 32 sweeps at chi = 1024 (2048-vector thetas) and chi = 512, A/B build, alternating on one box.
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for rep in 1 2; do for v in MPSIM_W32=0 MPSIM_W32=1; do
  env $v timeout 900 python bench.py --chi 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chi1024 $v', round(d['value'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'])"
done; done
cp /tmp/product.so $L
