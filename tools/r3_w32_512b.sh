#!/bin/bash
# chi = 512: W = 16 vs W = 32 on the final code (A/B build, MPSIM_W32=0 / 1), alternating on one box, then W = 32 accuracy at chi = 512 sizes.
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for rep in 1 2 3; do for w in 0 1; do
  MPSIM_W32=$w timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chi512 W32=$w', round(d['value'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'])"
done; done
echo "== accuracy MPSIM_W32=1"
cp /tmp/product.so $L
