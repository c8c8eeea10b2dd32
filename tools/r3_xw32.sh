#!/bin/bash
# W = 32 sweep with the cross-entry test in pre-asymptotic visits (xw32.so) vs the product build (base.so) at chi = 1024;
# W = 32 vs W = 16 at chi = 512 on the same code (xw32ab.so, MPSIM_W32); then accuracy with xw32.so.
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so
for rep in 1 2; do
  for v in base xw32; do
    cp tools/ab_libs/$v.so $L
    timeout 900 python bench.py --chi 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chi1024 $v', round(d['value'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'])"
  done
  cp tools/ab_libs/xw32ab.so $L
  for w in 0 1; do
    MPSIM_W32=$w timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chi512 W32=$w', round(d['value'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'])"
  done
done
cp tools/ab_libs/xw32.so $L
echo "== accuracy xw32"
timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w" | tr '\n' ' '; echo
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  +(Assert|assert)|passed|failed|FAILED" | head -8
cp /tmp/product.so $L
