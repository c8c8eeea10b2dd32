#!/bin/bash
# W = 32 sweeps with the FP32 inner sweep + FP64 polar factor in pre-asymptotic
# sweeps (MPSIM_EVD32_MAXOFF): accuracy gates, then the bench A/B with clocks.
L=paper_2601_04422_b200/libmpsim_gpu.so
cp $L /tmp/product.so; cp tools/ab_libs/ab.so $L
for x in 1e-2 1e-3; do
  echo "== W32 EVD32_MAXOFF=$x"
  MPSIM_W32=1 MPSIM_EVD32_MAXOFF=$x timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_svd.py -q -m gpu 2>&1 | grep -E "^E  +(Assert|assert)|passed|failed|FAILED" | head -8
  MPSIM_W32=1 MPSIM_EVD32_MAXOFF=$x timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w" | tr '\n' ' '; echo
done
for rep in 1 2; do for v in "MPSIM_W32=0" "MPSIM_W32=1" "MPSIM_W32=1 MPSIM_EVD32_MAXOFF=1e-2" "MPSIM_W32=1 MPSIM_EVD32_MAXOFF=1e-3"; do
  env $v timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'])"
done; done
cp /tmp/product.so $L
