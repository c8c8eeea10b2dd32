#!/bin/bash
# A/B of prebuilt library variants on the full bench: tools/ab_bench.sh a.so b.so (alternating, twice)
for rep in 1 2; do
  for l in "$@"; do
    cp "$l" paper_2601_04422_b200/libmpsim_gpu.so
    v=$(python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), d['clocks']['sm_mhz'])")
    echo "$l $v"
  done
done
