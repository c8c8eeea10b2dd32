#!/bin/bash
# A/B of prebuilt library variants: tools/ab_lib.sh tools/ab_libs/a.so tools/ab_libs/b.so
for l in "$@"; do
  cp "$l" paper_2601_04422_b200/libmpsim_gpu.so
  echo "== $l"; NGATES=32 timeout 300 python tools/ncu_case.py 2>&1 | grep -o "'sweeps': [0-9]*\|'jacobi_ms': [0-9.]*" | tr '\n' ' '; echo
  timeout 300 python tools/perf_probe.py 512 64 2>&1 | tail -1
done
