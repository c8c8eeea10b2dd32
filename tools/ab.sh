#!/bin/bash
# A/B of Jacobi modes on the 32-gate chi=512 case: total Jacobi ms and sweeps.
for mode in "$@"; do
  echo "== $mode"; MPSIM_JACOBI=$mode NGATES=32 timeout 300 python tools/ncu_case.py 2>&1 | grep -o "'sweeps': [0-9]*\|'jacobi_ms': [0-9.]*" | tr '\n' ' '; echo
  MPSIM_JACOBI=$mode timeout 300 python tools/perf_probe.py 512 32 2>&1 | tail -2
done
