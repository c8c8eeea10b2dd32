#!/bin/bash
# A/B of env settings on the 32-gate chi=512 case: usage ab_env.sh "VAR=a" "VAR=b" ...
# The MPSIM_* A/B switches are read only by an A/B build of the library:
#   make -C paper_2601_04422_b200/csrc clean && make -C paper_2601_04422_b200/csrc AB=1
for e in "$@"; do
  echo "== $e"; env $e NGATES=32 timeout 300 python tools/ncu_case.py 2>&1 | grep -o "'sweeps': [0-9]*\|'jacobi_ms': [0-9.]*" | tr '\n' ' '; echo
  env $e timeout 300 python tools/perf_probe.py 512 32 2>&1 | tail -2
done
