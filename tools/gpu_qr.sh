#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
MPSIM_SWEEP_DEBUG=1 NGATES=32 timeout 300 python tools/ncu_case.py 2>&1 | grep -E "sweep|ok|rror" | cut -c1-220
for q in 1 0; do echo "== MPSIM_QR=$q"; MPSIM_QR=$q timeout 300 python tools/perf_probe.py 512 32 2>&1 | tail -2; done
