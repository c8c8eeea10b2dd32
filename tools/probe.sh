#!/bin/bash
# Phase timing of the pair kernel: one sweep over 64 gates, Gram only / Gram+EVD / full.
for pr in 1 2 0; do
  echo "== probe $pr"; MPSIM_PHASE_PROBE=$pr MPSIM_SWEEP_DEBUG=1 NGATES=64 timeout 300 python tools/ncu_case.py 2>&1 | grep "sweep 0" | cut -c1-200
done
