#!/bin/bash
# Baseline on a fresh box: bench (N=1) and the per-sweep profile of one 128-gate layer.
mkdir -p gpurun_out
timeout 600 python bench.py --steps 4 --warmup 3 --no-pipeline --no-cpu-baseline > gpurun_out/r3_base_bench.json 2> gpurun_out/r3_base_bench.err
tail -1 gpurun_out/r3_base_bench.json | cut -c1-400
MPSIM_SWEEP_DEBUG=1 timeout 300 python tools/perf_probe.py 512 128 > gpurun_out/r3_base_probe.txt 2>&1
tail -20 gpurun_out/r3_base_probe.txt
