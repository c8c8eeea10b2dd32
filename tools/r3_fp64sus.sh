#!/bin/bash
# Sustained FP64 DMMA rate with SM clocks sampled alongside (nvidia-smi).
(for i in $(seq 1 16); do nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader; sleep 0.5; done) > gpurun_out/r3_fp64sus_clk.txt &
./tools/microbench/fp64_peak 8
wait
cat gpurun_out/r3_fp64sus_clk.txt | tail -8
