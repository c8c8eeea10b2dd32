#!/bin/bash
# Per-kernel ncu counters (time, DRAM bytes, DRAM throughput, DMMA / FP64 pipe) for every
# kernel of one bench step and of one centre-move sweep (tools/qr_case.py).
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $M --clock-control none -k regex:"qrp|theta|cross_gram|ortho|derijk|truncate|copy_factor" --csv --log-file gpurun_out/r3_kern_gate.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-pipeline > /dev/null 2>&1
REPS=1 timeout 900 ncu --metrics $M --clock-control none -k regex:"site_qr|cgemm|site_matrix" --csv --log-file gpurun_out/r3_kern_qr.csv python tools/qr_case.py > /dev/null 2>&1
ls -la gpurun_out/r3_kern_*.csv
