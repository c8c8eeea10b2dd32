#!/bin/bash
# Round-end evidence: bench line, launch list of one bench step, full capture of one pair-kernel launch.
mkdir -p gpurun_out
python bench.py --steps 4 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-pipeline > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:jacobi_sweep -s 3 -c 1 \
  -o gpurun_out/full_pair env NGATES=64 python tools/ncu_case.py > gpurun_out/ncu_full.log 2>&1
tail -c 600 gpurun_out/bench.json
