#!/bin/bash
# Dev loop on the GPU box: parity subset, sweep timing, per-kernel ncu times.
set -o pipefail
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_svd.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu 2>&1 | tail -3
MPSIM_SWEEP_DEBUG=1 NGATES=32 timeout 300 python tools/ncu_case.py 2>&1 | grep -E "sweep|ok" | cut -c1-220
timeout 300 python tools/perf_probe.py 512 32 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -s 30 -c 9 --csv --log-file gpurun_out/iter.csv env NGATES=32 python tools/ncu_case.py > /dev/null 2>&1
python tools/ncu_parse.py gpurun_out/iter.csv
