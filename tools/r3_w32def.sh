#!/bin/bash
# Product build with 32-vector blocks from 2048-vector thetas: full GPU suite, C4 window errors, chi = 1024 and 512 benches.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/w32def_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|^E  +(Assert|assert)" gpurun_out/w32def_pytest.log | head -6
timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w" | tr '\n' ' '; echo
timeout 900 python bench.py --chi 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/w32def_chi1024.json 2>/dev/null; tail -1 gpurun_out/w32def_chi1024.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chi1024', round(d['value'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'], d['gpu_launches'])"
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chi512', round(d['value'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'], d['svd_sweeps'])"
