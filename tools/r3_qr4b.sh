#!/bin/bash
# Product build with the n >= 512 four-step default: full GPU suite, bench, C4 errors.
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E  +(Assert|assert)|passed|failed" | head -6
timeout 600 python tools/c4_errors.py c4_window 2>&1 | grep -E "amp rel|max rel w" | tr '\n' ' '; echo
timeout 900 python bench.py --no-pipeline > gpurun_out/r3_qr4b_bench.json 2>/dev/null; tail -1 gpurun_out/r3_qr4b_bench.json | cut -c1-120
python -c "import json; d=json.loads(open('gpurun_out/r3_qr4b_bench.json').read().strip().splitlines()[-1]); print(d['clocks']['sm_mhz'], d['svd_sweeps'], d['roofline']['frac'])"
