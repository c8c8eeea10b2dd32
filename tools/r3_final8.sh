#!/bin/bash
# Final evidence of round 2 (second session) on one B200: full GPU suite, smoke, bench.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -rxX --durations=8 > gpurun_out/rf15_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rf15_pytest.log
grep -E "passed|failed|XFAIL|FAILED|rc=" gpurun_out/rf15_pytest.log | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf15_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rf15_smoke.log; tail -2 gpurun_out/rf15_smoke.log
timeout 900 python bench.py > gpurun_out/rf15_bench.json 2> gpurun_out/rf15_bench.err; tail -1 gpurun_out/rf15_bench.json | cut -c1-180
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/rf15_bench_ref.json 2> gpurun_out/rf15_bench_ref.err; tail -1 gpurun_out/rf15_bench_ref.json | cut -c1-180
timeout 900 python bench.py --chi 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/rf15_bench_chi1024.json 2>/dev/null; tail -1 gpurun_out/rf15_bench_chi1024.json | cut -c1-120
KREGEX=jacobi_sweep_w32 SKIP=3 OUT=w32_512 CHI=512 bash tools/r3_ncu_full.sh > gpurun_out/ncu_w32_512.log 2>&1; tail -2 gpurun_out/ncu_w32_512.log
