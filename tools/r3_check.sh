#!/bin/bash
# Full GPU suite, smoke and the default bench on the product build.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r3_pytest.log
tail -3 gpurun_out/r3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r3_smoke.log
timeout 900 python bench.py > gpurun_out/r3_bench.json 2> gpurun_out/r3_bench.err; echo "bench rc=$?"
tail -1 gpurun_out/r3_bench.json | cut -c1-300
