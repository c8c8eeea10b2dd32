#!/bin/bash
# Final round-2 (second session) evidence on one B200: full GPU suite, smoke,
# bench (default and other bond dimensions), ncu launch list of one bench step,
# ncu --set full of one 64-gate sweep launch, centre-move timings.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/rf4_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/rf4_pytest.log; tail -3 gpurun_out/rf4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf4_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/rf4_smoke.log; tail -2 gpurun_out/rf4_smoke.log
timeout 900 python bench.py > gpurun_out/rf4_bench.json 2> gpurun_out/rf4_bench.err; tail -1 gpurun_out/rf4_bench.json | cut -c1-160
timeout 900 python bench.py --chi 128 --qubits 1000 --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/rf4_bench_chi128.json 2>&1
timeout 900 python bench.py --chi 1024 --steps 2 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/rf4_bench_chi1024.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rf4_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-pipeline > gpurun_out/rf4_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:jacobi_sweep -s 3 -c 1 -o gpurun_out/rf4_sweep -f env NGATES=64 python tools/ncu_case.py > gpurun_out/rf4_sweep.log 2>&1
REPS=3 timeout 300 python tools/qr_case.py > gpurun_out/rf4_qr_case.txt 2>&1
timeout 300 python tools/sample_probe.py > gpurun_out/rf4_sample_probe.txt 2>&1
echo done
