# Final round-2 evidence on one B200: full GPU suite, smoke, bench (default
# and other bond dimensions), ncu of the 128-gate sweep launch and of the QR
# kernels (gate-path preconditioning and centre moves).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/rf_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/rf_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/rf_smoke.log
timeout 900 python bench.py > gpurun_out/rf_bench.json 2> gpurun_out/rf_bench.err
timeout 900 python bench.py --chi 128 --qubits 1000 --steps 3 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/rf_bench_chi128.json 2>&1
timeout 900 python bench.py --chi 1024 --steps 2 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/rf_bench_chi1024.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:jacobi_sweep -s 3 -c 1 -o gpurun_out/rf_sweep128 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-pipeline > gpurun_out/rf_sweep128.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"qrp|theta|cross_gram|derijk" -c 400 --csv --log-file gpurun_out/rf_gatepath_ncu.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-pipeline > /dev/null 2>&1
python tools/ncu_parse.py gpurun_out/rf_gatepath_ncu.csv > gpurun_out/rf_gatepath_ncu.txt 2>&1
REPS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 3000 --csv --log-file gpurun_out/rf_qr_ncu.csv python tools/qr_case.py > /dev/null 2>&1
python tools/ncu_parse.py gpurun_out/rf_qr_ncu.csv > gpurun_out/rf_qr_ncu.txt 2>&1
REPS=3 timeout 300 python tools/qr_case.py > gpurun_out/rf_qr_case.txt 2>&1
timeout 300 python tools/sample_probe.py > gpurun_out/rf_sample_probe.txt 2>&1
