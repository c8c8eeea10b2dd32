mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -k "not golden" --durations=12 > gpurun_out/r2_pytest4.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest4.log
timeout 600 python bench.py --steps 4 --warmup 3 --no-pipeline > gpurun_out/r2_bench4.json 2> gpurun_out/r2_bench4.err
echo "bench rc=$?" >> gpurun_out/r2_bench4.err
timeout 300 python tools/qr_case.py > gpurun_out/r2_qr_case.txt 2>&1
REPS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 3000 --csv --log-file gpurun_out/r2_qr_ncu.csv python tools/qr_case.py > /dev/null 2>&1
python tools/ncu_parse.py gpurun_out/r2_qr_ncu.csv > gpurun_out/r2_qr_ncu.txt 2>&1
MPSIM_SWEEP_DEBUG=1 NGATES=64 timeout 300 python tools/ncu_case.py > gpurun_out/r2_sweeps.txt 2>&1
