mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_queries.py tests/test_gpu_acceptance.py tests/test_gpu_shard.py tests/test_cpp_facade.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/r2_pytest8.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest8.log
REPS=3 timeout 300 python tools/qr_case.py > gpurun_out/r2_qr_case8.txt 2>&1
timeout 300 python tools/sample_probe.py > gpurun_out/r2_sample_probe8.txt 2>&1
REPS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 3000 --csv --log-file gpurun_out/r2_qr_ncu8.csv python tools/qr_case.py > /dev/null 2>&1
python tools/ncu_parse.py gpurun_out/r2_qr_ncu8.csv > gpurun_out/r2_qr_ncu8.txt 2>&1
