mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_queries.py tests/test_gpu_acceptance.py tests/test_gpu_shard.py tests/test_cpp_facade.py -q -m gpu -x > gpurun_out/r2_pytest7.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest7.log
REPS=3 timeout 300 python tools/qr_case.py > gpurun_out/r2_qr_case7.txt 2>&1
timeout 300 python tools/sample_probe.py > gpurun_out/r2_sample_probe7.txt 2>&1
REPS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 5000 --csv --log-file gpurun_out/r2_qr_ncu7.csv python tools/qr_case.py > /dev/null 2>&1
python tools/ncu_parse.py gpurun_out/r2_qr_ncu7.csv > gpurun_out/r2_qr_ncu7.txt 2>&1
NGATES=64 timeout 900 ncu --set full --import-source on --clock-control none -k regex:jacobi_sweep -s 3 -c 1 -o gpurun_out/r2_jacobi_sweep python tools/ncu_case.py > gpurun_out/r2_jacobi_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/r2_launches_bench.log 2>&1
