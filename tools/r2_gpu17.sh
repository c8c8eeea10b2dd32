mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_queries.py -q -m gpu > gpurun_out/r2_pytest17.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest17.log
