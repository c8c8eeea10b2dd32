mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_queries.py tests/test_gpu_acceptance.py tests/test_gpu_shard.py tests/test_cpp_facade.py -q -m gpu -x > gpurun_out/r2_pytest15.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest15.log
REPS=3 timeout 300 python tools/qr_case.py > gpurun_out/r2_qr_case15.txt 2>&1
timeout 300 python tools/sample_probe.py > gpurun_out/r2_sample_probe15.txt 2>&1
