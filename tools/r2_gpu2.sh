mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -k "not golden" --durations=10 > gpurun_out/r2_pytest2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest2.log
timeout 600 python bench.py --steps 4 --warmup 3 --no-pipeline > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err
echo "bench rc=$?" >> gpurun_out/r2_bench2.err
