mkdir -p gpurun_out
nproc > gpurun_out/r2_nproc.txt; free -g >> gpurun_out/r2_nproc.txt
timeout 1500 python -m pytest tests -q -m gpu -k "not golden" -x --durations=15 > gpurun_out/r2_pytest1.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest1.log
timeout 600 python bench.py --steps 4 --warmup 3 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
echo "bench rc=$?" >> gpurun_out/r2_bench1.err
