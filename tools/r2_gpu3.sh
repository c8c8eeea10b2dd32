# N=2 box: TMA theta parity subset, multi-GPU parity of the C++ shard layer,
# bench at N=2, theta TMA vs cp.async under ncu (AB build in a copy).
mkdir -p gpurun_out
export MASTER_ADDR=127.0.0.1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_shard.py tests/test_gpu_acceptance.py tests/test_gpu_fullsize.py -k "not bench_step" -q -x -m gpu > gpurun_out/r2_pytest3.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest3.log
MGPU_TMP=/tmp/mgpu timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/mgpu_check.py > gpurun_out/r2_mgpu2.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/r2_mgpu2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 2 --steps 3 --warmup 3 --no-pipeline > gpurun_out/r2_bench_n2.json 2> gpurun_out/r2_bench_n2.err
echo "bench2 rc=$?" >> gpurun_out/r2_bench_n2.err
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:theta --csv --log-file gpurun_out/r2_theta_tma.csv env NGATES=64 python tools/ncu_case.py > /dev/null 2>&1
rm -rf /tmp/abrepo && cp -r . /tmp/abrepo && (cd /tmp/abrepo/paper_2601_04422_b200/csrc && make -s clean && make -s AB=1 -j16 > /dev/null 2>&1)
(cd /tmp/abrepo && MPSIM_THETA=cpasync timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:theta --csv --log-file $GRAFT_REPO_ROOT/gpurun_out/r2_theta_cpasync.csv env NGATES=64 python tools/ncu_case.py > /dev/null 2>&1)
python tools/ncu_parse.py gpurun_out/r2_theta_tma.csv > gpurun_out/r2_theta_ab.txt 2>&1
python tools/ncu_parse.py gpurun_out/r2_theta_cpasync.csv >> gpurun_out/r2_theta_ab.txt 2>&1
