#!/bin/bash
# N-GPU bench through torchrun (weak, then strong) and the sharded parity check.
N=${N:-2}
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/r3_bench_n${N}.json 2> gpurun_out/r3_bench_n${N}.err
echo "weak rc=$?"; tail -1 gpurun_out/r3_bench_n${N}.json | cut -c1-200
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline --scaling strong > gpurun_out/r3_bench_n${N}_strong.json 2> gpurun_out/r3_bench_n${N}_strong.err
echo "strong rc=$?"; tail -1 gpurun_out/r3_bench_n${N}_strong.json | cut -c1-200
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29515 tools/mgpu_check.py > gpurun_out/r3_mgpu_check_n${N}.txt 2>&1
echo "mgpu_check rc=$?"; tail -12 gpurun_out/r3_mgpu_check_n${N}.txt
