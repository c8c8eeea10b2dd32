# N=2 box: multi-GPU parity of the C++ shard layer (Python harness and the C++
# facade program), bench at N=2 (weak) and N=2 strong.
mkdir -p gpurun_out
export MASTER_ADDR=127.0.0.1
MGPU_TMP=/tmp/mgpu timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/mgpu_check.py > gpurun_out/r2_mgpu2b.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/r2_mgpu2b.log
g++ -std=c++17 -O1 -I include -I /usr/local/cuda/include tests/cpp/shard_main.cpp -o /tmp/shard_main -L paper_2601_04422_b200 -lmpsim_gpu -Wl,-rpath,$PWD/paper_2601_04422_b200
rm -f /tmp/ncclid; (timeout 300 /tmp/shard_main 1 2 /tmp/ncclid 1 > gpurun_out/r2_shard_main_r1.log 2>&1 &) ; timeout 300 /tmp/shard_main 0 2 /tmp/ncclid 0 > gpurun_out/r2_shard_main_r0.log 2>&1; echo "rc=$?" >> gpurun_out/r2_shard_main_r0.log
sleep 2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 2 --steps 4 --warmup 3 --no-pipeline > gpurun_out/r2_bench_n2b.json 2> gpurun_out/r2_bench_n2b.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 --steps 4 --warmup 3 --no-pipeline --scaling strong > gpurun_out/r2_bench_n2s.json 2> gpurun_out/r2_bench_n2s.err
