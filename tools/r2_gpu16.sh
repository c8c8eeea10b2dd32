# N=4 box: multi-GPU parity (Python harness + C++ facade program), bench weak and strong at N=2 and N=4
mkdir -p gpurun_out
export MASTER_ADDR=127.0.0.1
MGPU_TMP=/tmp/mgpu4 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 tools/mgpu_check.py > gpurun_out/r2_mgpu4.log 2>&1
echo "mgpu rc=$?" >> gpurun_out/r2_mgpu4.log
g++ -std=c++17 -O1 -I include -I /usr/local/cuda/include tests/cpp/shard_main.cpp -o /tmp/shard_main -L paper_2601_04422_b200 -lmpsim_gpu -Wl,-rpath,$PWD/paper_2601_04422_b200
rm -f /tmp/ncclid4; for r in 1 2 3; do (timeout 300 /tmp/shard_main $r 4 /tmp/ncclid4 $r > gpurun_out/r2_shard4_r$r.log 2>&1 &); done; timeout 300 /tmp/shard_main 0 4 /tmp/ncclid4 0 > gpurun_out/r2_shard4_r0.log 2>&1; echo "rc=$?" >> gpurun_out/r2_shard4_r0.log
sleep 3
for N in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2972$N bench.py --gpus $N --steps 4 --warmup 3 --no-pipeline > gpurun_out/r2_bench_n${N}w.json 2> gpurun_out/r2_bench_n${N}w.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2973$N bench.py --gpus $N --steps 4 --warmup 3 --no-pipeline --scaling strong > gpurun_out/r2_bench_n${N}s.json 2> gpurun_out/r2_bench_n${N}s.err
done
timeout 600 python bench.py --steps 4 --warmup 3 --no-pipeline --no-cpu-baseline > gpurun_out/r2_bench_n1_on4.json 2> gpurun_out/r2_bench_n1_on4.err
