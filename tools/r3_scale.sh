#!/bin/bash
# Final-build scaling on one 4-GPU box: N=1 bench, then N=2 / N=4 weak and strong via torchrun, and the N=4 sharded checks.
mkdir -p gpurun_out
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/sc_n1.json 2> gpurun_out/sc_n1.err; echo "n1 rc=$?"
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N bench.py --gpus $N --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline > gpurun_out/sc_n${N}.json 2> gpurun_out/sc_n${N}.err; echo "n$N weak rc=$?"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline --scaling strong > gpurun_out/sc_n${N}_strong.json 2> gpurun_out/sc_n${N}_strong.err; echo "n$N strong rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tools/mgpu_check.py > gpurun_out/sc_mgpu_check_n4.txt 2>&1; echo "mgpu_check rc=$?"
for f in gpurun_out/sc_n*.json; do echo "$f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],2), d['n_gpus'], d['scaling'], d['clocks']['sm_mhz'], d['clocks']['reasons'])")"; done
tail -8 gpurun_out/sc_mgpu_check_n4.txt
