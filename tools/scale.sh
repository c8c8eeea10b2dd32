#!/bin/bash
# Strong-scaling sweep of bench.py on one node: N = 1, 2, 4, 8 (as many as visible).
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for n in 1 2 4 8; do
  [ $n -gt $NG ] && break
  if [ $n -eq 1 ]; then
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/scale_$n.json
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n)) \
      bench.py --gpus $n --steps 4 --warmup 3 2>/dev/null | tail -1 > gpurun_out/scale_$n.json
  fi
  python -c "import json; d=json.load(open('gpurun_out/scale_$n.json')); print($n, round(d['value'],1), round(d['ms_per_step'],1), d['clocks'])"
done
