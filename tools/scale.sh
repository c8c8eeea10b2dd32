#!/bin/bash
# Scaling sweep of bench.py on one node: N = 1, 2, 4, 8 (as many as visible).
# SCALING=weak (default: 256 qubits per GPU) or SCALING=strong (one 256-qubit chain).
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
SC=${SCALING:-weak}
for n in 1 2 4 8; do
  [ $n -gt $NG ] && break
  if [ $n -eq 1 ]; then
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-pipeline --scaling $SC 2>/dev/null | tail -1 > gpurun_out/scale_${SC}_$n.json
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n)) \
      bench.py --gpus $n --steps 4 --warmup 3 --scaling $SC 2>/dev/null | tail -1 > gpurun_out/scale_${SC}_$n.json
  fi
  python -c "import json; d=json.load(open('gpurun_out/scale_${SC}_$n.json')); print('$SC', $n, round(d['value'],1), round(d['ms_per_step'],1), d['config']['n_qubits'], d['clocks'])"
done
