"""Per-rank time split of a sharded brick layer (exchange in / execute / exchange out).

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/mgpu_probe.py
"""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench as B  # noqa: E402
from paper_2601_04422_b200 import sharded  # noqa: E402
from paper_2601_04422_b200.mps import execute  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl")
n, chi = int(os.environ.get("NQ", "256")), 512
rng = np.random.default_rng(1234)
bonds = B.chain_bonds(n, chi)
ch = sharded.ShardedChain(n, chi, rank, world, device=local, dist=dist)
for i in range(ch.lo, ch.hi):
    ch.set_site(i, B.random_site(np.random.default_rng(10_000 + i), bonds[i], bonds[i + 1]))
ch.finalize_setup()
steps = [B.layer_gates(n, s % 2, rng) for s in range(7)]
acc = np.zeros(3)
for s, layer in enumerate(steps):
    local_g, sl, sr = sharded.partition_layer(layer, ch.lo, ch.hi, rank, world)
    torch.cuda.synchronize(); dist.barrier()
    t0 = time.perf_counter()
    ch._exchange_in(sl, sr); torch.cuda.synchronize(); t1 = time.perf_counter()
    st = execute(ch.state, local_g, chi, 1e-12); torch.cuda.synchronize(); t2 = time.perf_counter()
    ch._exchange_out(sl, sr); torch.cuda.synchronize(); t3 = time.perf_counter()
    c = ch.state.counters()
    if s >= 3:
        acc += [t1 - t0, t2 - t1, t3 - t2]
    print(f"rank {rank} step {s}: gates {len(local_g)} in {1e3*(t1-t0):.1f} exec {1e3*(t2-t1):.1f} out {1e3*(t3-t2):.1f} ms "
          f"sweeps {c['sweeps']}", flush=True)
    ch.state.reset_counters()
print(f"rank {rank} avg in/exec/out ms: {np.round(1e3 * acc / 4, 1)}", flush=True)
dist.destroy_process_group()
