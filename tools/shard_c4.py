"""The C4 stability study sharded over the GPUs of one node (one process per
GPU under torchrun): (window, restart) units partitioned contiguously, each
rank runs its share as ONE engine plan, rank 0 gathers and merges in unit
order (sharding.run_sharded).  --check recomputes everything in one process
on rank 0 and requires bit-identical results.

    python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 tools/shard_c4.py
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402
from paper_2204_12346_b200 import sharding  # noqa: E402
from tools.bench_configs import stage2  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--windows", type=int, default=139)
    ap.add_argument("--restarts", type=int, default=1024)
    ap.add_argument("--particles", type=int, default=256)
    ap.add_argument("--iters", type=int, default=500)
    ap.add_argument("--backend", default=os.environ.get("SG_SHARD_BACKEND", "nccl"))
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    import torch.distributed as dist
    dev = local % max(torch.cuda.device_count(), 1)
    if world > 1:
        torch.cuda.set_device(dev)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(args.backend)
    I, R, D = bench.load_series()
    N = bench.POPULATION
    ctx = eng.Context(dev)
    wins = []
    for w in range(args.windows):
        a = w * bench.DELTA
        sl = slice(a, a + 36)
        wins.append(eng.Window(ctx, I[sl], R[sl], D[sl], [N - I[a] - R[a] - D[a], I[a], R[a], D[a]], N, bench.SPEC))
    units = sharding.units(args.windows, args.restarts)

    def compute(indices):
        swarms = [dict(window=wins[units[i][0]], lower=[0] * 6, upper=stage2(35), n_particles=args.particles,
                       max_iters=args.iters,
                       seed=bench.mix_seed(sharding.restart_seed(bench.BASE_SEED, units[i][1]), units[i][0]))
                  for i in indices]
        out = ctx.fit_swarms(swarms)
        return [(st, best.tobytes(), cost) for st, best, cost, _ in out]

    if world > 1:
        dist.barrier()
    t = time.perf_counter()
    merged = sharding.run_sharded(len(units), compute)
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - t
    if rank == 0:
        line = {"config": "C4-sharded", "ranks": world, "units": len(units), "wall_s": wall,
                "evals": len(units) * args.particles * args.iters,
                "evals_per_s": len(units) * args.particles * args.iters / wall,
                "failed": sum(r[0] != 0 for r in merged)}
        if args.check:
            single = compute(list(range(len(units))))
            line["identical_to_single_process"] = single == merged
        print(json.dumps(line), flush=True)
        if args.check and not line["identical_to_single_process"]:
            return 1
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
