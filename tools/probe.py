"""Quick device probe: FP64 rate, eval kernel throughput, swarm sweep timing."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2204_12346_b200 as eng  # noqa: E402


def poland():
    a = np.genfromtxt(Path(__file__).resolve().parents[1] / "tests/golden/poland_like.csv", delimiter=",", names=True)
    return a["infectious"], a["recovered_cum"], a["deaths_cum"]


def window(ctx, I, R, D, w, tau=35, spec="ird-mxse"):
    a = 3 * w
    N = 38e6
    sl = slice(a, a + tau + 1)
    return eng.Window(ctx, I[sl], R[sl], D[sl], [N - I[a] - R[a] - D[a], I[a], R[a], D[a]], N, spec)


def main():
    ctx = eng.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    rate = eng.probe_fp64_rate(ctx)
    print(f"fp64 probe: {rate/1e12:.2f} T lane-ops/s")
    I, R, D = poland()
    # eval kernel
    for spec, variant in (("ird-mxse", "random"), ("ird-mxse", "noramp"), ("ird-mxse", "sorted_t1"),
                          ("ird-mxse", "sorted_2d"), ("d-mse", "random"), ("ird-mape", "random")):
        win = window(ctx, I, R, D, 60, spec=spec)
        n = 1 << 20
        g = torch.Generator(device="cuda").manual_seed(1)
        pos = torch.rand((n, 6), dtype=torch.float64, device="cuda", generator=g)
        pos *= torch.tensor([2, 2, 28, 28, 1, 0.1], dtype=torch.float64, device="cuda")
        t1 = torch.minimum(pos[:, 2], pos[:, 3])
        t2 = torch.maximum(pos[:, 2], pos[:, 3])
        pos[:, 2], pos[:, 3] = t1, t2
        if variant == "noramp":
            pos[:, 3] = pos[:, 2]
        elif variant == "sorted_t1":
            pos = pos[torch.argsort(pos[:, 2])].contiguous()
        elif variant == "sorted_2d":
            b1 = (pos[:, 2] / 28 * 32).long().clamp(0, 31)
            b2 = (pos[:, 3] / 28 * 32).long().clamp(0, 31)
            pos = pos[torch.argsort(b1 * 64 + b2 * 1.0 + pos[:, 3] / 28)].contiguous()
        costs = torch.empty(n, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        for _ in range(3):
            win.eval_costs_device(pos.data_ptr(), n, costs.data_ptr(), ctx.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(5):
                win.eval_costs_device(pos.data_ptr(), n, costs.data_ptr(), ctx.stream)
            e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 5
        evals = n / (ms * 1e-3)
        A = 35 * 24 * 14 + 36 * 12
        print(f"eval {spec} {variant}: {ms:.3f} ms per 1M particles -> {evals/1e9:.3f} G evals/s; "
              f"floor ops {A} -> {evals*A/1e12:.2f} T ops/s = {evals*A/rate:.3f} of probe")
    # sweep: 139 windows x 4096 x iters
    for iters in (20, 100):
        wins = [window(ctx, I, R, D, w) for w in range(139)]
        swarms = [dict(window=wins[w], lower=[0] * 6, upper=[2, 2, 28, 28, 1, 0.1], n_particles=4096,
                       max_iters=iters, seed=w) for w in range(139)]
        plan = eng.Plan(ctx, swarms)
        plan.run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            plan.run()
            e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"sweep 139x4096x{iters}: {ms:.1f} ms -> {plan.evals/(ms*1e-3)/1e9:.3f} G evals/s")
        res = plan.results()
        print("  best costs w0..3:", [r[2] for r in res[:4]])
        plan.close()
    # C1
    win = window(ctx, I, R, D, 0, tau=20)
    plan = eng.Plan(ctx, [dict(window=win, lower=[0] * 6, upper=[2, 2, 13, 13, 1, 0.1], n_particles=256,
                               max_iters=500, seed=1)])
    plan.run()
    torch.cuda.synchronize()
    t = time.perf_counter()
    plan.run()
    plan.results()
    print(f"C1 256x500: {1e3*(time.perf_counter()-t):.2f} ms wall")


if __name__ == "__main__":
    main()
