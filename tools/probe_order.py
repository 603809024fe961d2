"""Eval-kernel throughput vs particle order within swarms of 4096 (ramp coherence experiment)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402


def morton(q1, q2, bits):
    key = torch.zeros_like(q1)
    for b in range(bits):
        key |= ((q1 >> b) & 1) << (2 * b + 1)
        key |= ((q2 >> b) & 1) << (2 * b)
    return key


def main():
    ctx = eng.Context(0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    I, R, D = bench.load_series()
    a = 180
    sl = slice(a, a + 36)
    win = eng.Window(ctx, I[sl], R[sl], D[sl], [bench.POPULATION - I[a] - R[a] - D[a], I[a], R[a], D[a]],
                     bench.POPULATION, "ird-mxse")
    n = 139 * 4096
    g = torch.Generator(device="cuda").manual_seed(3)
    pos = torch.rand((n, 6), dtype=torch.float64, device="cuda", generator=g)
    pos *= torch.tensor(bench.STAGE2_HI, dtype=torch.float64, device="cuda")
    t1 = torch.minimum(pos[:, 2], pos[:, 3])
    t2 = torch.maximum(pos[:, 2], pos[:, 3])
    pos[:, 2], pos[:, 3] = t1, t2
    grp = torch.arange(n, device="cuda") // 4096

    def order(key):
        return pos[torch.argsort(grp * (1 << 40) + key)].contiguous()

    variants = {"random": pos}
    for bits in (3, 4, 5, 6):
        q1 = (t1 / 28 * (1 << bits)).long().clamp(0, (1 << bits) - 1)
        q2 = (t2 / 28 * (1 << bits)).long().clamp(0, (1 << bits) - 1)
        variants[f"morton{bits}"] = order(morton(q1, q2, bits))
    variants["t1_only"] = order((t1 * 1e6).long())
    variants["t2_only"] = order((t2 * 1e6).long())
    q1 = (t1 / 28 * 8).long().clamp(0, 7)
    variants["rows8_t2"] = order(q1 * (1 << 30) + (t2 * 1e6).long())
    costs = torch.empty(n, dtype=torch.float64, device="cuda")
    ref = None
    for name, p in variants.items():
        for _ in range(2):
            win.eval_costs_device(p.data_ptr(), n, costs.data_ptr(), ctx.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(5):
                win.eval_costs_device(p.data_ptr(), n, costs.data_ptr(), ctx.stream)
            e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 5
        s = float(costs.sum().item()) if name == "random" else None
        print(f"{name:10s} {ms:.3f} ms  {n / ms / 1e6:.3f} G evals/s", flush=True)


if __name__ == "__main__":
    main()
