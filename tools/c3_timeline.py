"""C3 device timeline (one 2^20-particle swarm): per-iteration step-kernel durations and the
gaps between consecutive launches, from CUPTI (torch.profiler), so the single swarm's
per-iteration barrier cost splits into launch gaps vs in-kernel fill/drain."""
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2204_12346_b200 as eng  # noqa: E402
from tools.bench_configs import stage2, window  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    ctx = eng.Context(0)
    win = window(ctx, 60, 35)
    plan = eng.Plan(ctx, [dict(window=win, lower=[0] * 6, upper=stage2(35), n_particles=1 << 20, max_iters=iters,
                               seed=7)])
    plan.run_timed()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        s, k = plan.run_timed()
        torch.cuda.synchronize()
    ev = sorted(((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                 if e.device_type.name == "CUDA" and "pso_step_kernel" in e.name), key=lambda x: x[0])
    durs = [b - a for a, b, _ in ev]
    gaps = [ev[i + 1][0] - ev[i][1] for i in range(len(ev) - 1)]
    print(json.dumps({"iters": iters, "steps_ms": k, "launches": len(ev), "kernel_us_mean": sum(durs) / len(durs),
                      "gap_us_mean": sum(gaps) / max(1, len(gaps)), "gap_us_max": max(gaps) if gaps else 0.0,
                      "per_iter_us": k * 1e3 / iters}, indent=1))


if __name__ == "__main__":
    main()
