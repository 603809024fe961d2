"""C2 launch timeline (the bench plan, --iters iterations): every lane's step-kernel launches
from CUPTI (torch.profiler) — start/end per stream — to see whether the lanes overlap each
other's fill and drain or run in phase."""
import collections
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    I, R, D = bench.load_series()
    ctx = eng.Context(0)
    wins = []
    for w in range(bench.n_windows(len(I))):
        a = w * bench.DELTA
        sl = slice(a, a + bench.TAU + 1)
        wins.append(eng.Window(ctx, I[sl], R[sl], D[sl], [bench.POPULATION - I[a] - R[a] - D[a], I[a], R[a], D[a]],
                               bench.POPULATION, bench.SPEC))
    swarms = [dict(window=w, lower=[0.0] * 6, upper=bench.STAGE2_HI, n_particles=bench.PARTICLES, max_iters=iters,
                   seed=bench.mix_seed(bench.BASE_SEED, k)) for k, w in enumerate(wins)]
    plan = eng.Plan(ctx, swarms)
    plan.run_timed()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        s, k = plan.run_timed()
        torch.cuda.synchronize()
    ev = sorted(((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0) or e.thread)
                 for e in prof.events() if e.device_type.name == "CUDA" and "pso_step_kernel" in e.name))
    by = collections.defaultdict(list)
    for a, b, st in ev:
        by[st].append((a, b))
    lanes = sorted(by)
    t0 = ev[0][0]
    # per iteration index: spread of the lanes' start times and end times
    n_it = min(len(v) for v in by.values())
    spreads_start = []
    spreads_end = []
    for i in range(n_it):
        st = [by[l][i][0] for l in lanes]
        en = [by[l][i][1] for l in lanes]
        spreads_start.append(max(st) - min(st))
        spreads_end.append(max(en) - min(en))
    # time with no step kernel running, and with only one lane running
    edges = sorted([(a, 1) for a, b, _ in ev] + [(b, -1) for a, b, _ in ev])
    active = 0
    last = edges[0][0]
    hist = collections.Counter()
    for t, d in edges:
        hist[active] += t - last
        active += d
        last = t
    total = edges[-1][0] - edges[0][0]
    print(json.dumps({"iters": iters, "steps_ms": k, "lanes": len(lanes), "launches": len(ev),
                      "per_iter_us": k * 1e3 / iters,
                      "launch_us_mean": sum(b - a for a, b, _ in ev) / len(ev),
                      "lane_start_spread_us_mean": sum(spreads_start) / n_it,
                      "lane_end_spread_us_mean": sum(spreads_end) / n_it,
                      "time_share_by_active_launches": {str(a): round(v / total, 4) for a, v in sorted(hist.items())}},
                     indent=1))


if __name__ == "__main__":
    main()
