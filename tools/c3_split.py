"""C3's work (2^20 particles x 100 iterations, one window) as 1, 2, 4, 8 swarms: what the single swarm's
per-iteration global barrier costs."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2204_12346_b200 as eng
from tools.bench_configs import stage2, window
import bench
ctx = eng.Context(0)
peak = eng.probe_fp64_rate(ctx)
win = window(ctx, 60, 35)
for k in (1, 2, 4, 8):
    plan = eng.Plan(ctx, [dict(window=win, lower=[0] * 6, upper=stage2(35), n_particles=(1 << 20) // k, max_iters=100,
                               seed=7 + j) for j in range(k)])
    plan.run_timed()
    s, t = plan.run_timed()
    ops = plan.evals * bench.ops_per_eval(36) + bench.RAMP_OPS * plan.ramp_substeps
    print(k, "swarms: ms", round(s + t, 2), "frac", round(ops / ((s + t) * 1e-3) / peak, 3), "launches", plan.step_launches)
