"""Throughput vs window length (tau): 40 swarms (--swarms=N) x 4096 particles x 100 iterations, ird-mxse,
stage2 box (the series' windows of that length, repeated with other seeds when there are fewer)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402
from tools.bench_configs import stage2, window  # noqa: E402


def main():
    ctx = eng.Context(0)
    peak = eng.probe_fp64_rate(ctx)
    args = [a for a in sys.argv[1:] if not a.startswith("--swarms=")]
    n_sw = int(next((a.split("=")[1] for a in sys.argv[1:] if a.startswith("--swarms=")), 40))
    for tau in [int(x) for x in args] or [20, 35, 60, 85, 86, 100, 150, 200]:
        n_win = max(1, min(n_sw, 1 + (450 - tau - 1) // bench.DELTA))
        wins = [window(ctx, w, tau) for w in range(n_win)]
        swarms = [dict(window=wins[k % n_win], lower=[0] * 6, upper=stage2(tau), n_particles=4096, max_iters=100,
                       seed=bench.mix_seed(5, k)) for k in range(n_sw)]
        plan = eng.Plan(ctx, swarms)
        plan.run_timed()
        s, k = plan.run_timed()
        ops = plan.evals * bench.ops_per_eval(tau + 1) + bench.RAMP_OPS * plan.ramp_substeps
        print(f"tau={tau:4d} days={tau + 1:4d} evals/s={plan.evals / (s + k) * 1e3:.3e} frac={ops / ((s + k) * 1e-3) / peak:.3f}",
              flush=True)
        plan.close()


if __name__ == "__main__":
    main()
