"""Throughput vs substep count (36-day windows): 40 windows x 4096 particles x 100 iterations."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402
from tools.bench_configs import stage2  # noqa: E402


def main():
    ctx = eng.Context(0)
    peak = eng.probe_fp64_rate(ctx)
    I, R, D = bench.load_series()
    N = bench.POPULATION
    args = [a for a in sys.argv[1:] if not a.startswith("--swarms=")]
    n_sw = int(next((a.split("=")[1] for a in sys.argv[1:] if a.startswith("--swarms=")), 40))
    for sub in [int(x) for x in args] or [6, 12, 24, 48, 96]:
        wins = []
        for w in range(n_sw):
            a = w * bench.DELTA
            sl = slice(a, a + 36)
            wins.append(eng.Window(ctx, I[sl], R[sl], D[sl], [N - I[a] - R[a] - D[a], I[a], R[a], D[a]], N,
                                   bench.SPEC, substeps=sub))
        swarms = [dict(window=wins[w], lower=[0] * 6, upper=stage2(35), n_particles=4096, max_iters=100,
                       seed=bench.mix_seed(5, w)) for w in range(n_sw)]
        plan = eng.Plan(ctx, swarms)
        plan.run_timed()
        s, k = plan.run_timed()
        ops = plan.evals * (35 * sub * 14 + 35 * 12) + bench.RAMP_OPS * plan.ramp_substeps
        print(f"substeps={sub:3d} evals/s={plan.evals / (s + k) * 1e3:.3e} frac={ops / ((s + k) * 1e-3) / peak:.3f}",
              flush=True)
        plan.close()


if __name__ == "__main__":
    main()
