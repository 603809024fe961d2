"""C1 alone (window 0, tau=20, 256 particles x 500 iterations): one persistent-swarm launch, for ncu."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402


def main():
    I, R, D = bench.load_series()
    N = bench.POPULATION
    ctx = eng.Context(0)
    win = eng.Window(ctx, I[:21], R[:21], D[:21], [N - I[0] - R[0] - D[0], I[0], R[0], D[0]], N, bench.SPEC)
    plan = eng.Plan(ctx, [dict(window=win, lower=[0] * 6, upper=[2.0, 2.0, 13.0, 13.0, 1.0, 0.1], n_particles=256,
                               max_iters=500, seed=bench.mix_seed(bench.BASE_SEED, 0))])
    for _ in range(3):
        s, k = plan.run_timed()
        print(f"C1 seed {s:.3f} ms steps {k:.3f} ms best {plan.results()[0][2]}", flush=True)


if __name__ == "__main__":
    main()
