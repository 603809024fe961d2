"""Small C2-shaped run for ncu: 139 windows x 4096 particles x --iters iterations."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=8)
    ap.add_argument("--spec", default=bench.SPEC)
    ap.add_argument("--reps", type=int, default=1, help="timed runs (the first includes lazy module loading)")
    ap.add_argument("--substeps", type=int, default=24)
    args = ap.parse_args()
    I, R, D = bench.load_series()
    ctx = eng.Context(0)
    wins = []
    for w in range(bench.n_windows(len(I))):
        a = w * bench.DELTA
        sl = slice(a, a + bench.TAU + 1)
        wins.append(eng.Window(ctx, I[sl], R[sl], D[sl], [bench.POPULATION - I[a] - R[a] - D[a], I[a], R[a], D[a]],
                               bench.POPULATION, args.spec, substeps=args.substeps))
    swarms = [dict(window=w, lower=[0.0] * 6, upper=bench.STAGE2_HI, n_particles=bench.PARTICLES,
                   max_iters=args.iters, seed=bench.mix_seed(bench.BASE_SEED, k)) for k, w in enumerate(wins)]
    plan = eng.Plan(ctx, swarms)
    for _ in range(args.reps):
        seed_ms, steps_ms = plan.run_timed()
        res = plan.results()
        print(f"seed {seed_ms:.3f} ms, steps {steps_ms:.3f} ms ({steps_ms / args.iters:.3f} ms/launch), "
              f"best w0 {res[0][2]!r}, launches {ctx.launch_count}")


if __name__ == "__main__":
    main()
