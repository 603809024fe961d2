"""Time the C2 sweep (139 x 4096 x --iters) for the library in $SG_LIB; prints one JSON line."""
import argparse
import hashlib
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    I, R, D = bench.load_series()
    ctx = eng.Context(0)
    wins = []
    for w in range(bench.n_windows(len(I))):
        a = w * bench.DELTA
        sl = slice(a, a + bench.TAU + 1)
        wins.append(eng.Window(ctx, I[sl], R[sl], D[sl], [bench.POPULATION - I[a] - R[a] - D[a], I[a], R[a], D[a]],
                               bench.POPULATION, bench.SPEC))
    swarms = [dict(window=w, lower=[0.0] * 6, upper=bench.STAGE2_HI, n_particles=bench.PARTICLES,
                   max_iters=args.iters, seed=bench.mix_seed(bench.BASE_SEED, k)) for k, w in enumerate(wins)]
    plan = eng.Plan(ctx, swarms)
    plan.run_timed()
    best = None
    for _ in range(args.reps):
        s, k = plan.run_timed()
        best = k if best is None else min(best, k)
    res = plan.results()
    h = hashlib.sha1(b"".join(r[3].tobytes() for r in res)).hexdigest()[:12]
    evals = plan.evals
    print(json.dumps({"lib": os.path.basename(os.environ.get("SG_LIB", "default")), "iters": args.iters,
                      "steps_ms": round(best, 3), "ms_per_iter": round(best / args.iters, 4),
                      "gevals_s": round(evals / (best * 1e-3) / 1e9, 4), "hist_sha": h}), flush=True)


if __name__ == "__main__":
    main()
