"""Launch-lane sweep (SG_PLAN_LANES) for rank 0's share of the C2 sweep at
N = 1 and 8 GPUs: device ms per run of the plan."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CODE = r"""
import sys, json
sys.path.insert(0, %r)
import bench, paper_2204_12346_b200 as eng
from paper_2204_12346_b200.sharding import partition
I, R, D = bench.load_series(); n_win = bench.n_windows(len(I)); ctx = eng.Context(0)
share = list(partition(n_win, %d, 0)); wins = []
for w in share:
    Iw, Rw, Dw, init = bench._window_inputs(I, R, D, w)
    wins.append(eng.Window(ctx, Iw, Rw, Dw, init, bench.POPULATION, bench.SPEC))
plan = eng.Plan(ctx, [dict(window=wins[k], lower=[0.0] * 6, upper=bench.STAGE2_HI, n_particles=bench.PARTICLES,
                           max_iters=%d, seed=bench.mix_seed(bench.BASE_SEED, w)) for k, w in enumerate(share)])
for _ in range(3): plan.run()
ms = min(sum(plan.run_timed()) for _ in range(3))
h = plan.results()
print(json.dumps({"ms": ms, "evals_per_s": plan.evals / ms * 1e3, "hist_hash": hash(tuple(float(x[3][-1]) for x in h))}))
"""


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    for n, lanes in [(8, 1), (8, 2), (8, 4), (8, 8), (8, 12), (8, 18), (1, 4), (1, 8), (1, 16), (2, 4), (2, 8), (4, 4), (4, 8)]:
        env = dict(os.environ, SG_PLAN_LANES=str(lanes))
        out = subprocess.run([sys.executable, "-c", CODE % (str(ROOT), n, iters)], capture_output=True, text=True,
                             env=env)
        d = json.loads(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else {"error": out.stderr[-300:]}
        d.update({"gpus": n, "lanes": lanes})
        print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()
