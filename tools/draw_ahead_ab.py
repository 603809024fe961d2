"""A/B of the draw-ahead experiment (SG_DRAW_AHEAD / SG_DRAW_PRIO): C2 plan
(139 windows, --iters), C3 (one 2^20 swarm, 30 iterations) and a 21-day
sweep; device ms per run and a history hash (must not change)."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CODE = r"""
import sys, json, hashlib
sys.path.insert(0, %r)
import numpy as np, bench, paper_2204_12346_b200 as eng
I, R, D = bench.load_series(); ctx = eng.Context(0); N = bench.POPULATION
def run(swarms, reps=3):
    plan = eng.Plan(ctx, swarms)
    for _ in range(3): plan.run()
    ms = min(sum(plan.run_timed()) for _ in range(reps))
    h = hashlib.sha1(b"".join(np.asarray(r[3]).tobytes() for r in plan.results())).hexdigest()[:12]
    plan.close(); return ms, h
def win(w, tau):
    a = w * bench.DELTA; sl = slice(a, a + tau + 1)
    return eng.Window(ctx, I[sl], R[sl], D[sl], [N - I[a] - R[a] - D[a], I[a], R[a], D[a]], N, bench.SPEC)
hi = lambda tau: [2.0, 2.0, float(tau - 7), float(tau - 7), 1.0, 0.1]
out = {}
ws = [win(w, 35) for w in range(139)]
out["c2"] = run([dict(window=ws[w], lower=[0]*6, upper=hi(35), n_particles=4096, max_iters=%d, seed=bench.mix_seed(2204, w)) for w in range(139)])
out["c3"] = run([dict(window=ws[60], lower=[0]*6, upper=hi(35), n_particles=1 << 20, max_iters=30, seed=7)], reps=2)
ws21 = [win(w, 20) for w in range(143)]
out["w21"] = run([dict(window=ws21[w], lower=[0]*6, upper=hi(20), n_particles=4096, max_iters=200, seed=w) for w in range(143)])
print(json.dumps(out))
"""


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    for da, prio in [("0", "low"), ("1", "low"), ("1", "equal")]:
        env = dict(os.environ, SG_DRAW_AHEAD=da, SG_DRAW_PRIO=prio)
        r = subprocess.run([sys.executable, "-c", CODE % (str(ROOT), iters)], capture_output=True, text=True, env=env)
        d = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {"error": r.stderr[-400:]}
        print(json.dumps({"draw_ahead": da, "prio": prio, **d}), flush=True)


if __name__ == "__main__":
    main()
