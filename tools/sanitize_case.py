"""Small cases of every kernel family for compute-sanitizer (memcheck / racecheck)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402


def main():
    I, R, D = bench.load_series()
    N = bench.POPULATION
    ctx = eng.Context(0)

    def win(a, n, spec, sub=24):
        sl = slice(a, a + n)
        return eng.Window(ctx, I[sl], R[sl], D[sl], [N - I[a] - R[a] - D[a], I[a], R[a], D[a]], N, spec, substeps=sub)

    w1, w2, w3 = win(0, 36, "ird-mxse"), win(50, 21, "d-mape"), win(100, 100, "ird-mse")
    rng = np.random.default_rng(1)
    pos = rng.uniform(0, 1, (300, 6)) * np.array([2, 2, 28, 28, 1, 0.1])
    for w in (w1, w2, w3):
        w.eval_costs(pos)
    # flat kernels (two-level fold: 4,200 particles = 33 CTAs), cluster kernel, generic substeps
    ctx.fit_swarms([dict(window=w1, lower=[0] * 6, upper=[2, 2, 28, 28, 1, 0.1], n_particles=4200, max_iters=3,
                         seed=1),
                    dict(window=w3, lower=[0] * 6, upper=[2, 2, 90, 90, 1, 0.1], n_particles=700, max_iters=3, seed=2)]
                   + [dict(window=w2, lower=[0] * 6, upper=[2, 2, 13, 13, 1, 0.1], n_particles=1, max_iters=1, seed=j)
                      for j in range(300)])
    ctx.fit_swarms([dict(window=w2, lower=[0] * 6, upper=[2, 2, 13, 13, 1, 0.1], n_particles=300, max_iters=4,
                         seed=3)])
    b, c, _ = w1.forecast_ensemble_bands([0] * 6, [2, 2, 28, 28, 1, 0.1], seed=5, n=20000, horizon=7)
    w1.forecast_ensemble([0] * 6, [2, 2, 28, 28, 1, 0.1], seed=5, n=5000, horizon=7)
    ctx.integrate_batch(pos[:50], [N - 100, 100, 0, 0], N, 30)
    print("sanitize case ok", float(b[0, -1]), int(c[-1]))


if __name__ == "__main__":
    main()
