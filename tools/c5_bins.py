"""C5 diagnostics: for one window of 10^6 samples, the band selection's
per-day key range shift and the sizes of the bins holding the wanted ranks
(what sel_finish_kernel has to rank), emulated on the host from the
ensemble's deaths (sg_forecast_ensemble)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402


def keys_of(x):
    b = x.view(np.uint64)
    return np.where(b >> np.uint64(63), ~b, b | np.uint64(1 << 63))


def main():
    I, R, D = bench.load_series()
    N = bench.POPULATION
    ctx = eng.Context(0)
    w = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    a = w * bench.DELTA
    sl = slice(a, a + 36)
    win = eng.Window(ctx, I[sl], R[sl], D[sl], [N - I[a] - R[a] - D[a], I[a], R[a], D[a]], N, bench.SPEC)
    _, _, deaths = win.forecast_ensemble([0] * 6, [2.0, 2.0, 28.0, 28.0, 1.0, 0.1], seed=bench.mix_seed(2204, w),
                                         n=1_000_000, horizon=21, want_costs=False, want_params=False)
    for d in range(deaths.shape[1]):
        col = deaths[:, d]
        col = col[np.isfinite(col)]
        k = col.size
        ks = keys_of(col.copy())
        kmin, kmax = int(ks.min()), int(ks.max())
        rng = kmax - kmin
        shift = max(0, rng.bit_length() - 12)
        bins = ((ks - np.uint64(kmin)) >> np.uint64(shift)).astype(np.int64)
        hist = np.bincount(bins, minlength=4096)
        cum = np.cumsum(hist)
        wanted = set()
        for p in (0.5, 0.25, 0.75, 0.05, 0.95, 0.025, 0.975):
            h = float(k - 1) * p
            lo = int(h)
            for r in ([k - 1] if lo + 1 >= k else [lo, lo + 1]):
                wanted.add(int(np.searchsorted(cum, r, side="right")))
        print(d, k, shift, sorted((b, int(hist[b])) for b in wanted), "max bin", int(hist.max()), flush=True)


if __name__ == "__main__":
    main()
