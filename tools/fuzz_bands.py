"""Extended version of test_ensemble_bands_batch_random_against_host_sort: many random
pipelined band batches against sorting each window's forecast deaths on the host."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

import paper_2204_12346_b200 as eng  # noqa: E402
from conftest import GOLDEN  # noqa: E402
from test_gpu_parity import _host_bands, _random_band_batch  # noqa: E402


def main():
    n_batches = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    base = int(sys.argv[2]) if len(sys.argv) > 2 else 800000
    a = np.genfromtxt(GOLDEN / "poland_like.csv", delimiter=",", names=True)
    poland = {"I": a["infectious"], "R": a["recovered_cum"], "D": a["deaths_cum"], "N": 38_000_000.0}
    ctx = eng.Context(0)
    bad = windows = 0
    for b in range(n_batches):
        rng = np.random.default_rng(base + b)
        wins, lo, hi, seeds, n, horizon = _random_band_batch(eng, ctx, poland, rng)
        bands, counts = ctx.forecast_ensemble_bands_batch(wins, lo, hi, seeds, n, horizon)
        for k, w in enumerate(wins):
            _, _, deaths = w.forecast_ensemble(lo, hi, seed=seeds[k], n=n, horizon=horizon, want_costs=False,
                                               want_params=False)
            want, want_counts = _host_bands(deaths)
            windows += 1
            ok = counts[k].tolist() == want_counts and np.array_equal(bands[k].view(np.uint64),
                                                                       want.view(np.uint64))
            if not ok:
                bad += 1
                print("MISMATCH batch", b, "window", k, flush=True)
    fused, passes, _ = ctx.band_stats
    print(f"fuzz_bands: {n_batches} batches, {windows} windows, {bad} mismatches "
          f"(days from the fused histogram {fused}, through the histogram pass {passes})", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
