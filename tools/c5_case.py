"""C5 for a few windows (10^6 sampled sets, 21-day forecast, device bands), for the ncu launch list."""
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
    if "--batch" in sys.argv:  # the pipelined many-window call (fused selection passes, samples drawn ahead)
        n_win = int(sys.argv[1]) if sys.argv[1] != "--batch" else 6
        wins = []
        for w in range(n_win):
            a = w * bench.DELTA
            sl = slice(a, a + 36)
            wins.append(eng.Window(ctx, I[sl], R[sl], D[sl], [N - I[a] - R[a] - D[a], I[a], R[a], D[a]], N,
                                   bench.SPEC))
        bands, counts = ctx.forecast_ensemble_bands_batch(wins, [0] * 6, [2.0, 2.0, 28.0, 28.0, 1.0, 0.1],
                                                          [bench.mix_seed(2204, w) for w in range(n_win)],
                                                          1_000_000, 21)
        print(float(bands[-1][0, -1]), int(counts[-1][-1]), flush=True)
        return
    for w in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
        a = w * bench.DELTA
        sl = slice(a, a + 36)
        win = eng.Window(ctx, I[sl], R[sl], D[sl], [N - I[a] - R[a] - D[a], I[a], R[a], D[a]], N, bench.SPEC)
        bands, counts, _ = win.forecast_ensemble_bands([0] * 6, [2.0, 2.0, 28.0, 28.0, 1.0, 0.1],
                                                       seed=bench.mix_seed(2204, w), n=1_000_000, horizon=21)
        print(w, float(bands[0, -1]), int(counts[-1]), flush=True)


if __name__ == "__main__":
    main()
