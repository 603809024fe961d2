"""Diagnostic: warp-day class histogram of the C2 sweep (needs a -DSG_DAY_COUNTERS=1 build in $SG_LIB)."""
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402
from paper_2204_12346_b200 import _capi  # noqa: E402


def main(iters):
    I, R, D = bench.load_series()
    ctx = eng.Context(0)
    wins = []
    for w in range(bench.n_windows(len(I))):
        a = w * bench.DELTA
        sl = slice(a, a + bench.TAU + 1)
        wins.append(eng.Window(ctx, I[sl], R[sl], D[sl], [bench.POPULATION - I[a] - R[a] - D[a], I[a], R[a], D[a]],
                               bench.POPULATION, bench.SPEC))
    out = (ctypes.c_ulonglong * 3)()
    _capi.lib().sg_debug_day_classes(out)
    for it in (1, 10, 100, iters):
        swarms = [dict(window=w, lower=[0.0] * 6, upper=bench.STAGE2_HI, n_particles=bench.PARTICLES, max_iters=it,
                       seed=bench.mix_seed(bench.BASE_SEED, k)) for k, w in enumerate(wins)]
        plan = eng.Plan(ctx, swarms)
        plan.run()
        ramp = plan.ramp_substeps
        _capi.lib().sg_debug_day_classes(out)
        tot = sum(out)
        warp_days = tot
        print(f"iters={it}: warp-days const {out[0]/tot:.3f} switch {out[1]/tot:.3f} ramp {out[2]/tot:.3f}; "
              f"ramp substeps/eval {ramp/plan.evals:.1f} -> lane-level ramp fraction {ramp/plan.evals/840:.3f}, "
              f"warp-level ramp-day substep fraction {out[2]/tot:.3f}")
        plan.close()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1000)
