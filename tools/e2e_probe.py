"""Alternate the device-timed C2 plan and the e2e sg_fit_all_windows_series call; print both with SM clocks."""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402
from paper_2204_12346_b200 import _capi  # noqa: E402


def main():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    I, R, D = bench.load_series()
    n_win = bench.n_windows(len(I))
    ctx = eng.Context(0)
    wins = []
    for w in range(n_win):
        a = w * bench.DELTA
        sl = slice(a, a + bench.TAU + 1)
        wins.append(eng.Window(ctx, I[sl], R[sl], D[sl], [bench.POPULATION - I[a] - R[a] - D[a], I[a], R[a], D[a]],
                               bench.POPULATION, bench.SPEC))
    swarms = [dict(window=w, lower=[0.0] * 6, upper=bench.STAGE2_HI, n_particles=bench.PARTICLES, max_iters=1000,
                   seed=bench.mix_seed(bench.BASE_SEED, k)) for k, w in enumerate(wins)]
    plan = eng.Plan(ctx, swarms)
    settings = _capi.sg_fit_settings(1, 0, 0.0, 2.0, 0.0, 1.0, 0.0, 0.1, 7, bench.PARTICLES, 1000, 0.5, 0.5, 0.5,
                                     bench.POPULATION, 24)
    recs = (_capi.sg_fit_record * n_win)()
    trajs = np.empty((n_win, bench.TAU + 1, 4))
    nw, failed, mean = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_double()
    I, R, D = (np.ascontiguousarray(a) for a in (I, R, D))

    def e2e():
        rc = _capi.lib().sg_fit_all_windows_series(ctx.handle, _capi._d(I), _capi._d(R), _capi._d(D), len(I),
                                                   bench.TAU, bench.DELTA, ctypes.byref(settings), bench.BASE_SEED,
                                                   n_win, ctypes.byref(nw), recs, _capi._d(trajs), ctypes.byref(mean),
                                                   ctypes.byref(failed))
        ctx.check(rc)

    e2e()
    ts = []
    for k in range(10):
        t = time.perf_counter()
        e2e()
        ts.append((time.perf_counter() - t) * 1e3)
    print("back-to-back e2e ms:", " ".join(f"{x:.1f}" for x in ts), flush=True)
    for k in range(3):
        s, kms = plan.run_timed()
        c1 = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        t = time.perf_counter()
        e2e()
        e = (time.perf_counter() - t) * 1e3
        c2 = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        print(f"rep {k}: plan seed {s:.2f} ms steps {kms:.2f} ms | e2e {e:.2f} ms | sm clk {c1} {c2}", flush=True)


if __name__ == "__main__":
    main()
