"""CTA start/end times of one step-kernel iteration of C3 (one 2^20-particle swarm) or C2 (argument c2:
the bench plan, every lane), from a
diagnostic build (-DSG_CTA_TIMES=<iteration>): the occupancy profile over the launch —
how long the grid fills, runs full, and drains.

    python -c "from paper_2204_12346_b200 import build; build.build(out='tools/libsirdgpu_ctatimes.so', extra=['-DSG_CTA_TIMES=5'])"
    SG_LIB=$PWD/tools/libsirdgpu_ctatimes.so python tools/cta_times.py
"""
import ctypes
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2204_12346_b200 as eng  # noqa: E402
from paper_2204_12346_b200 import _capi  # noqa: E402
from tools.bench_configs import stage2, window  # noqa: E402


def main():
    ctx = eng.Context(0)
    if len(sys.argv) > 1 and sys.argv[1] == "c2":  # the bench plan: 139 windows x 4096, all lanes
        import bench
        wins = [window(ctx, w, 35) for w in range(139)]
        swarms = [dict(window=w, lower=[0.0] * 6, upper=bench.STAGE2_HI, n_particles=4096, max_iters=12,
                       seed=bench.mix_seed(bench.BASE_SEED, k)) for k, w in enumerate(wins)]
        n = 139 * 32
    else:  # C3: one swarm of 2^20 particles
        win = window(ctx, 60, 35)
        swarms = [dict(window=win, lower=[0] * 6, upper=stage2(35), n_particles=1 << 20, max_iters=12, seed=7)]
        n = 8192
    plan = eng.Plan(ctx, swarms)
    plan.run_timed()
    buf = np.zeros((6 * 8192, 3), dtype=np.uint64)
    _capi.lib().sg_cta_times(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    t = buf.reshape(6, 8192, 3)[:, :n].astype(np.int64)  # iterations T..T+5
    t0 = t[..., 0].min()
    st, en = (t[..., 0] - t0) / 1e3, (t[..., 1] - t0) / 1e3  # us
    # a window inside which every running CTA belongs to a recorded iteration:
    # from the first start of iteration T+2 to the last end of iteration T+3
    a, b = st[2].min(), en[3].max()
    grid = np.arange(int(a), int(b))
    occ = np.array([np.count_nonzero((st <= g) & (en > g)) for g in grid])
    one = t[0]
    d0 = (one[:, 1] - one[:, 0]) / 1e3
    print(json.dumps({"window_us": [float(a), float(b)], "max_resident": int(occ.max()),
                      "slot_utilisation_in_window": float(occ.mean() / occ.max()),
                      "cta_us_mean": float(d0.mean()), "cta_us_p10": float(np.percentile(d0, 10)),
                      "cta_us_p90": float(np.percentile(d0, 90)),
                      "one_iteration_span_us": float((one[:, 1].max() - one[:, 0].min()) / 1e3),
                      "occupancy_profile_every_25us": [int(occ[g]) for g in range(0, len(occ), 25)]}, indent=1))


if __name__ == "__main__":
    main()
