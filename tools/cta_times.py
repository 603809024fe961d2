"""CTA start/end times of one step-kernel launch of C3 (one 2^20-particle swarm), from a
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
    win = window(ctx, 60, 35)
    plan = eng.Plan(ctx, [dict(window=win, lower=[0] * 6, upper=stage2(35), n_particles=1 << 20, max_iters=8,
                               seed=7)])
    plan.run_timed()
    buf = np.zeros((1 << 14, 3), dtype=np.uint64)
    _capi.lib().sg_cta_times(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    n = 8192
    t = buf[:n].astype(np.int64)
    t0 = t[:, 0].min()
    st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3  # us
    span = en.max()
    dur = en - st
    # occupancy over time: CTAs resident at each microsecond
    grid = np.arange(0, int(span) + 1)
    occ = np.array([np.count_nonzero((st <= g) & (en > g)) for g in grid])
    full = occ.max()
    busy = dur.sum() / (full * span)
    drain_start = float(np.max(st))  # the last CTA starts
    print(json.dumps({"span_us": float(span), "cta_us_mean": float(dur.mean()), "cta_us_p10": float(np.percentile(dur, 10)),
                      "cta_us_p90": float(np.percentile(dur, 90)), "max_resident": int(full),
                      "slot_utilisation": float(busy), "last_start_us": drain_start,
                      "drain_us": float(span - drain_start),
                      "occupancy_profile_every_50us": [int(occ[g]) for g in range(0, len(occ), 50)]}, indent=1))


if __name__ == "__main__":
    main()
