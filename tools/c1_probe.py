"""C1 phase breakdown from a diagnostic build (-DSG_C1_PROBE=1): clock64 stamps per
(warp, iteration) of pso_swarm_kernel — iteration start, move done, eval done, warp
argmin done, cluster barrier passed, gbest published.

    python -c "from paper_2204_12346_b200 import build; build.build(out='tools/libsirdgpu_c1probe.so', extra=['-DSG_C1_PROBE=1'])"
    SG_LIB=$PWD/tools/libsirdgpu_c1probe.so python tools/c1_probe.py
"""
import ctypes
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402
from paper_2204_12346_b200 import _capi  # noqa: E402


def main():
    I, R, D = bench.load_series()
    N = bench.POPULATION
    ctx = eng.Context(0)
    win = eng.Window(ctx, I[:21], R[:21], D[:21], [N - I[0] - R[0] - D[0], I[0], R[0], D[0]], N, bench.SPEC)
    plan = eng.Plan(ctx, [dict(window=win, lower=[0] * 6, upper=[2.0, 2.0, 13.0, 13.0, 1.0, 0.1], n_particles=256,
                               max_iters=500, seed=bench.mix_seed(bench.BASE_SEED, 0))])
    s, k = plan.run_timed()
    buf = np.zeros((8, 512, 6), dtype=np.uint64)
    _capi.lib().sg_c1_probe(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    t = buf[:, 1:500, :].astype(np.int64)  # iterations 1..499 (0 has no move)
    ph = {"move": t[..., 1] - t[..., 0], "eval": t[..., 2] - t[..., 1], "argmin": t[..., 3] - t[..., 2],
          "cta_fold+cluster_sync": t[..., 4] - t[..., 3], "gbest": t[..., 5] - t[..., 4],
          "iteration": t[..., 5] - t[..., 0]}
    out = {"device_ms": k, "per_iter_us": k * 1e3 / 500,
           "cycles_mean": {n: float(v.mean()) for n, v in ph.items()},
           "eval_cycles_per_warp_mean": [float(x) for x in ph["eval"].mean(axis=1)],
           "eval_max_over_warps_mean": float(ph["eval"].max(axis=0).mean()),
           "eval_min_over_warps_mean": float(ph["eval"].min(axis=0).mean())}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
