"""The full C4 parameter-stability study on ONE GPU: 139 windows x 1024 restarts
x 256 particles x 500 iterations (1.82e10 evaluations) as a single plan."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402
from tools.bench_configs import stage2, window  # noqa: E402


def main():
    restarts = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    ctx = eng.Context(0)
    peak = eng.probe_fp64_rate(ctx)
    wins = [window(ctx, w, 35) for w in range(139)]
    swarms = [dict(window=wins[w], lower=[0] * 6, upper=stage2(35), n_particles=256, max_iters=500,
                   seed=bench.mix_seed(bench.BASE_SEED + r, w)) for r in range(restarts) for w in range(139)]
    t = time.perf_counter()
    plan = eng.Plan(ctx, swarms)
    setup = time.perf_counter() - t
    seed_ms, steps_ms = plan.run_timed()
    res = plan.results()
    evals = plan.evals
    ms = seed_ms + steps_ms
    ops = evals * bench.ops_per_eval(36) + bench.RAMP_OPS * plan.ramp_substeps
    print(json.dumps({"config": "C4-full", "restarts": restarts, "swarms": len(swarms), "evals": evals,
                      "plan_setup_s": setup, "device_ms": ms, "evals_per_s": evals / ms * 1e3,
                      "fp64_frac": ops / (ms * 1e-3) / peak, "failed": sum(r[0] != 0 for r in res),
                      "best_w0_r0": res[0][2]}), flush=True)


if __name__ == "__main__":
    main()
