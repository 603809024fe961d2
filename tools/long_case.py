"""One long-window plan for ncu: 40 windows of tau days x 4096 particles x 3 iterations (tools/long_windows.py shape)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402
from tools.bench_configs import stage2, window  # noqa: E402


def main():
    tau = int(sys.argv[1]) if len(sys.argv) > 1 else 201
    ctx = eng.Context(0)
    wins = [window(ctx, w, tau) for w in range(40)]
    plan = eng.Plan(ctx, [dict(window=wins[w], lower=[0] * 6, upper=stage2(tau), n_particles=4096, max_iters=3,
                               seed=bench.mix_seed(5, w)) for w in range(40)])
    print(tau, plan.run_timed(), plan.ramp_substeps / plan.evals)


if __name__ == "__main__":
    main()
