"""Plans of S small swarms (256 particles x 500 iterations, 21-day windows): device ms per plan run."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402
from tools.bench_configs import window  # noqa: E402


def main():
    ctx = eng.Context(0)
    wins = [window(ctx, w, 20) for w in range(139)]
    for S in [int(x) for x in sys.argv[1:]] or [1, 4, 16, 64, 148]:
        swarms = [dict(window=wins[k % 139], lower=[0] * 6, upper=[2.0, 2.0, 13.0, 13.0, 1.0, 0.1], n_particles=256,
                       max_iters=500, seed=bench.mix_seed(7, k)) for k in range(S)]
        plan = eng.Plan(ctx, swarms)
        plan.run_timed()
        s, k = plan.run_timed()
        print(f"S={S:4d} launches={plan.step_launches:5d} device_ms={s + k:8.2f} evals/s={plan.evals / (s + k) * 1e3:.3e}",
              flush=True)


if __name__ == "__main__":
    main()
