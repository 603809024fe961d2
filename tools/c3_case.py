"""C3 alone: one 36-day window, one swarm of 2^20 particles x 100 iterations (prints device ms)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2204_12346_b200 as eng  # noqa: E402
from tools.bench_configs import stage2, window  # noqa: E402


def main():
    ctx = eng.Context(0)
    win = window(ctx, 60, 35)
    plan = eng.Plan(ctx, [dict(window=win, lower=[0] * 6, upper=stage2(35), n_particles=1 << 20, max_iters=100,
                               seed=7)])
    for _ in range(2):
        s, k = plan.run_timed()
        print(f"C3 seed {s:.2f} ms steps {k:.2f} ms ({k / 100:.3f} ms/iter) best {plan.results()[0][2]}", flush=True)


if __name__ == "__main__":
    main()
