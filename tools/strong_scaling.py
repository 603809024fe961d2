"""Strong-scaling projection of the C2 sweep on one B200.

bench.py --split windows gives rank r of N the contiguous share
sharding.partition(139, N, r); ranks never exchange data, so the N-GPU step
time is the slowest rank's plan time — rank 0's, whose share is the largest
(ceil(139 / N) windows).  This runs rank 0's share of N = 1, 2, 4, 8 on one
GPU and reports the projected efficiency t_1 / (N * t_N), i.e. what the
driver's SCALE run would see from the work split alone (no NCCL on the path).
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402
from paper_2204_12346_b200.sharding import partition  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else bench.ITERS
    I, R, D = bench.load_series()
    n_win = bench.n_windows(len(I))
    ctx = eng.Context(0)
    wins = []
    for w in range(n_win):
        Iw, Rw, Dw, init = bench._window_inputs(I, R, D, w)
        wins.append(eng.Window(ctx, Iw, Rw, Dw, init, bench.POPULATION, bench.SPEC))
    t1 = None
    for n in (1, 2, 4, 8):
        share = list(partition(n_win, n, 0))
        plan = eng.Plan(ctx, [dict(window=wins[w], lower=[0.0] * 6, upper=bench.STAGE2_HI,
                                   n_particles=bench.PARTICLES, max_iters=iters, seed=bench.mix_seed(bench.BASE_SEED, w))
                              for w in share])
        for _ in range(3):
            plan.run()
        ms = min(sum(plan.run_timed()) for _ in range(3))
        if n == 1:
            t1 = ms
        evals = plan.evals
        plan.close()
        print(json.dumps({"gpus": n, "rank0_windows": len(share), "rank0_particles": len(share) * bench.PARTICLES,
                          "iters": iters, "rank0_ms": ms, "per_gpu_evals_per_s": evals / ms * 1e3,
                          "projected_job_evals_per_s": n_win * bench.PARTICLES * iters / ms * 1e3,
                          "projected_efficiency": t1 / (n * ms)}), flush=True)


if __name__ == "__main__":
    main()
