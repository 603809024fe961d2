"""The other BASELINE.json configs on one GPU (bench.py measures configs[1], C2).

  C1  single 21-day window (tau=20), 256 particles x 500 iterations
  C3  single 36-day window, one swarm of 1,048,576 particles x --c3-iters iterations
  C4  parameter-stability restarts: 139 windows x R restarts x 256 particles x 500
      iterations (R = --c4-restarts; BASELINE's 1024 restarts shard over 8 GPUs)
  C5  forecast-scenario ensemble: 10^6 sampled parameter sets per window, 21-day
      forecast, all 139 windows (device time per window; host copy excluded)

Each prints one JSON line (evals/s device-timed with CUDA events; the
reference CPU path timed on a bounded sample beside it when --cpu).
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402

I, R, D = bench.load_series()
N = bench.POPULATION


def window(ctx, w, tau, spec=bench.SPEC):
    a = w * bench.DELTA
    sl = slice(a, a + tau + 1)
    return eng.Window(ctx, I[sl], R[sl], D[sl], [N - I[a] - R[a] - D[a], I[a], R[a], D[a]], N, spec)


def stage2(tau):
    return [2.0, 2.0, float(tau - 7), float(tau - 7), 1.0, 0.1]


def timed_plan(ctx, swarms, reps=2):
    plan = eng.Plan(ctx, swarms)
    plan.run_timed()
    best = min(plan.run_timed()[1] for _ in range(reps))
    ramp = plan.ramp_substeps
    res = plan.results()
    evals = plan.evals
    plan.close()
    return best, evals, ramp, res


def cpu_sample(w, tau, n, iters):
    from oracle import oracle_py
    ora = oracle_py.load("reference" if oracle_py.REF_SO.exists() else "port")
    a = w * bench.DELTA
    sl = slice(a, a + tau + 1)
    import os
    t = time.perf_counter()
    ora.fit_swarm(bench.SPEC, I[sl], R[sl], D[sl], [N - I[a] - R[a] - D[a], I[a], R[a], D[a]], N, [0] * 6,
                  stage2(tau), n, iters, seed=bench.mix_seed(bench.BASE_SEED, w), n_threads=os.cpu_count())
    dt = time.perf_counter() - t
    return n * iters / dt, dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c3-iters", type=int, default=100)
    ap.add_argument("--c4-restarts", type=int, default=32)
    ap.add_argument("--c5-windows", type=int, default=139)
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--only", default="c1,c3,c4,c5", help="comma-separated subset of c1,c3,c4,c5")
    args = ap.parse_args()
    only = set(args.only.split(","))
    ctx = eng.Context(0)
    peak = eng.probe_fp64_rate(ctx)
    # nominal FP64 lane-op rate (bench.py's roofline denominator): SMs x 64 x max SM clock
    import subprocess
    try:
        mhz = float(subprocess.run(["nvidia-smi", "--query-gpu=clocks.max.sm", "--format=csv,noheader,nounits"],
                                   capture_output=True, text=True, timeout=30).stdout.split()[0])
        nominal = torch.cuda.get_device_properties(0).multi_processor_count * 64 * mhz * 1e6
    except Exception:  # noqa: BLE001 - no nvidia-smi: the probe stands in
        nominal = peak

    if "c1" in only:
        # C1
        win = window(ctx, 0, 20)
        ms, evals, ramp, res = timed_plan(ctx, [dict(window=win, lower=[0] * 6, upper=stage2(20), n_particles=256,
                                                     max_iters=500, seed=bench.mix_seed(bench.BASE_SEED, 0))], reps=5)
        line = {"config": "C1", "evals": evals, "device_ms": ms, "evals_per_s": evals / ms * 1e3, "best": res[0][2]}
        # C1 end to end through the public fit_window (host series in, FitResult
        # out: window setup, swarm, re-integration, R^2)
        import paper_2204_12346_b200.sirdfit as sf
        data = sf.EpiSeries(infectious=list(I), recovered_cum=list(R), deaths_cum=list(D), new_cases=[0.0] * len(I))
        win0 = sf.Window(index=0, start=0, length=21)
        kw = dict(objective=bench.SPEC, particles=256, iters=500, seed=bench.mix_seed(bench.BASE_SEED, 0))
        sf.fit_window(data, win0, N, **kw)  # warm
        t0 = time.perf_counter()
        for _ in range(5):
            fit = sf.fit_window(data, win0, N, **kw)
        line["e2e_ms"] = (time.perf_counter() - t0) / 5 * 1e3
        line["e2e_objective_matches"] = fit.objective == res[0][2]
        if args.cpu:
            v, dt = cpu_sample(0, 20, 256, 500)
            line["cpu_reference_evals_per_s"] = v
            line["cpu_reference_s"] = dt
        print(json.dumps(line), flush=True)

    if "c3" in only:
        # C3
        win = window(ctx, 60, 35)
        ms, evals, ramp, res = timed_plan(ctx, [dict(window=win, lower=[0] * 6, upper=stage2(35), n_particles=1 << 20,
                                                     max_iters=args.c3_iters, seed=7)], reps=1)
        ops = evals * bench.ops_per_eval(36) + bench.RAMP_OPS * ramp
        print(json.dumps({"config": "C3", "particles": 1 << 20, "iters": args.c3_iters, "device_ms": ms,
                          "evals_per_s": evals / ms * 1e3, "fp64_frac": ops / (ms * 1e-3) / peak, "best": res[0][2]}),
              flush=True)

    wins = [window(ctx, w, 35) for w in range(139)]
    if "c4" in only:
        # C4 (fraction of the restarts)
        swarms = [dict(window=wins[w], lower=[0] * 6, upper=stage2(35), n_particles=256, max_iters=500,
                       seed=bench.mix_seed(bench.BASE_SEED + r, w)) for r in range(args.c4_restarts) for w in range(139)]
        ms, evals, ramp, res = timed_plan(ctx, swarms, reps=1)
        ops = evals * bench.ops_per_eval(36) + bench.RAMP_OPS * ramp
        full = 139 * 1024 * 256 * 500
        print(json.dumps({"config": "C4", "restarts": args.c4_restarts, "swarms": len(swarms), "device_ms": ms,
                          "evals_per_s": evals / ms * 1e3, "fp64_frac": ops / (ms * 1e-3) / peak,
                          "full_c4_evals": full, "full_c4_projected_s_1gpu": full / (evals / ms * 1e3),
                          "full_c4_projected_s_8gpu": full / (evals / ms * 1e3) / 8}), flush=True)

    if "c5" in only:
        # C5 ensemble: 1e6 sampled parameter sets per window, 21-day forecast,
        # reduced to per-day quantile bands on the device (nothing but the bands
        # leaves HBM)
        n = 1_000_000
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream = torch.cuda.ExternalStream(ctx.stream)
        wins[0].forecast_ensemble_bands([0] * 6, stage2(35), seed=1, n=n, horizon=21)  # warm
        seeds = [bench.mix_seed(2204, w) for w in range(args.c5_windows)]
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            e0.record(stream)
            for w in range(args.c5_windows):
                bands, counts, _ = wins[w].forecast_ensemble_bands([0] * 6, stage2(35), seed=seeds[w], n=n, horizon=21)
            e1.record(stream)
        e1.synchronize()
        wall_single = time.perf_counter() - t0
        single_ms = e0.elapsed_time(e1)
        # the same work through the pipelined many-window call (warmed once:
        # the first call grows the device pool by the pipeline's buffers)
        ctx.forecast_ensemble_bands_batch(wins[:2], [0] * 6, stage2(35), seeds[:2], n, 21)
        ramp0 = ctx.band_stats[2]
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            e0.record(stream)
            all_bands, all_counts = ctx.forecast_ensemble_bands_batch(wins[:args.c5_windows], [0] * 6, stage2(35), seeds,
                                                                      n, 21)
            e1.record(stream)
        e1.synchronize()
        wall = time.perf_counter() - t0
        dev_ms = e0.elapsed_time(e1)
        assert np.array_equal(all_bands[-1], bands, equal_nan=True)
        ramp = ctx.band_stats[2] - ramp0  # the timed call's ramp substeps (counted by the ensemble kernel)
        ops = (35 * 24 * 14 + 21 * 24 * 14)  # window + forecast substeps per sample, no ramp credit
        print(json.dumps({"config": "C5", "windows": args.c5_windows, "samples_per_window": n, "horizon": 21,
                          "device_ms": dev_ms, "wall_ms": wall * 1e3, "per_window_calls_device_ms": single_ms,
                          "per_window_calls_wall_ms": wall_single * 1e3,
                          "samples_per_s": args.c5_windows * n / (dev_ms * 1e-3),
                          "fp64_frac_floor": args.c5_windows * n * ops / (dev_ms * 1e-3) / peak,
                          "ramp_substeps_per_sample": ramp / (args.c5_windows * n),
                          "fp64_frac_ramp_credit": (args.c5_windows * n * ops + bench.RAMP_OPS * ramp)
                          / (dev_ms * 1e-3) / peak,
                          "fp64_frac_floor_nominal": args.c5_windows * n * ops / (dev_ms * 1e-3) / nominal,
                          "fp64_frac_ramp_credit_nominal": (args.c5_windows * n * ops + bench.RAMP_OPS * ramp)
                          / (dev_ms * 1e-3) / nominal,
                          "last_window_day21_median_deaths": float(bands[0, -1]), "finite_last": int(counts[-1])}),
              flush=True)


if __name__ == "__main__":
    main()
