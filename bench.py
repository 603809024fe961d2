#!/usr/bin/env python
"""bench.py — particle-window cost evaluations/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "C2"): the full overlapping moving-window
sweep of the synthetic Poland-like series (tests/golden/poland_like.csv,
450 days; tau=35, delta=3 -> 139 windows of 36 days), one PSO swarm of 4096
particles x 1000 iterations per window, objective ird-mxse, stage-2 bounds,
window w seeded mix_seed(base, w) (calibration.cpp:199).  One "step" = that
whole sweep = 139 x 4096 x 1000 = 5.69e8 particle-window evaluations.

Multi-GPU (torchrun, one process per GPU): the unit of work is a
(window, restart) swarm; rank r runs restart r of the 139-window sweep
(base seed + r), i.e. the C4 restart study sharded one restart per GPU.
There is no cross-GPU data exchange on the path; torch.distributed (NCCL)
only carries the barrier and the max-over-ranks timing.  scaling = "weak".

  value        evals/s over the job: device-timed (CUDA events on the engine
               stream) with windows resident in HBM, max over ranks.
  e2e          same metric through the public C-ABI calibration call
               (sg_fit_all_windows_series: host series in, host results out;
               H2D of the series and D2H of fits/histories inside the timed
               region).
  roofline     the fused integrate-and-score step kernel (pso_step_kernel):
               algorithmic FP64 ops per launch / its average device time, vs
               the FP64 issue rate measured on this GPU (sg_probe_fp64_rate).
  cpu_baseline the reference C++ (oracle/_ref, built unmodified from
               /root/reference) on the host cores, bounded sample.

`--impl reference` times the reference's own CPU implementation (oracle/_ref,
else the C restatement) on the same workload and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "particle-window cost evals/sec (SIRD integrations/sec)"
UNIT = "evals/s"
TAU, DELTA = 35, 3
PARTICLES, ITERS = 4096, 1000
SPEC = "ird-mxse"
STAGE2_HI = [2.0, 2.0, float(TAU - 7), float(TAU - 7), 1.0, 0.1]
BASE_SEED = 2204
POPULATION = 38_000_000.0


def load_series():
    a = np.genfromtxt(ROOT / "tests" / "golden" / "poland_like.csv", delimiter=",", names=True)
    return (np.ascontiguousarray(a["infectious"]), np.ascontiguousarray(a["recovered_cum"]),
            np.ascontiguousarray(a["deaths_cum"]))


def n_windows(n_days):
    return 1 + (n_days - 1 - TAU) // DELTA


def mix_seed(base, index):
    m = 0xFFFFFFFFFFFFFFFF
    z = (base + 0x9E3779B97F4A7C15 * (index + 1)) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def ops_per_eval(n_days, c_score=12, substeps=24):
    """Algorithmic FP64 ops of one particle-window evaluation without ramp credit
    (SURVEY.md §8d): 14 per Euler substep (model.cpp:66-74, 96-99) + c_score per
    scored day (12 for IRD-MXSE: 3 x {sub, mul, mul, max}, objectives.cpp:15-39).
    Day 0 scores the initial state, identical for every particle; the engine
    scores it once per window, so it is not credited per evaluation."""
    return (n_days - 1) * substeps * 14 + (n_days - 1) * c_score


RAMP_OPS = 5  # per ramp substep: t, t - t1, slope*, beta1+, beta/N (model.cpp:62-63, 67)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, flag in zip(names, parts[4:8]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# Collective plumbing: NCCL between GPUs.  SG_BENCH_BACKEND=gloo (with ranks
# sharing a GPU) exists only to exercise the multi-rank code path on a
# one-GPU box; ranks never wait on each other inside kernels.
BACKEND = os.environ.get("SG_BENCH_BACKEND", "nccl")


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        local = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local)
        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(BACKEND)
    return world, rank, local


def _coll_device():
    return "cuda" if BACKEND == "nccl" else "cpu"


def allreduce_max(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def load_profile_traffic():
    """DRAM bytes and executed FP64 ops per particle-iteration of the step
    kernel from the committed ncu --set full summary
    (profiles/ncu_step_kernel_*.json), if any."""
    for p in sorted((ROOT / "profiles").glob("ncu_step_kernel_r*.json"), reverse=True):
        try:
            d = json.loads(p.read_text())
            return d.get("dram_bytes_per_particle"), p.name, d.get("fp64_ops_per_particle_executed")
        except (OSError, ValueError):
            continue
    return None, None, None


# ---------------------------------------------------------------------------------------------
def cpu_reference_sample(I, R, D, budget_s=12.0, threads=None):
    """The reference C++ (oracle/_ref) or, absent, the C restatement, on the
    host cores: whole window swarms of the sweep (PARTICLES particles, up to
    ITERS iterations, the workload's seeds) until the time budget is spent;
    returns (evals/s, kind, cores, sample description)."""
    from oracle import oracle_py
    kind = "reference" if oracle_py.REF_SO.exists() else "port"
    ora = oracle_py.load(kind)
    threads = threads or os.cpu_count() or 1
    lo = [0.0] * 6

    def run(w, iters):
        a = w * DELTA
        sl = slice(a, a + TAU + 1)
        init = [POPULATION - I[a] - R[a] - D[a], I[a], R[a], D[a]]
        t = time.perf_counter()
        ora.fit_swarm(SPEC, I[sl], R[sl], D[sl], init, POPULATION, lo, STAGE2_HI, PARTICLES, iters,
                      seed=mix_seed(BASE_SEED, w), n_threads=threads)
        return time.perf_counter() - t

    t2 = run(60, 2)
    iters = int(max(2, min(ITERS, budget_s / max(t2 / 2, 1e-6))))
    spent, evals, windows = 0.0, 0, []
    for w in range(0, n_windows(len(I)), 17):
        spent += run(w, iters)
        evals += PARTICLES * iters
        windows.append(w)
        if spent >= budget_s:
            break
    return evals / spent, kind, threads, f"windows {windows} of the sweep, {PARTICLES} particles x {iters} " \
                                         f"iterations each ({evals} evals, {spent:.1f} s)"


def bench_reference(args):
    world, rank, _ = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return 0
    I, R, D = load_series()
    for _ in range(args.warmup):
        cpu_reference_sample(I, R, D, budget_s=2.0)
    vals, samples = [], []
    for _ in range(args.steps):
        v, kind, cores, sample = cpu_reference_sample(I, R, D, budget_s=args.ref_budget)
        vals.append(v)
        samples.append(sample)
    v = statistics.median(vals)
    n_win = n_windows(len(I))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * n_win * PARTICLES * ITERS / v, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C2 window sweep ({n_win} windows x {PARTICLES} particles x {ITERS} iterations, "
                               f"{SPEC}, stage2); each reference step times a bounded sample of it",
                   "windows": n_win, "particles": PARTICLES, "iterations": ITERS, "objective": SPEC},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": samples[-1]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
def bench_ours(args):
    import torch

    world, rank, local = dist_setup()
    import paper_2204_12346_b200 as eng
    from paper_2204_12346_b200 import _capi

    I, R, D = load_series()
    n_win = n_windows(len(I))
    iters = args.iters
    base = BASE_SEED + rank  # restart r of the sweep on rank r

    ctx = eng.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=local)
    fp64_peak = eng.probe_fp64_rate(ctx)

    wins = []
    for w in range(n_win):
        a = w * DELTA
        sl = slice(a, a + TAU + 1)
        wins.append(eng.Window(ctx, I[sl], R[sl], D[sl], [POPULATION - I[a] - R[a] - D[a], I[a], R[a], D[a]],
                               POPULATION, SPEC))
    swarms = [dict(window=wins[w], lower=[0.0] * 6, upper=STAGE2_HI, n_particles=PARTICLES, max_iters=iters,
                   seed=mix_seed(base, w)) for w in range(n_win)]
    plan = eng.Plan(ctx, swarms)
    evals_per_step = plan.evals
    step_launches = plan.step_launches

    for _ in range(args.warmup):
        plan.run()
    torch.cuda.synchronize(local)

    # ---- device-timed value (windows resident in HBM) ----
    launches0 = ctx.launch_count
    step_ms, seed_ms = [], []
    with ClockSampler(local) as clocks:
        barrier(world)
        torch.cuda.synchronize(local)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                s_ms, k_ms = plan.run_timed()
                seed_ms.append(s_ms)
                step_ms.append(k_ms)
            e1.record(stream)
        e1.synchronize()
        torch.cuda.synchronize(local)
        barrier(world)
    launches = ctx.launch_count - launches0
    ms_total = e0.elapsed_time(e1)
    ms_per_step = allreduce_max(ms_total / args.steps, world)
    total_evals = allreduce_sum(evals_per_step, world)
    value = total_evals / (ms_per_step * 1e-3)

    # roofline: the fused step kernel, all its launches of a step (the
    # partition lanes overlap, so the per-launch figure is the aggregate:
    # algorithmic ops of every step launch / device time of the step launches)
    ramp_substeps = plan.ramp_substeps  # of the last timed run (identical every run)
    ops_floor = evals_per_step * ops_per_eval(TAU + 1)
    ops_step = ops_floor + RAMP_OPS * ramp_substeps
    steps_kernel_ms = statistics.mean(step_ms)
    kernel_ms = steps_kernel_ms / (step_launches if step_launches else 1)
    achieved = ops_step / (steps_kernel_ms * 1e-3) / 1e12
    achieved_floor = ops_floor / (steps_kernel_ms * 1e-3) / 1e12
    bytes_per_particle, prof, fp64_exec = load_profile_traffic()
    # nominal FP64 lane-op rate: SMs x 64 lanes x max SM clock
    clk = clocks.summary() if hasattr(clocks, "summary") else {}
    sm_max = (clk or {}).get("sm_max_mhz") or 0.0
    nominal_peak = torch.cuda.get_device_properties(local).multi_processor_count * 64 * sm_max * 1e6
    # one "launch" of the roofline = one iteration of the sweep (all lanes)
    traffic = bytes_per_particle * n_win * PARTICLES if bytes_per_particle else None

    # ---- e2e through the public calibration C-ABI with host buffers ----
    settings = _capi.sg_fit_settings(1, 0, 0.0, 2.0, 0.0, 1.0, 0.0, 0.1, 7, PARTICLES, iters, 0.5, 0.5, 0.5,
                                     POPULATION, 24)
    import ctypes
    recs = (_capi.sg_fit_record * n_win)()
    trajs = np.empty((n_win, TAU + 1, 4))
    nw, failed, mean = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_double()
    pinned = [torch.from_numpy(x).pin_memory() for x in (I, R, D)]
    ptrs = [ctypes.cast(t.data_ptr(), _capi._dp) for t in pinned]

    def e2e_call():
        rc = _capi.lib().sg_fit_all_windows_series(ctx.handle, *ptrs, len(I), TAU, DELTA, ctypes.byref(settings),
                                                   base, n_win, ctypes.byref(nw), recs, _capi._d(trajs),
                                                   ctypes.byref(mean), ctypes.byref(failed))
        ctx.check(rc)

    e2e_call()  # warm (allocations, module load)
    e2e_steps = max(1, min(args.steps, 3))
    barrier(world)
    t = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    e2e_s = allreduce_max((time.perf_counter() - t) / e2e_steps, world)
    e2e_value = total_evals / e2e_s
    h2d = 3 * len(I) * 8
    d2h = n_win * (ctypes.sizeof(_capi.sg_fit_record) + (TAU + 1) * 4 * 8)

    # parity spot check of the e2e result against the device-timed plan
    res = plan.results()
    ok = all(abs(recs[w].objective - res[w][2]) == 0.0 for w in range(n_win))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, kind, cores, sample = cpu_reference_sample(I, R, D, budget_s=args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}
    gpu_launches = int(allreduce_sum(launches, world))
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C2 window sweep: {n_win} windows x {PARTICLES} particles x {iters} iterations "
                                   f"(tau={TAU}, delta={DELTA}, {SPEC}, stage2), one sweep restart per GPU",
                       "windows": n_win, "particles": PARTICLES, "iterations": iters, "objective": SPEC,
                       "series": "tests/golden/poland_like.csv (synthetic Poland-like, 450 days)",
                       "parallelism": f"restarts x{world} (one per GPU, no collective)",
                       "l2": "working set (MT19937-64 engines 312 x 8 B per particle = 1.4 GB) exceeds L2"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "call": "sg_fit_all_windows_series (fit_all_windows) with host buffers",
                    "matches_device_run": ok},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": fp64_peak / 1e12, "unit": "TFLOP/s",
                         "frac": achieved * 1e12 / fp64_peak, "traffic": traffic,
                         "kernel": "pso_step_kernel<IRD,MXSE,24> (fused move+integrate+score+argmin)",
                         "ops_per_eval_floor": ops_per_eval(TAU + 1),
                         "ramp_substeps_per_eval": ramp_substeps / evals_per_step,
                         "ops_per_eval": ops_step / evals_per_step,
                         "fp64_ops_per_eval_executed": fp64_exec,  # ncu SASS counts (profile), incl. PSO move/setup
                         "frac_floor": achieved_floor * 1e12 / fp64_peak,
                         "ops_note": "algorithmic FP64 ops (SURVEY.md §8d: 14/substep + 5/ramp substep + 12/scored day), "
                                     "DADD/DMUL without FMA for bit parity (the kernel scores MXSE with 2 of the "
                                     "credited 4 ops per compartment-day, exactly, DESIGN.md §3); peak = FP64 issue "
                                     "rate measured "
                                     "on this GPU by sg_probe_fp64_rate (neither MEASURED_PEAKS.json nor "
                                     "B200_PROFILING.md has an FP64 figure)",
                         "peak_nominal": nominal_peak / 1e12,
                         "frac_nominal": achieved * 1e12 / nominal_peak if nominal_peak else None,
                         "peak_nominal_note": "SMs x 64 FP64 lanes x max SM clock (the probe reaches "
                                              f"{fp64_peak / nominal_peak:.3f} of it)" if nominal_peak else None,
                         "kernel_ms_per_launch": kernel_ms, "launches_per_step": step_launches,
                         "step_kernels_ms": steps_kernel_ms, "seed_ms": statistics.mean(seed_ms), "profile": prof},
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "gpu_launches": gpu_launches,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--iters", type=int, default=ITERS, help="PSO iterations per swarm (default: the config's 1000)")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--ref-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return bench_reference(args)
    return bench_ours(args)


if __name__ == "__main__":
    sys.exit(main())
