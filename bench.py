#!/usr/bin/env python
"""bench.py — particle-window cost evaluations/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "C2"): the full overlapping moving-window
sweep of the synthetic Poland-like series (tests/golden/poland_like.csv,
450 days; tau=35, delta=3 -> 139 windows of 36 days), one PSO swarm of 4096
particles x 1000 iterations per window, objective ird-mxse, stage-2 bounds,
window w seeded mix_seed(base, w) (calibration.cpp:199).  One "step" = that
whole sweep = 139 x 4096 x 1000 = 5.69e8 particle-window evaluations.

Multi-GPU (torchrun, one process per GPU; --split):
  windows   (default) the ONE sweep's 139 windows split into contiguous,
            balanced shares (paper_2204_12346_b200/sharding.partition); each
            rank runs its share as one plan.  Seeds depend on the window only
            (calibration.cpp:199), so the shards are the single-GPU sweep bit
            for bit.  scaling = "strong" (total work fixed).
  restarts  rank r runs restart r of the whole sweep (base seed + r): the C4
            restart study, one restart per GPU.  scaling = "weak".
There is no cross-GPU data exchange on the path; torch.distributed (NCCL)
only carries the barrier and the max-over-ranks timing.

  value        evals/s over the job: device-timed (CUDA events on the engine
               stream) with windows resident in HBM, max over ranks.
  e2e          same metric through the public C-ABI calibration call
               (sg_fit_all_windows_series / its per-rank window range: host
               series in, host results out), every step; the byte counts are
               every copy the call made, counted by the engine.
  roofline     the fused integrate-and-score step kernel (pso_step_kernel):
               algorithmic FP64 ops per launch / its average device time, vs
               the nominal FP64 lane-op rate (SMs x 64 x max clock).
  cpu_baseline the reference C++ (oracle/_ref, built unmodified from
               /root/reference) on all host cores, a bounded stratified sample
               of whole windows (rank 0), plus the same on one thread.
  parity       the device plan's histories / bests for the windows the
               cpu_baseline sample ran, compared bit for bit with the
               reference's.

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
def stratified(windows):
    """Windows in van der Corput order (0, 1/2, 1/4, 3/4, ... of the range), so
    that every prefix of the list spreads over the whole sweep: a time-bounded
    sample of whole windows then sees early, middle and late windows (their
    ramp shares, and so their cost, differ)."""
    windows = list(windows)
    n = len(windows)
    order, seen, k = [], set(), 0
    while len(order) < n and k < 64 * n + 64:
        x, f, i = 0.0, 0.5, k
        while i:
            x += f * (i & 1)
            i >>= 1
            f *= 0.5
        j = min(n - 1, int(round(x * (n - 1))))
        if j not in seen:
            seen.add(j)
            order.append(windows[j])
        k += 1
    return order + [w for w in windows if w not in set(order)]


def _window_inputs(I, R, D, w):
    a = w * DELTA
    sl = slice(a, a + TAU + 1)
    return I[sl], R[sl], D[sl], [POPULATION - I[a] - R[a] - D[a], I[a], R[a], D[a]]


def cpu_reference_sample(I, R, D, budget_s=12.0, threads=None, windows=None, base=BASE_SEED, max_iters=ITERS):
    """The reference C++ (oracle/_ref) or, absent, the C restatement, on the
    host cores: whole window swarms of the sweep (PARTICLES particles, up to
    ITERS iterations, the workload's seeds mix_seed(base, w)), windows in
    stratified order, until the time budget is spent.  Returns (evals/s, kind,
    cores, sample description, {window: (status, best, cost, history)})."""
    from oracle import oracle_py
    kind = "reference" if oracle_py.REF_SO.exists() else "port"
    ora = oracle_py.load(kind)
    threads = threads or os.cpu_count() or 1
    lo = [0.0] * 6
    results = {}

    def run(w, iters, n_threads):
        Iw, Rw, Dw, init = _window_inputs(I, R, D, w)
        t = time.perf_counter()
        out = ora.fit_swarm(SPEC, Iw, Rw, Dw, init, POPULATION, lo, STAGE2_HI, PARTICLES, iters,
                            seed=mix_seed(base, w), n_threads=n_threads)
        return time.perf_counter() - t, out

    order = stratified(windows if windows is not None else range(n_windows(len(I))))
    t2, _ = run(order[0], 2, threads)
    iters = int(max(min(2, max_iters), min(max_iters, budget_s / max(t2 / 2, 1e-6))))
    spent, evals, sampled = 0.0, 0, []
    for w in order:
        dt, out = run(w, iters, threads)
        spent += dt
        evals += PARTICLES * iters
        sampled.append(w)
        results[w] = out
        if spent >= budget_s:
            break
    return evals / spent, kind, threads, {"windows": sampled, "iterations": iters, "particles": PARTICLES,
                                          "evals": evals, "seconds": spent}, results


def cpu_reference_one_thread(I, R, D, budget_s=3.0, w=69, base=BASE_SEED, max_iters=ITERS):
    """The same reference path on ONE host thread (SURVEY.md
    §8d: the reference is sometimes faster single-threaded, since
    parallel_for spawns threads per call): one window, a bounded number of
    iterations."""
    from oracle import oracle_py
    ora = oracle_py.load("reference" if oracle_py.REF_SO.exists() else "port")
    Iw, Rw, Dw, init = _window_inputs(I, R, D, w)
    t = time.perf_counter()
    ora.fit_swarm(SPEC, Iw, Rw, Dw, init, POPULATION, [0.0] * 6, STAGE2_HI, PARTICLES, 2, seed=mix_seed(base, w),
                  n_threads=1)
    per_iter = (time.perf_counter() - t) / 2
    iters = int(max(min(2, max_iters), min(max_iters, budget_s / max(per_iter, 1e-6))))
    t = time.perf_counter()
    ora.fit_swarm(SPEC, Iw, Rw, Dw, init, POPULATION, [0.0] * 6, STAGE2_HI, PARTICLES, iters, seed=mix_seed(base, w),
                  n_threads=1)
    dt = time.perf_counter() - t
    return PARTICLES * iters / dt, f"window {w}, {PARTICLES} particles x {iters} iterations on 1 thread ({dt:.1f} s)"


def parity_vs_reference(cpu_results, plan_results, window_slot):
    """Bitwise comparison of the reference's whole-window fits (the
    cpu_baseline sample) with the device plan's results for the same windows
    and seeds: histories over the sampled iterations; best cost, position and
    status when the sample ran all ITERS iterations (a shorter run is a
    prefix of the same trajectory, pso.cpp:129-143)."""
    checked, ok, iters = [], True, None
    for w, (rc, best, cost, hist) in sorted(cpu_results.items()):
        if w not in window_slot:
            continue
        status, gbest, gcost, ghist = plan_results[window_slot[w]]
        iters = len(hist)
        same = np.array_equal(np.asarray(ghist[:iters]).view(np.uint64), np.asarray(hist).view(np.uint64))
        if iters == len(ghist):
            same = same and status == rc and (rc != 0 or (gcost == cost and np.array_equal(
                np.asarray(gbest).view(np.uint64), np.asarray(best).view(np.uint64))))
        checked.append(w)
        ok = ok and bool(same)
    return {"windows": checked, "iters": iters, "particles": PARTICLES, "bit_exact": ok if checked else None,
            "against": "reference C++ (oracle/_ref) optimize() on the host, same seeds and bounds",
            "compared": "cost history (every iteration), best cost, best position, status"}


def bench_reference(args):
    world, rank, _ = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), 0
    if rank != 0:
        return 0
    I, R, D = load_series()
    for _ in range(args.warmup):
        cpu_reference_sample(I, R, D, budget_s=2.0)
    vals, samples = [], []
    for _ in range(args.steps):
        v, kind, cores, sample, _ = cpu_reference_sample(I, R, D, budget_s=args.ref_budget)
        vals.append(v)
        samples.append(sample)
    v = statistics.median(vals)
    n_win = n_windows(len(I))
    sweep_evals = n_win * PARTICLES * ITERS
    s = samples[-1]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * sweep_evals / v, "higher_is_better": True,
        "scaling": "strong" if args.split == "windows" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"C2 window sweep ({n_win} windows x {PARTICLES} particles x {ITERS} iterations, "
                               f"{SPEC}, stage2); each reference step times a bounded, stratified sample of its "
                               f"whole windows",
                   "windows": n_win, "particles": PARTICLES, "iterations": ITERS, "objective": SPEC},
        "sampled": True,
        "sample": {"windows_per_step": s["windows"], "iterations": s["iterations"],
                   "evals_per_step": s["evals"], "seconds_per_step": s["seconds"],
                   "order": "van der Corput over the 139 windows (early/middle/late mixed)"},
        "extrapolated": {"field": "ms_per_step", "how": "full-sweep evaluations / the sampled evals/s "
                                                        "(the rate is evals per wall second of whole windows)"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": f"windows {s['windows']}, {PARTICLES} particles x {s['iterations']} iterations "
                                   f"each ({s['evals']} evals, {s['seconds']:.1f} s)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------------
def bench_ours(args):
    import ctypes

    import torch

    world, rank, local = dist_setup()
    import paper_2204_12346_b200 as eng
    from paper_2204_12346_b200 import _capi
    from paper_2204_12346_b200.sharding import partition

    I, R, D = load_series()
    n_win = n_windows(len(I))
    iters = args.iters
    if args.split == "windows":
        # strong scaling: the ONE sweep's windows split over the GPUs
        # (contiguous balanced shares; seeds depend on the window only,
        # calibration.cpp:199, so the shards are the single-GPU sweep bit for bit)
        mine = list(partition(n_win, world, rank))
        base = BASE_SEED
    else:
        # weak scaling (C4): restart r of the whole sweep on rank r
        mine = list(range(n_win))
        base = BASE_SEED + rank

    ctx = eng.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=local)
    fp64_probe = eng.probe_fp64_rate(ctx)

    wins = {}
    for w in mine:
        Iw, Rw, Dw, init = _window_inputs(I, R, D, w)
        wins[w] = eng.Window(ctx, Iw, Rw, Dw, init, POPULATION, SPEC)
    swarms = [dict(window=wins[w], lower=[0.0] * 6, upper=STAGE2_HI, n_particles=PARTICLES, max_iters=iters,
                   seed=mix_seed(base, w)) for w in mine]
    slot = {w: k for k, w in enumerate(mine)}
    plan = eng.Plan(ctx, swarms) if swarms else None
    evals_per_step = plan.evals if plan else 0
    step_launches = plan.step_launches if plan else 0

    for _ in range(args.warmup):
        if plan:
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
                if plan:
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
    ramp_substeps = plan.ramp_substeps if plan else 0  # of the last timed run (identical every run)
    ops_floor = evals_per_step * ops_per_eval(TAU + 1)
    ops_step = ops_floor + RAMP_OPS * ramp_substeps
    steps_kernel_ms = statistics.mean(step_ms) if step_ms else float("nan")
    kernel_ms = steps_kernel_ms / (step_launches if step_launches else 1)
    achieved = ops_step / (steps_kernel_ms * 1e-3) / 1e12
    achieved_floor = ops_floor / (steps_kernel_ms * 1e-3) / 1e12
    bytes_per_particle, prof, fp64_exec = load_profile_traffic()
    clk = clocks.summary()
    sm_max = clk.get("sm_max_mhz") or 0.0
    n_sm = torch.cuda.get_device_properties(local).multi_processor_count
    # FP64 lane-op rate: SMs x 64 FP64 lanes x max SM clock (neither
    # MEASURED_PEAKS.json nor B200_PROFILING.md carries an FP64 figure)
    nominal_peak = n_sm * 64 * sm_max * 1e6 if sm_max else fp64_probe
    # one "launch" of the roofline = one iteration of the sweep (all lanes)
    traffic = bytes_per_particle * len(mine) * PARTICLES if bytes_per_particle else None

    # ---- e2e through the public calibration C-ABI with host buffers ----
    settings = _capi.sg_fit_settings(1, 0, 0.0, 2.0, 0.0, 1.0, 0.0, 0.1, 7, PARTICLES, iters, 0.5, 0.5, 0.5,
                                     POPULATION, 24)
    recs = (_capi.sg_fit_record * max(len(mine), 1))()
    trajs = np.empty((max(len(mine), 1), TAU + 1, 4))
    nw, failed, mean = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_double()
    pinned = [torch.from_numpy(x).pin_memory() for x in (I, R, D)]
    ptrs = [ctypes.cast(t.data_ptr(), _capi._dp) for t in pinned]
    L = _capi.lib()
    if args.split == "windows":
        call_name = "sg_fit_window_range_series (fit_all_windows over this rank's windows) with host buffers"

        def e2e_call():
            if mine:
                ctx.check(L.sg_fit_window_range_series(ctx.handle, *ptrs, len(I), TAU, DELTA, ctypes.byref(settings),
                                                       base, mine[0], len(mine), ctypes.byref(nw), recs,
                                                       _capi._d(trajs)))
    else:
        call_name = "sg_fit_all_windows_series (fit_all_windows) with host buffers"

        def e2e_call():
            ctx.check(L.sg_fit_all_windows_series(ctx.handle, *ptrs, len(I), TAU, DELTA, ctypes.byref(settings), base,
                                                  n_win, ctypes.byref(nw), recs, _capi._d(trajs), ctypes.byref(mean),
                                                  ctypes.byref(failed)))

    e2e_call()  # warm (allocations, module load)
    barrier(world)
    c0 = ctx.copy_bytes
    t = time.perf_counter()
    for _ in range(args.steps):
        e2e_call()
    e2e_s = allreduce_max((time.perf_counter() - t) / args.steps, world)
    c1 = ctx.copy_bytes
    e2e_value = total_evals / e2e_s
    h2d = allreduce_sum((c1[0] - c0[0]) / args.steps, world)
    d2h = allreduce_sum((c1[1] - c0[1]) / args.steps, world)

    # spot check of the e2e result against the device-timed plan (same engine)
    res = plan.results() if plan else []
    ok = all(recs[k].objective == res[k][2] for k in range(len(mine)))

    cpu, parity = None, None
    if rank == 0 and not args.no_cpu:
        v, kind, cores, sample, cpu_res = cpu_reference_sample(I, R, D, budget_s=args.cpu_budget, windows=mine,
                                                               base=base, max_iters=iters)
        v1, sample1 = cpu_reference_one_thread(I, R, D, budget_s=args.cpu1_budget, w=mine[len(mine) // 2], base=base,
                                               max_iters=iters)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
               "sample": f"windows {sample['windows']} of the sweep, {PARTICLES} particles x {sample['iterations']} "
                         f"iterations each ({sample['evals']} evals, {sample['seconds']:.1f} s)",
               "value_1thread": v1, "sample_1thread": sample1}
        parity = parity_vs_reference(cpu_res, res, slot)
    gpu_launches = int(allreduce_sum(launches, world))
    if rank == 0:
        strong = args.split == "windows"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C2 window sweep: {n_win} windows x {PARTICLES} particles x {iters} iterations "
                                   f"(tau={TAU}, delta={DELTA}, {SPEC}, stage2)"
                                   + (f", its windows split over {world} GPU(s)" if strong else
                                      f", one sweep restart per GPU (C4-style, x{world})"),
                       "windows": n_win, "particles": PARTICLES, "iterations": iters, "objective": SPEC,
                       "series": "tests/golden/poland_like.csv (synthetic Poland-like, 450 days)",
                       "split": args.split,
                       "parallelism": (f"windows / {world} GPUs (contiguous shares, no collective)" if strong else
                                       f"restarts x{world} (one per GPU, no collective)"),
                       "windows_rank0": len(mine),
                       "l2": "working set (MT19937-64 engines 312 x 8 B per particle = 1.4 GB) exceeds L2"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "call": call_name, "steps": args.steps,
                    "bytes": "every host<->device copy the call made (series, windows, plan descriptors in; "
                             "histories, best states, re-integrated trajectories, R2 out), counted by the engine",
                    "matches_device_run": ok},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": nominal_peak / 1e12, "unit": "TFLOP/s",
                         "frac": achieved * 1e12 / nominal_peak, "traffic": traffic,
                         "kernel": "pso_step_kernel<IRD,MXSE,24> (fused move+integrate+score+argmin)",
                         "peak_note": "SMs x 64 FP64 lanes x max SM clock, no FMA (FMA is banned for bit parity, "
                                      "so this is half the FMA-counted TFLOPS figure); neither MEASURED_PEAKS.json "
                                      "nor B200_PROFILING.md has an FP64 number",
                         "ops_per_eval_floor": ops_per_eval(TAU + 1),
                         "ramp_substeps_per_eval": ramp_substeps / evals_per_step if evals_per_step else None,
                         "ops_per_eval": ops_step / evals_per_step if evals_per_step else None,
                         "fp64_ops_per_eval_executed": fp64_exec,  # ncu SASS counts (profile), incl. PSO move/setup
                         "frac_floor": achieved_floor * 1e12 / nominal_peak,
                         "ops_note": "algorithmic FP64 ops (SURVEY.md §8d: 14/substep + 5/ramp substep + 12/scored "
                                     "day), DADD/DMUL without FMA for bit parity (the kernel scores MXSE with 2 of "
                                     "the credited 4 ops per compartment-day, exactly, DESIGN.md §3)",
                         "peak_probe": fp64_probe / 1e12, "frac_probe": achieved * 1e12 / fp64_probe,
                         "peak_probe_note": "FP64 DADD/DMUL issue rate measured on this GPU by sg_probe_fp64_rate "
                                            f"({fp64_probe / nominal_peak:.3f} of nominal)",
                         "kernel_ms_per_launch": kernel_ms, "launches_per_step": step_launches,
                         "step_kernels_ms": steps_kernel_ms,
                         "seed_ms": statistics.mean(seed_ms) if seed_ms else None, "profile": prof,
                         "rank": 0},
            "parity": parity,
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": gpu_launches,
        }
        print(json.dumps(line), flush=True)
    if plan:
        plan.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--iters", type=int, default=ITERS, help="PSO iterations per swarm (default: the config's 1000)")
    ap.add_argument("--split", choices=["windows", "restarts"], default="windows",
                    help="N>1: split the sweep's windows over the GPUs (strong scaling, default) or run one "
                         "restart of the whole sweep per GPU (weak, C4-style)")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--cpu1-budget", type=float, default=3.0)
    ap.add_argument("--ref-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return bench_reference(args)
    return bench_ours(args)


if __name__ == "__main__":
    sys.exit(main())
