"""Plan-level parity: the launch machinery around the step kernels.

Every swarm of a mixed plan (all 8 objective specs, window lengths on both
sides of the shared-memory time-table limit, substep counts 24/7/1,
different particle counts, iteration counts, coefficients, repair on/off)
must follow the C restatement's optimize() bit for bit — which exercises the
CTA task table, the lane partition, the generic-substep kernels, CTAs whose
swarm has finished early, and the cluster kernel at every cluster size.
Mirrors test_pso.cpp:78-131 (reproducibility, first iteration, best-so-far
monotone) at the plan level.
"""
import numpy as np
import pytest

from helpers import assert_bitwise

pytestmark = pytest.mark.gpu

SPECS = [f"{f}-{m}" for f in ("d", "ird") for m in ("mxse", "mse", "mae", "mape")]


def _window(eng, ctx, poland, start, n_days, spec, substeps=24):
    I, R, D = (poland[k][start:start + n_days] for k in ("I", "R", "D"))
    N = poland["N"]
    init = [N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
    return eng.Window(ctx, I, R, D, init, N, spec, substeps=substeps), (I, R, D, init, N)


def _check(port, swarms, data, out):
    for k, (s, (I, R, D, init, N, substeps)) in enumerate(zip(swarms, data)):
        rc, best, cost, hist = port.fit_swarm((s["window"].family, s["window"].metric), I, R, D, init, N, s["lower"],
                                              s["upper"], s["n_particles"], s["max_iters"],
                                              inertia=s.get("inertia", 0.5), cognitive=s.get("cognitive", 0.5),
                                              social=s.get("social", 0.5), seed=s["seed"],
                                              repair=s.get("repair", True), substeps=substeps)
        status, gbest, gcost, ghist = out[k]
        assert status == rc, k
        assert_bitwise(ghist, hist, f"swarm {k} history")
        if rc == 0:
            assert_bitwise(gbest, best, f"swarm {k} best")
            assert gcost == cost
        assert np.all(np.diff(ghist) <= 0) or not np.all(np.isfinite(ghist))


def test_mixed_plan_matches_oracle(ctx, port, poland):
    import paper_2204_12346_b200 as eng
    rng = np.random.default_rng(2204)
    cases = [  # (start, n_days, spec, substeps, particles, iters)
        (0, 8, "ird-mxse", 24, 300, 17), (30, 36, "d-mse", 24, 1500, 9), (90, 100, "ird-mae", 24, 257, 6),
        (120, 21, "ird-mape", 7, 640, 12), (200, 36, "d-mxse", 1, 129, 25), (260, 15, "d-mae", 24, 33, 40),
        (300, 36, "ird-mse", 24, 2048, 5), (400, 30, "d-mape", 24, 700, 11),
        (150, 230, "ird-mxse", 24, 300, 4),  # past the 201-day time table: the generic kernels
    ]
    swarms, data, keep = [], [], []
    for k, (a, n, spec, sub, n_p, iters) in enumerate(cases):
        win, (I, R, D, init, N) = _window(eng, ctx, poland, a, n, spec, sub)
        keep.append(win)
        tau = n - 1
        hi = [2.0, 2.0, float(tau), float(tau), 1.0, 0.1] if k % 2 else [0.9, 0.9, 0.8 * tau, 0.8 * tau, 0.3, 0.05]
        swarms.append(dict(window=win, lower=[0.0] * 6, upper=hi, n_particles=n_p, max_iters=iters,
                           inertia=float(rng.uniform(0.2, 0.9)), cognitive=float(rng.uniform(0.2, 1.5)),
                           social=float(rng.uniform(0.2, 1.5)), seed=int(rng.integers(1 << 62)),
                           repair=k != 3))
        data.append((I, R, D, init, N, sub))
    out = ctx.fit_swarms(swarms)
    _check(port, swarms, data, out)


@pytest.mark.parametrize("n_particles", [1, 31, 33, 128, 129, 257, 600, 1024])
def test_cluster_kernel_every_cluster_size(ctx, port, poland, n_particles):
    """Plans of <= 1024 particles run as one thread-block cluster per swarm
    (cluster size ceil(n/128)); two swarms per plan when they still fit."""
    import paper_2204_12346_b200 as eng
    win, (I, R, D, init, N) = _window(eng, ctx, poland, 150, 21, "ird-mxse")
    swarms, data = [], []
    for j in range(2 if 2 * n_particles <= 1024 else 1):
        swarms.append(dict(window=win, lower=[0.0] * 6, upper=[2, 2, 13, 13, 1, 0.1], n_particles=n_particles,
                           max_iters=30, seed=77 + j))
        data.append((I, R, D, init, N, 24))
    plan = eng.Plan(ctx, swarms)
    assert plan.step_launches == 1  # one persistent launch
    plan.run()
    _check(port, swarms, data, plan.results())


@pytest.mark.parametrize("n_days,substeps,spec", [(118, 48, "ird-mse"), (117, 48, "d-mae"), (217, 24, "ird-mxse"),
                                                   (230, 24, "ird-mape")])
def test_cluster_kernel_shared_memory_edges(ctx, port, poland, n_days, substeps, spec):
    """Windows whose staged image (~47 KB) plus the cluster kernel's static
    shared memory (2.6 KB) passes the 48 KB a launch gets without opting in:
    the launcher opts in above 40 KB (tools/fuzz_long.py batch 81 of seed
    base 4000000 — an ird-mse window of 118 days at 48 substeps — once
    failed with cudaErrorInvalidValue)."""
    import paper_2204_12346_b200 as eng
    win, (I, R, D, init, N) = _window(eng, ctx, poland, 100, n_days, spec, substeps)
    swarms = [dict(window=win, lower=[0.0] * 6, upper=[2, 2, n_days - 8, n_days - 8, 1, 0.1], n_particles=178,
                   max_iters=4, seed=5)]
    plan = eng.Plan(ctx, swarms)
    assert plan.step_launches == 1  # the persistent cluster kernel
    plan.run()
    _check(port, swarms, [(I, R, D, init, N, substeps)], plan.results())


def test_plan_reruns_are_identical(ctx, poland):
    import paper_2204_12346_b200 as eng
    wins = [_window(eng, ctx, poland, 3 * w, 36, "ird-mxse")[0] for w in range(12)]
    swarms = [dict(window=w, lower=[0.0] * 6, upper=[2, 2, 28, 28, 1, 0.1], n_particles=1100, max_iters=20, seed=k)
              for k, w in enumerate(wins)]
    plan = eng.Plan(ctx, swarms)
    assert plan.step_launches > 1  # flat per-iteration kernels
    runs = []
    for _ in range(4):  # the third run captures the CUDA graph, the fourth replays it
        plan.run()
        runs.append(plan.results())
    c = ctx.fit_swarms(swarms)
    for k, z in enumerate(c):
        assert z[0] == 0
        for r in runs:
            assert r[k][0] == 0
            assert_bitwise(r[k][3], z[3], "rerun history")
            assert_bitwise(r[k][1], z[1], "rerun best")


def test_two_level_fold_for_large_swarms(ctx, port, poland):
    """Swarms of more than 32 CTAs (4096 particles) fold their warp minima
    per group of 32 CTAs, then across groups; 10,000 particles = 79 CTAs =
    3 groups (the last ragged), next to a 4,097-particle swarm (2 groups)."""
    import paper_2204_12346_b200 as eng
    w1, (I1, R1, D1, init1, N) = _window(eng, ctx, poland, 210, 36, "ird-mxse")
    w2, (I2, R2, D2, init2, _) = _window(eng, ctx, poland, 330, 21, "d-mae")
    swarms = [dict(window=w1, lower=[0.0] * 6, upper=[2, 2, 28, 28, 1, 0.1], n_particles=10_000, max_iters=8, seed=5),
              dict(window=w2, lower=[0.0] * 6, upper=[2, 2, 13, 13, 1, 0.1], n_particles=4_097, max_iters=12,
                   seed=6)]
    data = [(I1, R1, D1, init1, N, 24), (I2, R2, D2, init2, N, 24)]
    plan = eng.Plan(ctx, swarms)
    plan.run()
    _check(port, swarms, data, plan.results())
    plan.run()  # group counters are reset by their last warp: a rerun must match again
    _check(port, swarms, data, plan.results())


def test_sharded_stability_study_matches_single_process(tmp_path):
    """tools/shard_c4.py under torchrun, two ranks sharing the one GPU
    (gloo): the merged shards equal the single-process run bit for bit."""
    import socket
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), str(root / "tools" / "shard_c4.py"), "--windows", "12",
           "--restarts", "3", "--iters", "15", "--backend", "gloo", "--check"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1]
    import json
    d = json.loads(line)
    assert d["ranks"] == 2 and d["units"] == 36 and d["identical_to_single_process"] is True


def test_oversized_calls_split_into_sequential_plans_identically(tmp_path):
    """sg_fit_swarms splits a call whose device state exceeds the memory
    budget into sequential plans; forcing a tiny budget (SG_PLAN_BUDGET_BYTES)
    must give the same results as one plan."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    script = tmp_path / "split.py"
    script.write_text(f"""
import sys, hashlib
sys.path.insert(0, {str(root)!r})
import numpy as np
import paper_2204_12346_b200 as eng
a = np.genfromtxt({str(root / 'tests' / 'golden' / 'poland_like.csv')!r}, delimiter=",", names=True)
ctx = eng.Context(0)
N = 38e6
swarms, wins = [], []
for k in range(12):
    s = 20 * k
    I, R, D = a["infectious"][s:s + 30], a["recovered_cum"][s:s + 30], a["deaths_cum"][s:s + 30]
    w = eng.Window(ctx, I, R, D, [N - I[0] - R[0] - D[0], I[0], R[0], D[0]], N, "ird-mxse")
    wins.append(w)
    swarms.append(dict(window=w, lower=[0] * 6, upper=[2, 2, 22, 22, 1, 0.1], n_particles=1500, max_iters=8, seed=k))
out = ctx.fit_swarms(swarms)
h = hashlib.sha1(b"".join(o[3].tobytes() + o[1].tobytes() for o in out)).hexdigest()
print(h, sum(o[0] for o in out))
""")
    plain = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300)
    env = dict(os.environ, SG_PLAN_BUDGET_BYTES=str(4 * 1500 * 331 * 8))  # ~4 swarms per plan
    split = subprocess.run([sys.executable, str(script)], capture_output=True, text=True, timeout=300, env=env)
    assert plain.returncode == 0 and split.returncode == 0, plain.stderr[-800:] + split.stderr[-800:]
    assert plain.stdout.split() == split.stdout.split() and plain.stdout.split()[1] == "0"


def test_no_device_memory_growth_across_calls(ctx, poland):
    """Repeated plans, band pipelines, single-window bands and reused plans
    on one context leave the device's free memory where it was after a
    warm-up (stream-ordered buffers are returned to the pool each call)."""
    import gc

    import torch

    import paper_2204_12346_b200 as eng

    def one_round():
        wins = [_window(eng, ctx, poland, 3 * w, 36, "ird-mxse")[0] for w in range(4)]
        box = [2, 2, 28, 28, 1, 0.1]
        ctx.fit_swarms([dict(window=w, lower=[0] * 6, upper=box, n_particles=300, max_iters=5, seed=k)
                        for k, w in enumerate(wins)])
        ctx.forecast_ensemble_bands_batch(wins, [0] * 6, box, [1, 2, 3, 4], 20000, 21)
        wins[0].forecast_ensemble_bands([0] * 6, box, 1, 5000, 21)
        plan = eng.Plan(ctx, [dict(window=wins[0], lower=[0] * 6, upper=box, n_particles=4096, max_iters=3, seed=1)])
        for _ in range(3):
            plan.run()
        plan.close()
        del wins
        gc.collect()

    def free():
        torch.cuda.synchronize()
        return torch.cuda.mem_get_info()[0]

    for _ in range(3):
        one_round()
    before = free()
    for _ in range(20):
        one_round()
    assert abs(before - free()) <= 2 << 20, (before, free())
