"""Parity at the BASELINE configurations themselves (VERDICT r01 "weak 1"):
the engine against the unmodified reference (oracle/_ref, the reference's own
C++ compiled from /root/reference, run on all host cores) at the exact sizes
the benchmark quotes, not just at test sizes.

  C1  window 0, tau = 20, 256 particles x 500 iterations, seed
      mix_seed(2204, 0) — the persistent cluster kernel
  C2  whole windows of the bench sweep, 4096 particles x 1000 iterations, the
      bench's seeds (calibration.cpp:199) — the flat step kernel as the bench
      runs it (139-window plan, four launch lanes)
  C3  one swarm of 2^20 particles (8,192 CTAs: the 256-group two-level
      global-best fold, kernels.cuh finish_step) x 3 iterations

Every history, best position and best cost must be bit-identical
(pso.cpp:77-143, calibration.cpp:157-216)."""
import os

import numpy as np
import pytest

from helpers import assert_bitwise

pytestmark = pytest.mark.gpu

BASE_SEED = 2204
THREADS = os.cpu_count() or 1


def _mix(base, index):
    m = (1 << 64) - 1
    z = (base + 0x9E3779B97F4A7C15 * (index + 1)) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def _slice(poland, start, tau):
    sl = slice(start, start + tau + 1)
    I, R, D = (np.ascontiguousarray(poland[k][sl]) for k in ("I", "R", "D"))
    N = poland["N"]
    return I, R, D, [N - I[0] - R[0] - D[0], I[0], R[0], D[0]], N


def _stage2(tau):
    return [0.0] * 6, [2.0, 2.0, float(tau - 7), float(tau - 7), 1.0, 0.1]


def _assert_same(got, want, what):
    status, best, cost, hist = got
    rc, best_r, cost_r, hist_r = want
    assert status == rc, what
    assert_bitwise(hist, hist_r, f"{what} history")
    if rc == 0:
        assert_bitwise(best, best_r, f"{what} best position")
        assert cost == cost_r, what


def test_c1_exact_config(ctx, reference, poland):
    import paper_2204_12346_b200 as eng
    I, R, D, init, N = _slice(poland, 0, 20)
    lo, hi = _stage2(20)
    seed = _mix(BASE_SEED, 0)
    w = eng.Window(ctx, I, R, D, init, N, "ird-mxse")
    got = ctx.fit_swarms([dict(window=w, lower=lo, upper=hi, n_particles=256, max_iters=500, seed=seed)])[0]
    want = reference.fit_swarm("ird-mxse", I, R, D, init, N, lo, hi, 256, 500, seed=seed, n_threads=THREADS)
    _assert_same(got, want, "C1 256 x 500")


def test_c2_whole_windows_in_the_bench_plan(ctx, reference, poland):
    """The bench's own plan shape (all 139 windows, 4096 x 1000, four lanes):
    windows at the start, in the middle and at the end of the sweep."""
    import paper_2204_12346_b200 as eng
    tau, delta = 35, 3
    n_win = 1 + (len(poland["D"]) - 1 - tau) // delta
    lo, hi = _stage2(tau)
    wins, swarms = [], []
    for k in range(n_win):
        I, R, D, init, N = _slice(poland, k * delta, tau)
        wins.append(eng.Window(ctx, I, R, D, init, N, "ird-mxse"))
        swarms.append(dict(window=wins[-1], lower=lo, upper=hi, n_particles=4096, max_iters=1000,
                           seed=_mix(BASE_SEED, k)))
    plan = eng.Plan(ctx, swarms)
    plan.run()
    res = plan.results()
    plan.close()
    for k in (0, 69, n_win - 1):
        I, R, D, init, N = _slice(poland, k * delta, tau)
        want = reference.fit_swarm("ird-mxse", I, R, D, init, N, lo, hi, 4096, 1000, seed=_mix(BASE_SEED, k),
                                   n_threads=THREADS)
        _assert_same(res[k], want, f"C2 window {k}")


def test_c3_million_particle_swarm(ctx, reference, poland):
    """2^20 particles: 8,192 step CTAs, 256 fold groups of 32 CTAs, the
    last group folding the group minima — the C3 path at its real size."""
    import paper_2204_12346_b200 as eng
    I, R, D, init, N = _slice(poland, 0, 35)
    lo, hi = _stage2(35)
    n, iters, seed = 1 << 20, 3, _mix(BASE_SEED, 0)
    w = eng.Window(ctx, I, R, D, init, N, "ird-mxse")
    got = ctx.fit_swarms([dict(window=w, lower=lo, upper=hi, n_particles=n, max_iters=iters, seed=seed)])[0]
    want = reference.fit_swarm("ird-mxse", I, R, D, init, N, lo, hi, n, iters, seed=seed, n_threads=THREADS)
    _assert_same(got, want, "C3 2^20 x 3")
