"""Seeded fuzz of the whole path against the C restatement: random series
(zeros, flat stretches, huge and tiny counts), random populations (integer,
fractional, tiny, huge), all 8 objective specs, random boxes (negative lower
bounds, inverted time boxes, zero-width dimensions), random PSO coefficients,
24 and odd substep counts.  Every case must follow the oracle's optimize()
bit for bit — this is where the exact-division fast paths and the regime
prefixes meet inputs nobody chose on purpose."""
import numpy as np
import pytest

from helpers import assert_bitwise

pytestmark = pytest.mark.gpu

SPECS = [f"{f}-{m}" for f in ("d", "ird") for m in ("mxse", "mse", "mae", "mape")]


def _case(rng):
    n_days = int(rng.integers(2, 60)) if rng.random() < 0.85 else int(rng.integers(60, 130))
    kind = rng.integers(0, 4)
    base = 10.0 ** rng.uniform(-2, 7)
    if kind == 0:      # smooth growth
        t = np.arange(n_days)
        D = base * np.exp(rng.uniform(0, 0.1) * t)
    elif kind == 1:    # noisy with zeros
        D = np.maximum(0.0, base * rng.uniform(-0.5, 1.5, n_days)).cumsum()
    elif kind == 2:    # flat
        D = np.full(n_days, base)
    else:              # integer counts
        D = np.floor(rng.uniform(0, base, n_days)).cumsum()
    I = np.abs(D * rng.uniform(0.5, 3.0) + rng.normal(0, base * 0.1, n_days))
    R = np.sort(np.abs(D * rng.uniform(1, 10)))
    if rng.random() < 0.2:
        I[: n_days // 2] = 0.0
    pop_kind = rng.integers(0, 4)
    N = [38e6, float(rng.integers(10 ** 5, 10 ** 9)) + 0.5, 1e3 * rng.uniform(1, 9), 1e12][pop_kind]
    N = max(N, float(I[0] + R[0] + D[0]) * 1.01 + 1.0)
    init = [N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
    tau = n_days - 1
    lo = [0.0, 0.0, 0.0, 0.0, 0.0, 0.0]
    hi = [float(rng.uniform(0.1, 5)), float(rng.uniform(0.1, 5)), float(tau), float(tau),
          float(rng.uniform(0.01, 2)), float(rng.uniform(0.001, 0.3))]
    if rng.random() < 0.3:
        lo[0] = -float(rng.uniform(0, 0.5))     # negative beta allowed by the box
    if rng.random() < 0.2:
        lo[4] = hi[4] = float(rng.uniform(0, 1))  # zero-width dimension
    if rng.random() < 0.2:
        lo[2], hi[2] = float(tau) * 0.6, float(tau)  # t1 late, t2 anywhere: repairs and t1 > t2
    sub = int(rng.choice([24, 24, 24, 7, 1, 48]))
    spec = SPECS[int(rng.integers(0, 8))]
    coeffs = dict(inertia=float(rng.uniform(0, 1.2)), cognitive=float(rng.uniform(0, 2)),
                  social=float(rng.uniform(0, 2)))
    return dict(I=I, R=R, D=D, init=init, N=N, lo=lo, hi=hi, sub=sub, spec=spec, coeffs=coeffs,
                n=int(rng.integers(1, 200)), iters=int(rng.integers(1, 12)), seed=int(rng.integers(1 << 62)),
                repair=bool(rng.random() < 0.8))


@pytest.mark.parametrize("batch", range(4))
def test_fuzz_plans_match_oracle(ctx, port, batch):
    import paper_2204_12346_b200 as eng
    rng = np.random.default_rng(20240 + batch)
    cases = [_case(rng) for _ in range(16)]
    wins, swarms = [], []
    for c in cases:
        w = eng.Window(ctx, c["I"], c["R"], c["D"], c["init"], c["N"], c["spec"], substeps=c["sub"])
        wins.append(w)
        swarms.append(dict(window=w, lower=c["lo"], upper=c["hi"], n_particles=c["n"], max_iters=c["iters"],
                           seed=c["seed"], repair=c["repair"], **c["coeffs"]))
    # two shapes of the same work: one plan (flat kernels: more small swarms
    # with the ballast than one wave of persistent clusters) and one swarm
    # per call (cluster kernel)
    ballast = [dict(swarms[0], n_particles=1, max_iters=1, seed=j) for j in range(300)]
    flat = ctx.fit_swarms(swarms + ballast)[:len(swarms)]
    for k, c in enumerate(cases):
        rc, best, cost, hist = port.fit_swarm(c["spec"], c["I"], c["R"], c["D"], c["init"], c["N"], c["lo"], c["hi"],
                                              c["n"], c["iters"], seed=c["seed"], repair=c["repair"],
                                              substeps=c["sub"], **c["coeffs"])
        single = ctx.fit_swarms([swarms[k]])[0]
        for name, got in (("flat", flat[k]), ("cluster", single)):
            assert got[0] == rc, (batch, k, name)
            assert_bitwise(got[3], hist, f"batch {batch} case {k} {name} {c['spec']} sub {c['sub']}")
            if rc == 0:
                assert_bitwise(got[1], best, f"batch {batch} case {k} {name} best")


def test_fuzz_costs_match_oracle(ctx, port):
    import paper_2204_12346_b200 as eng
    rng = np.random.default_rng(777)
    for _ in range(30):
        c = _case(rng)
        w = eng.Window(ctx, c["I"], c["R"], c["D"], c["init"], c["N"], c["spec"], substeps=c["sub"])
        pos = rng.uniform(np.array(c["lo"]) - 0.1, np.array(c["hi"]) * 1.5 + 0.1, (257, 6))
        pos[::7, 2], pos[::7, 3] = pos[::7, 3], pos[::7, 2]      # some t1 > t2
        pos[::11, 0] = 0.0
        pos[::13, 1] = -0.0
        pos[5, 2] = np.nan
        pos[6, 3] = np.inf
        assert_bitwise(w.eval_costs(pos), port.eval_costs(c["spec"], c["I"], c["R"], c["D"], c["init"], c["N"], pos,
                                                          substeps=c["sub"]), c["spec"])


@pytest.mark.parametrize("edge", ["subnormal_range", "inf_obs", "nan_obs", "flat_zero", "plain"])
def test_mxse_largest_residual_shortcut_edges(ctx, port, poland, edge):
    """MXSE keeps max |obs - pred| and scales/squares once (exact for finite
    positive scales); windows whose scale is +inf (subnormal range) or 0
    (infinite observation) take the per-day path — both must equal the
    reference's per-day max of squared scaled residuals."""
    import paper_2204_12346_b200 as eng
    a = 70
    I, R, D = (poland[k][a:a + 30].copy() for k in ("I", "R", "D"))
    if edge == "subnormal_range":
        I[:] = 0.0
        I[3] = 1e-310             # I's range subnormal: scale = 1/range = inf
    elif edge == "inf_obs":
        D[11] = np.inf            # range inf: scale 0
    elif edge == "nan_obs":
        R[5] = np.nan
    elif edge == "flat_zero":
        I[:] = 0.0
    N = poland["N"]
    init = [N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
    rng = np.random.default_rng(9)
    pos = rng.uniform([0, 0, 0, 0, 0, 0], [2, 2, 28, 28, 1, 0.1], (300, 6))
    for spec in ("ird-mxse", "d-mxse", "ird-mse"):
        w = eng.Window(ctx, I, R, D, init, N, spec)
        assert_bitwise(w.eval_costs(pos), port.eval_costs(spec, I, R, D, init, N, pos), f"{edge} {spec}")


@pytest.mark.parametrize("edge", ["I0", "R0", "D0", "I0_mid"])
def test_nan_first_observation(ctx, port, reference, poland, edge):
    """A NaN first observation (init supplied separately, as
    make_window_objective allows): the reference seeds MXSE with
    std::max(0.0, NaN) = 0 and picks the IRD scale with std::minmax_element
    over a NaN-led series (engine.cu:339).  Checked against the
    reference itself, all specs."""
    import paper_2204_12346_b200 as eng
    a = 120
    I, R, D = (poland[k][a:a + 36].copy() for k in ("I", "R", "D"))
    N = poland["N"]
    init = [N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
    {"I0": I, "R0": R, "D0": D, "I0_mid": I}[edge][0] = np.nan
    if edge == "I0_mid":
        D[17] = np.nan
    rng = np.random.default_rng(4)
    pos = rng.uniform([0, 0, 0, 0, 0, 0], [2, 2, 28, 28, 1, 0.1], (300, 6))
    for spec in SPECS:
        w = eng.Window(ctx, I, R, D, init, N, spec)
        assert_bitwise(w.eval_costs(pos), reference.eval_costs(spec, I, R, D, init, N, pos), f"{edge} {spec}")


def test_long_window_one_substep_flat_plan(ctx, port):
    """substeps = 1 and a ~3,000-day window keep the substep-time table
    (SUB = -1 kernels, bulk-copied staging) and 72 KB of observations: the
    CTA task's byte counts no longer fit 16 bits (engine.cu:764).
    A flat plan (more swarms than one wave of clusters) must follow optimize()."""
    import paper_2204_12346_b200 as eng
    n_days = 3001
    N = 5e6
    st, fin = port.integrate([0.12, 0.08, 700.0, 1900.0, 0.1, 0.003], [N - 50, 50, 0, 0], N, n_days, 1)
    assert fin
    I, R, D = st[:, 1].copy(), st[:, 2].copy(), st[:, 3].copy()
    rng = np.random.default_rng(5)
    D *= rng.uniform(0.98, 1.02, n_days)
    init = list(st[0])
    hi = [0.3, 0.3, float(n_days - 1), float(n_days - 1), 0.3, 0.01]
    for spec in ("ird-mxse", "d-mape"):
        w = eng.Window(ctx, I, R, D, init, N, spec, substeps=1)
        swarms = [dict(window=w, lower=[0.0] * 6, upper=hi, n_particles=1100, max_iters=3, seed=31)]
        swarms += [dict(window=w, lower=[0.0] * 6, upper=hi, n_particles=1, max_iters=1, seed=j) for j in range(300)]
        got = ctx.fit_swarms(swarms)
        for k in (0, 1, 299):
            s = swarms[k]
            rc, best, cost, hist = port.fit_swarm(spec, I, R, D, init, N, s["lower"], s["upper"], s["n_particles"],
                                                  s["max_iters"], seed=s["seed"], substeps=1)
            assert got[k][0] == rc
            assert_bitwise(got[k][3], hist, f"{spec} swarm {k} history")
            if rc == 0:
                assert_bitwise(got[k][1], best, f"{spec} swarm {k} best")


@pytest.mark.parametrize("n_days", [230, 301, 560])
def test_long_windows_all_kernel_paths(ctx, port, n_days):
    """Windows past the 5-CTA shared-memory table (202-534 days stage a
    larger t_k table at lower occupancy) and past the table altogether (560
    days: the compile-time-24 kernels that compute t_k, SUB = -24), through
    the flat plan (with ballast swarms), the cluster kernel and boundary 1."""
    import paper_2204_12346_b200 as eng
    N = 2e7
    st, fin = port.integrate([0.21, 0.12, 90.0, 400.0, 0.1, 0.004], [N - 300, 300, 0, 0], N, n_days)
    assert fin
    I, R, D = st[:, 1].copy(), st[:, 2].copy(), st[:, 3].copy()
    D *= np.random.default_rng(n_days).uniform(0.99, 1.01, n_days)
    init = list(st[0])
    hi = [0.5, 0.5, float(n_days - 8), float(n_days - 8), 0.5, 0.02]
    for spec in ("ird-mxse", "d-mape"):
        w = eng.Window(ctx, I, R, D, init, N, spec)
        pos = np.random.default_rng(2).uniform(0, 1, (257, 6)) * np.array(hi)
        assert_bitwise(w.eval_costs(pos), port.eval_costs(spec, I, R, D, init, N, pos), f"{n_days} {spec} costs")
        main = dict(window=w, lower=[0.0] * 6, upper=hi, n_particles=700, max_iters=4, seed=17)
        flat = ctx.fit_swarms([main] + [dict(main, n_particles=1, max_iters=1, seed=j) for j in range(300)])[0]
        single = ctx.fit_swarms([main])[0]
        rc, best, cost, hist = port.fit_swarm(spec, I, R, D, init, N, main["lower"], main["upper"], 700, 4, seed=17)
        for name, got in (("flat", flat), ("cluster", single)):
            assert got[0] == rc
            assert_bitwise(got[3], hist, f"{n_days} {spec} {name} history")
            if rc == 0:
                assert_bitwise(got[1], best, f"{n_days} {spec} {name} best")
