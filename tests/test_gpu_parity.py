"""CUDA path vs the reference, through the C-ABI (include/sirdgpu.h).

Bar: bit-identical doubles (NaN == NaN).  The golden costs/fits/forecasts in
tests/golden/ were produced by the unmodified reference (oracle/gen_golden.py);
the on-the-fly comparisons use the C restatement (oracle/), itself pinned to
the same goldens by tests/test_oracle.py.  Mirrors the reference's own
pins: test_calibration.cpp:139-164 (batch objective == serial
objective_value), test_pso.cpp:78-93 (bitwise reproducibility), 133-216
(first iteration, ties, all-infeasible), test_model.cpp:50-58, 116-148.
"""
import json

import numpy as np
import pytest

from helpers import assert_bitwise

pytestmark = pytest.mark.gpu

SPECS = [f"{f}-{m}" for f in ("d", "ird") for m in ("mxse", "mse", "mae", "mape")]


@pytest.fixture(scope="module")
def golden_costs():
    from conftest import GOLDEN
    return dict(np.load(GOLDEN / "costs.npz"))


def _cases(g):
    return sorted({k.split("/")[0] for k in g})


def test_costs_match_reference_goldens(ctx, golden_costs):
    import paper_2204_12346_b200 as eng
    g = golden_costs
    checked = 0
    for case in _cases(g):
        I, R, D = g[f"{case}/obs"]
        init, N = g[f"{case}/init"], float(g[f"{case}/N"][0])
        sets = sorted({k.split("/")[1] for k in g if k.startswith(case + "/") and k.count("/") == 2})
        for spec in SPECS:
            win = eng.Window(ctx, I, R, D, init, N, spec)
            for s in sets:
                got = win.eval_costs(g[f"{case}/{s}/positions"])
                assert_bitwise(got, g[f"{case}/{s}/{spec}"], f"{case}/{s}/{spec}")
                checked += got.size
    assert checked > 5000


@pytest.mark.parametrize("spec", SPECS)
def test_costs_match_oracle_random_poland_windows(ctx, port, poland, spec):
    import paper_2204_12346_b200 as eng
    rng = np.random.default_rng(hash(spec) & 0xFFFF)
    for w in (0, 17, 77, 138):
        a = 3 * w
        I, R, D = poland["I"][a:a + 36], poland["R"][a:a + 36], poland["D"][a:a + 36]
        N = poland["N"]
        init = [N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
        win = eng.Window(ctx, I, R, D, init, N, spec)
        for hi in ([2, 2, 28, 28, 1, 0.1], [10, 10, 35, 35, 10, 10]):
            pos = rng.random((700, 6)) * np.array(hi)
            assert_bitwise(win.eval_costs(pos), port.eval_costs(spec, I, R, D, init, N, pos), f"w{w} {spec}")


def test_costs_non_default_substeps_and_populations(ctx, port, poland):
    import paper_2204_12346_b200 as eng
    rng = np.random.default_rng(5)
    I, R, D = poland["I"][30:51], poland["R"][30:51], poland["D"][30:51]
    for N, substeps in ((38e6, 7), (38e6 + 0.3, 24), (1.0 / 3.0 * 1e8, 24), (38e6, 1), (38e6, 50)):
        init = [N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
        pos = rng.random((300, 6)) * np.array([2, 2, 20, 20, 1, 0.1])
        for spec in ("ird-mxse", "d-mape"):
            win = eng.Window(ctx, I, R, D, init, N, spec, substeps=substeps)
            assert_bitwise(win.eval_costs(pos), port.eval_costs(spec, I, R, D, init, N, pos, substeps=substeps),
                           f"N={N} S={substeps} {spec}")


def test_single_day_window_and_empty_batch(ctx, port):
    import paper_2204_12346_b200 as eng
    I, R, D = np.array([5.0]), np.array([1.0]), np.array([0.5])
    init = [100 - 6.5, 5.0, 1.0, 0.5]
    pos = np.array([[0.5, 0.5, 0, 0, 0.1, 0.01], [9, 9, 0, 0, 9, 9]])
    for spec in SPECS:
        win = eng.Window(ctx, I, R, D, init, 100.0, spec)
        assert_bitwise(win.eval_costs(pos), port.eval_costs(spec, I, R, D, init, 100.0, pos), spec)
        assert win.eval_costs(np.zeros((0, 6))).size == 0


def test_non_finite_initial_state_costs_infinity(ctx):
    import paper_2204_12346_b200 as eng
    I = R = D = np.ones(5)
    win = eng.Window(ctx, I, R, D, [np.inf, 1, 1, 1], 10.0, "ird-mse")
    assert np.all(np.isposinf(win.eval_costs(np.full((3, 6), 0.1))))


def test_rejects_non_six_dim_positions(ctx):
    import paper_2204_12346_b200 as eng
    from paper_2204_12346_b200 import _capi
    win = eng.Window(ctx, np.ones(5), np.ones(5), np.ones(5), [7, 1, 1, 1], 10.0, "ird-mse")
    costs = np.empty(2)
    rc = _capi.lib().sg_eval_costs(win.handle, _capi._d(np.zeros(10)), 2, 5, _capi._d(costs))
    assert rc == 1
    with pytest.raises(eng.errors.Error):
        eng.Window(ctx, np.ones(5), np.ones(5), np.ones(5), [7, 1, 1, 1], 0.0, "ird-mse")


def test_integrate_batch_matches_reference_trajectories(ctx, port):
    from conftest import GOLDEN
    g = np.load(GOLDEN / "forecast.npz")
    pos, init, N = g["positions"], g["init"], float(g["N"][0])
    states, fin = ctx.integrate_batch(pos, init, N, 36)
    assert_bitwise(states, g["window"], "window trajectories")
    assert np.array_equal(fin, g["window_finite"])
    # day 0 is the initial state bit for bit (test_model.cpp:50-58)
    assert_bitwise(states[:, 0, :], np.broadcast_to(init, (len(pos), 4)), "day 0")


def test_forecast_batch_matches_reference(ctx):
    from conftest import GOLDEN
    g = np.load(GOLDEN / "forecast.npz")
    ok = g["window_finite"]
    junction = g["window"][ok, -1, :]
    states, fin = ctx.forecast_batch(g["positions"][ok], junction, float(g["N"][0]), 21)
    assert_bitwise(states[fin], g["forecast"][ok][fin], "forecast")
    assert np.array_equal(fin, g["forecast_finite"][ok])


def test_integrate_random_parameters_match_oracle(ctx, port):
    rng = np.random.default_rng(17)
    N = 1e6
    init = [N - 300, 200, 80, 20]
    pos = rng.random((400, 6)) * np.array([10, 10, 35, 35, 10, 10])
    states, fin = ctx.integrate_batch(pos, init, N, 36)
    for k in range(0, 400, 7):
        want, wf = port.integrate(pos[k], init, N, 36)
        assert_bitwise(states[k], want, f"trajectory {k}")
        assert fin[k] == wf


def _unhex(v):
    return np.array([float.fromhex(x) for x in v])


@pytest.fixture(scope="module")
def golden_fits():
    from conftest import GOLDEN
    return json.loads((GOLDEN / "fits.json").read_text())


@pytest.mark.parametrize("mode", ["persistent", "flat"])
def test_swarms_match_reference_goldens(ctx, golden_fits, mode):
    """All golden swarms in ONE sg_fit_swarms call (mixed specs, sizes, windows).
    Small plans run one persistent cluster per swarm (pso_swarm_kernel); 300
    one-particle ballast swarms push the same swarms onto the flat
    per-iteration kernels (pso_step_kernel)."""
    import paper_2204_12346_b200 as eng
    wins, descs = [], []
    for c in golden_fits:
        win = eng.Window(ctx, _unhex(c["I"]), _unhex(c["R"]), _unhex(c["D"]), _unhex(c["init"]), c["N"], c["spec"])
        wins.append(win)
        descs.append(dict(window=win, lower=c["lower"], upper=c["upper"], n_particles=c["n"], max_iters=c["iters"],
                          inertia=c["w"], cognitive=c["c1"], social=c["c2"], seed=c["seed"]))
    if mode == "flat":
        # more small swarms than one wave of persistent clusters: flat kernels
        descs += [dict(descs[1], n_particles=1, max_iters=1, seed=12345 + j) for j in range(300)]
    out = ctx.fit_swarms(descs)
    for c, (status, best, cost, hist) in zip(golden_fits, out):
        assert status == c["status"], c["name"]
        assert_bitwise(hist, _unhex(c["history"]), c["name"] + " history")
        if status == 0:
            assert_bitwise(best, _unhex(c["best"]), c["name"] + " best")
            assert cost == float.fromhex(c["best_cost"])


def test_swarm_matches_oracle_and_is_reproducible(ctx, port, poland):
    import paper_2204_12346_b200 as eng
    a = 60
    I, R, D = poland["I"][a:a + 36], poland["R"][a:a + 36], poland["D"][a:a + 36]
    N = poland["N"]
    init = [N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
    lo, hi = [0] * 6, [2, 2, 28, 28, 1, 0.1]
    win = eng.Window(ctx, I, R, D, init, N, "ird-mxse")
    # 700 particles -> 6 CTAs incl. a ragged one; 60 iterations -> 714 draws, the engine twists three times
    desc = dict(window=win, lower=lo, upper=hi, n_particles=700, max_iters=60, seed=99)
    (s1, b1, c1, h1), (s2, b2, c2, h2) = ctx.fit_swarms([desc, desc])
    rc, bo, co, ho = port.fit_swarm("ird-mxse", I, R, D, init, N, lo, hi, 700, 60, seed=99)
    assert s1 == s2 == rc == 0
    assert_bitwise(h1, ho, "history")
    assert_bitwise(b1, bo, "best")
    assert_bitwise(h2, h1, "reproducible")
    assert np.all(np.diff(h1) <= 0)  # best-so-far never increases (test_pso.cpp:95-107)


def test_invalid_swarm_config_is_reported_per_swarm(ctx, poland):
    import paper_2204_12346_b200 as eng
    I, R, D = poland["I"][:21], poland["R"][:21], poland["D"][:21]
    N = poland["N"]
    win = eng.Window(ctx, I, R, D, [N - I[0] - R[0] - D[0], I[0], R[0], D[0]], N, "d-mse")
    good = dict(window=win, lower=[0] * 6, upper=[2, 2, 13, 13, 1, 0.1], n_particles=40, max_iters=3, seed=1)
    bad = dict(good, lower=[0, 0, 0, 5, 0, 0], upper=[2, 2, 13, 4, 1, 0.1])
    out = ctx.fit_swarms([good, bad, dict(good, inertia=float("nan"))])
    assert out[0][0] == 0 and out[1][0] == 1 and out[2][0] == 1


def test_forecast_ensemble_matches_oracle(ctx, port, poland):
    import paper_2204_12346_b200 as eng
    a = 414
    I, R, D = poland["I"][a:a + 36], poland["R"][a:a + 36], poland["D"][a:a + 36]
    N = poland["N"]
    init = [N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
    win = eng.Window(ctx, I, R, D, init, N, "ird-mxse")
    lo, hi = np.zeros(6), np.array([2, 2, 28, 28, 1, 0.1])
    costs, params, deaths = win.forecast_ensemble(lo, hi, seed=2204, n=300, horizon=21)
    for k in range(0, 300, 11):
        u = port.uniform01(port.mix_seed(2204, k), 6)
        x = lo + u * (hi - lo)
        if x[2] > x[3]:
            x[2], x[3] = x[3], x[2]
        assert_bitwise(params[k], x, f"sample {k}")
        c = port.eval_costs("ird-mxse", I, R, D, init, N, x[None, :])
        assert_bitwise(costs[k:k + 1], c, f"cost {k}")
        st, fin = port.integrate(x, init, N, 36)
        if fin:
            fc, ff = port.forecast(x, st[-1], N, 21)
            if ff:
                assert_bitwise(deaths[k], fc[:, 3], f"forecast {k}")
                continue
        assert np.all(np.isnan(deaths[k]))


def test_forecast_ensemble_bands_match_reference(ctx):
    """Device quantile bands of forecast ensembles == the reference's
    build_quantile_bands (calibration.cpp:337-361) over the same samples,
    blown-up samples dropped (tests/golden/ensemble_bands.json)."""
    import paper_2204_12346_b200 as eng
    from conftest import GOLDEN
    for c in json.loads((GOLDEN / "ensemble_bands.json").read_text()):
        I, R, D = _unhex(c["I"]), _unhex(c["R"]), _unhex(c["D"])
        win = eng.Window(ctx, I, R, D, _unhex(c["init"]), c["N"], "ird-mxse")
        bands, counts, _ = win.forecast_ensemble_bands(_unhex(c["lower"]), _unhex(c["upper"]), c["seed"], c["n"],
                                                       c["horizon"])
        assert counts.tolist() == c["counts"], c["name"]
        assert_bitwise(bands.ravel(), _unhex(c["bands"]), c["name"])


def _host_bands(deaths):
    """build_quantile_bands (calibration.cpp:337-361) on the host: per day,
    the finite values sorted ascending, then quantile_sorted (324-335)."""
    ps = [0.5, 0.25, 0.75, 0.05, 0.95, 0.025, 0.975]
    n_days = deaths.shape[1]
    bands = np.full((7, n_days), np.nan)
    counts = []
    for d in range(n_days):
        col = np.sort(deaths[:, d][np.isfinite(deaths[:, d])])
        k = col.size
        counts.append(k)
        for q, p in enumerate(ps):
            if k == 0:
                continue
            h = float(k - 1) * p
            lo = int(h)
            if lo + 1 >= k:
                bands[q, d] = col[k - 1]
            else:
                a, b = float(col[lo]), float(col[lo + 1])
                bands[q, d] = a + (h - lo) * (b - a)
    return bands, counts


@pytest.mark.parametrize("case", ["wide", "narrow", "identical", "tiny", "blowups", "long_horizon"])
def test_ensemble_band_selection_equals_full_sort(ctx, poland, case):
    """The device bands select 14 order statistics per day through key bins
    instead of sorting; they must equal sorting the same ensemble's deaths
    (sg_forecast_ensemble) on the host, for wide and narrow spreads, all
    samples identical (one bin holds everything), tiny ensembles and
    ensembles with many non-finite forecasts."""
    import paper_2204_12346_b200 as eng
    a = 120
    I, R, D = poland["I"][a:a + 36], poland["R"][a:a + 36], poland["D"][a:a + 36]
    N = poland["N"]
    init = [N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
    win = eng.Window(ctx, I, R, D, init, N, "ird-mxse")
    lo, hi, n = [0.0] * 6, [2.0, 2.0, 28.0, 28.0, 1.0, 0.1], 300_000
    if case == "narrow":
        lo, hi = [0.2, 0.1, 10.0, 20.0, 0.1, 0.002], [0.2000001, 0.1000001, 10.0, 20.0, 0.1, 0.002]
    elif case == "identical":
        lo = hi = [0.2, 0.1, 10.0, 20.0, 0.1, 0.002]
        n = 50_000
    elif case == "tiny":
        n = 3
    elif case == "blowups":
        hi = [1e150, 1e150, 28.0, 28.0, 1e150, 1e150]
        n = 100_000
    horizon = 40 if case == "long_horizon" else 21  # past 31 days: the key-range pass instead of the fused one
    bands, counts, _ = win.forecast_ensemble_bands(lo, hi, seed=99, n=n, horizon=horizon)
    _, _, deaths = win.forecast_ensemble(lo, hi, seed=99, n=n, horizon=horizon, want_costs=False, want_params=False)
    want, want_counts = _host_bands(deaths)
    assert counts.tolist() == want_counts
    assert_bitwise(bands.ravel(), want.ravel(), case)


def test_ensemble_bands_batch_equals_per_window_calls(ctx, poland):
    """The pipelined many-window call gives each window exactly its
    single-window bands."""
    import paper_2204_12346_b200 as eng
    N = poland["N"]
    wins = []
    for a in (0, 33, 66, 99, 132):
        I, R, D = poland["I"][a:a + 36], poland["R"][a:a + 36], poland["D"][a:a + 36]
        wins.append(eng.Window(ctx, I, R, D, [N - I[0] - R[0] - D[0], I[0], R[0], D[0]], N, "ird-mxse"))
    lo, hi, seeds = [0.0] * 6, [2.0, 2.0, 28.0, 28.0, 1.0, 0.1], [11, 12, 13, 14, 15]
    bands, counts = ctx.forecast_ensemble_bands_batch(wins, lo, hi, seeds, 50_000, 21)
    for k, w in enumerate(wins):
        b1, c1, _ = w.forecast_ensemble_bands(lo, hi, seeds[k], 50_000, 21)
        assert counts[k].tolist() == c1.tolist()
        assert_bitwise(bands[k].ravel(), b1.ravel(), f"window {k}")


def test_ensemble_bands_batch_prediction_hits_and_misses(ctx, poland):
    """The pipelined call predicts each window's histogram bins from the
    window two back (the same slot); windows whose deaths scale jumps
    (populations 1e3x apart) miss and take the histogram pass, repeated
    windows hit.  Both paths give each window its single-window bands."""
    import paper_2204_12346_b200 as eng
    N = poland["N"]
    wins = []
    for a, scale in ((0, 1.0), (3, 1.0), (6, 1e3), (9, 1e3), (12, 1.0), (12, 1.0), (12, 1.0), (15, 1e-3)):
        I, R, D = (poland[c][a:a + 36] * scale for c in "IRD")
        Ns = N * scale
        wins.append(eng.Window(ctx, I, R, D, [Ns - I[0] - R[0] - D[0], I[0], R[0], D[0]], Ns, "ird-mxse"))
    lo, hi = [0.0] * 6, [2.0, 2.0, 28.0, 28.0, 1.0, 0.1]
    seeds = [21, 22, 23, 24, 25, 26, 27, 28]
    f0, p0, _ = ctx.band_stats
    bands, counts = ctx.forecast_ensemble_bands_batch(wins, lo, hi, seeds, 40_000, 21)
    f1, p1, _ = ctx.band_stats
    assert f1 - f0 > 0 and p1 - p0 > 0, (f1 - f0, p1 - p0)
    for k, w in enumerate(wins):
        b1, c1, _ = w.forecast_ensemble_bands(lo, hi, seeds[k], 40_000, 21)
        assert counts[k].tolist() == c1.tolist()
        assert_bitwise(bands[k].ravel(), b1.ravel(), f"window {k}")


def _random_band_batch(eng, ctx, poland, rng):
    """A batch of random ensemble windows (lengths, populations, boxes, a
    horizon on either side of the fused-range limit of 31 days, sample
    counts that are no multiple of the CTA) for the pipelined band call."""
    N0 = poland["N"]
    horizon = int(rng.choice([0, 1, 7, 21, 31, 32, 40]))
    n = int(rng.choice([1, 2, 127, 129, 1000, 4099, 20000]))
    wins, seeds = [], []
    for _ in range(int(rng.integers(1, 6))):
        a, days = int(rng.integers(0, 300)), int(rng.integers(2, 60))
        scale = float(10.0 ** rng.uniform(-3, 3))
        I, R, D = (poland[c][a:a + days] * scale for c in "IRD")
        N = N0 * scale
        wins.append(eng.Window(ctx, I, R, D, [N - I[0] - R[0] - D[0], I[0], R[0], D[0]], N,
                               str(rng.choice(["ird-mxse", "d-mse", "ird-mape"]))))
        seeds.append(int(rng.integers(1 << 62)))
    tmax = float(rng.uniform(0.0, 80.0))
    hi = [float(rng.uniform(0.0, 3.0)), float(rng.uniform(0.0, 3.0)), tmax, tmax,
          float(rng.uniform(0.0, 2.0)), float(rng.uniform(0.0, 0.5))]
    if rng.random() < 0.2:
        hi = [1e150, 1e150, tmax, tmax, 1e150, 1e150]  # many blow-ups
    return wins, [0.0] * 6, hi, seeds, n, horizon


@pytest.mark.parametrize("seed", range(12))
def test_ensemble_bands_batch_random_against_host_sort(ctx, poland, seed):
    """Random pipelined band batches (the fused range and predicted-bin
    histogram, misses and hits, the non-fused path past 31 days, blow-ups,
    tiny and ragged ensembles) against sorting each window's forecast
    deaths on the host, bit for bit."""
    import paper_2204_12346_b200 as eng
    rng = np.random.default_rng(7000 + seed)
    wins, lo, hi, seeds, n, horizon = _random_band_batch(eng, ctx, poland, rng)
    bands, counts = ctx.forecast_ensemble_bands_batch(wins, lo, hi, seeds, n, horizon)
    for k, w in enumerate(wins):
        _, _, deaths = w.forecast_ensemble(lo, hi, seed=seeds[k], n=n, horizon=horizon, want_costs=False,
                                           want_params=False)
        want, want_counts = _host_bands(deaths)
        assert counts[k].tolist() == want_counts, (seed, k)
        assert_bitwise(bands[k].ravel(), want.ravel(), f"seed {seed} window {k}")


def test_ensemble_bands_batch_with_a_non_finite_window(ctx, poland):
    """A window whose initial state is not finite forecasts NaN for every
    sample (calibration.cpp:301-303): its bands are NaN with zero counts,
    and it does not disturb the pipeline around it — the samples it draws
    for the window two ahead, the next windows' predicted bins."""
    import paper_2204_12346_b200 as eng
    N = poland["N"]
    wins = []
    for k, a in enumerate((0, 3, 6, 9, 12)):
        I, R, D = poland["I"][a:a + 36], poland["R"][a:a + 36], poland["D"][a:a + 36]
        init = [N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
        if k == 1:
            init[1] = float("nan")
        wins.append(eng.Window(ctx, I, R, D, init, N, "ird-mxse"))
    lo, hi, seeds = [0.0] * 6, [2.0, 2.0, 28.0, 28.0, 1.0, 0.1], [31, 32, 33, 34, 35]
    bands, counts = ctx.forecast_ensemble_bands_batch(wins, lo, hi, seeds, 30_000, 21)
    assert counts[1].tolist() == [0] * 22 and np.all(np.isnan(bands[1]))
    for k in (0, 2, 3, 4):
        b1, c1, _ = wins[k].forecast_ensemble_bands(lo, hi, seeds[k], 30_000, 21)
        assert counts[k].tolist() == c1.tolist() and c1[0] == 30_000
        assert_bitwise(bands[k].ravel(), b1.ravel(), f"window {k}")


def test_ensemble_ramp_telemetry_is_exact(ctx, poland):
    """The band path's ramp-substep count (the roofline's ramp credit) is
    exact: switch times pinned by the box (t1 = 0, t2 = 10 days) ramp on
    10 x 24 substeps in every sample; t1 = t2 never ramps."""
    import paper_2204_12346_b200 as eng
    N = poland["N"]
    I, R, D = poland["I"][:36], poland["R"][:36], poland["D"][:36]
    win = eng.Window(ctx, I, R, D, [N - I[0] - R[0] - D[0], I[0], R[0], D[0]], N, "ird-mxse")
    n = 5000
    for t1, t2, want in ((0.0, 10.0, 240), (7.0, 7.0, 0)):
        lo, hi = [0.0, 0.0, t1, t2, 0.0, 0.0], [2.0, 2.0, t1, t2, 1.0, 0.1]
        r0 = ctx.band_stats[2]
        ctx.forecast_ensemble_bands_batch([win, win], lo, hi, [1, 2], n, 21)
        assert ctx.band_stats[2] - r0 == 2 * n * want, (t1, t2)


@pytest.mark.parametrize("case", ["cluster_outliers", "two_clusters", "spiky_key_range", "nan_mix", "constant",
                                  "tiny_counts"])
def test_quantile_bands_selection_paths(ctx, reference, case):
    """sg_quantile_bands (build_quantile_bands, calibration.cpp:337-361) on
    synthetic columns that drive every path of the selection: a bin too full
    for one CTA's shared memory (a dense cluster plus far outliers, so the
    bins are wide and one holds > 8,192 values: the finer histogram levels),
    two clusters, a key range collapsing to single keys, NaN/inf mixed in,
    constant columns and columns with 0-3 finite values.  Against the
    reference's own build_quantile_bands (oracle/_ref), bit for bit."""
    import ctypes
    rng = np.random.default_rng(31)
    n, n_days = 60_000, 5
    cols = np.empty((n_days, n))
    for d in range(n_days):
        if case == "cluster_outliers":
            c = 1000.0 + rng.random(n) * 1e-3 * (d + 1)
            c[rng.choice(n, 40, replace=False)] = 10.0 ** rng.uniform(6, 12, 40)
        elif case == "two_clusters":
            c = np.where(rng.random(n) < 0.3, 5.0 + rng.random(n) * 1e-6, 7e5 + rng.random(n))
        elif case == "spiky_key_range":
            c = 2.0 + np.floor(rng.random(n) * 37) * np.finfo(float).eps * 2  # 37 distinct neighbouring doubles
        elif case == "nan_mix":
            c = rng.normal(1e4, 50.0, n)
            c[rng.random(n) < 0.2] = np.nan
            c[rng.random(n) < 0.01] = np.inf
            c[rng.random(n) < 0.01] = -np.inf
        elif case == "constant":
            c = np.full(n, 3.25)
        else:
            c = np.full(n, np.nan)
            c[:d % 4] = rng.random(d % 4)
        cols[d] = c
    bands, counts = ctx.quantile_bands(cols)
    want = np.zeros((7, n_days))
    want_counts = np.zeros(n_days, dtype=np.uint64)
    samples = np.ascontiguousarray(cols.T)  # the shim takes sample-major values
    dp = ctypes.POINTER(ctypes.c_double)
    rc = reference.lib.ref_quantile_bands(samples.ctypes.data_as(dp), n, n_days, want.ctypes.data_as(dp),
                                          want_counts.ctypes.data_as(ctypes.POINTER(ctypes.c_size_t)))
    assert rc == 0
    assert counts.tolist() == want_counts.tolist()
    assert_bitwise(bands.ravel(), want.ravel(), case)
