"""Calibration-level parity: the reference's fit_window / fit_all_windows /
stability_study / forecast_extension (calibration.cpp:157-436) against the
Python mirror of its module (paper_2204_12346_b200.sirdfit -> C++ host layer
-> C-ABI -> CUDA), on golden results of the unmodified reference
(tests/golden/calibration.json, oracle/gen_golden.py).

Mirrors test_calibration.cpp:166-492 and test_smoke.py:35-86.  Bar: bit
identical params, objectives, R^2, trajectories, forecasts, bands; the same
exception type and message for failures.
"""
import json
import math

import numpy as np
import pytest

from helpers import assert_bitwise

pytestmark = pytest.mark.gpu


def unhex(v):
    return np.array([float.fromhex(x) for x in v])


@pytest.fixture(scope="module")
def golden():
    from conftest import GOLDEN
    return json.loads((GOLDEN / "calibration.json").read_text())


@pytest.fixture(scope="module")
def sirdfit(ctx):
    from paper_2204_12346_b200 import sirdfit as m
    m.set_context(ctx)
    return m


def series(sf, c):
    return sf.EpiSeries(unhex(c["I"]).tolist(), unhex(c["R"]).tolist(), unhex(c["D"]).tolist(), [0.0] * len(c["I"]))


BOUNDS = {1: "stage1", 2: "stage2"}


def test_fit_window_matches_reference(golden, sirdfit):
    from paper_2204_12346_b200 import errors
    by_status = {2: errors.SchemeError, 3: errors.InsufficientPopulationError, 4: errors.AllInfeasibleError}
    for c in golden["fit_window"]:
        data = series(sirdfit, c)
        w = sirdfit.Window(0, c["start"], c["length"])
        kw = dict(objective=c["spec"], bounds=BOUNDS[c["stage"]], particles=c["n"], iters=c["iters"], seed=c["seed"])
        if c["status"]:
            with pytest.raises(by_status[c["status"]]) as exc:
                sirdfit.fit_window(data, w, c["N"], **kw)
            assert str(exc.value) == c["error"], c["name"]
            continue
        fit = sirdfit.fit_window(data, w, c["N"], **kw)
        assert fit.ok
        assert_bitwise(fit.params.as_array(), unhex(c["params"]), c["name"] + " params")
        assert fit.objective == float.fromhex(c["objective"]), c["name"]
        r2 = float.fromhex(c["r2"])
        assert (math.isnan(r2) and math.isnan(fit.r2_d)) or fit.r2_d == r2, c["name"]
        traj = np.array([[s.S, s.I, s.R, s.D] for s in fit.trajectory.states])
        assert_bitwise(traj.ravel(), unhex(c["trajectory"]), c["name"] + " trajectory")
        if c["forecast"] is not None:
            fc = sirdfit.forecast_extension(fit, c["horizon"])
            assert fc.junction_day == c["start"] + c["length"] - 1
            got = np.array([[s.S, s.I, s.R, s.D] for s in fc.trajectory.states])
            assert_bitwise(got.ravel(), unhex(c["forecast"]), c["name"] + " forecast")
            # the junction state is shared bit for bit (test_calibration.cpp:193-196)
            assert fc.trajectory.states[0].D == fit.trajectory.states[-1].D


def test_appendix_a_values(golden, sirdfit):
    """fit_window 64 x 10, seed 1, ird-mxse."""
    c = next(c for c in golden["fit_window"] if c["name"] == "appendixA")
    fit = sirdfit.fit_window(series(sirdfit, c), sirdfit.Window(0, 0, 21), 1e6, particles=64, iters=10, seed=1)
    assert fit.objective == 0.24655820930891381
    assert fit.params.beta1 == 0.43878783065997495 and fit.params.mu == 0.02785236525356902
    assert fit.r2_d == 0.80104735188667031
    assert sirdfit.forecast_extension(fit, 21).trajectory.states[21].D == 53473.272220453611


def test_fit_all_windows_matches_reference(golden, sirdfit):
    for c in golden["fit_all_windows"]:
        res = sirdfit.fit_all_windows(series(sirdfit, c), c["N"], tau=c["tau"], delta=c["delta"], objective=c["spec"],
                                      bounds=BOUNDS[c["stage"]], particles=c["n"], iters=c["iters"], seed=c["seed"])
        assert len(res.fits) == c["n_windows"], c["name"]
        assert [int(f.ok) for f in res.fits] == c["ok"], c["name"]
        assert res.failed_count == c["failed"]
        params, obj, r2 = unhex(c["params"]).reshape(-1, 6), unhex(c["objective"]), unhex(c["r2"])
        for k, f in enumerate(res.fits):
            assert f.window.index == k and f.window.start == k * c["delta"] and f.window.length == c["tau"] + 1
            if not f.ok:
                assert f.failure.startswith("population smaller than I+R+D"), f.failure
                continue
            assert_bitwise(f.params.as_array(), params[k], f"{c['name']} window {k}")
            assert f.objective == obj[k]
            assert (math.isnan(r2[k]) and math.isnan(f.r2_d)) or f.r2_d == r2[k]
        mean = float.fromhex(c["mean_r2"])
        assert (math.isnan(mean) and math.isnan(res.mean_r2_d)) or res.mean_r2_d == mean


def test_stability_study_matches_reference(golden, sirdfit):
    for c in golden["stability"]:
        st = sirdfit.stability_study(series(sirdfit, c), sirdfit.Window(0, c["start"], c["length"]), c["N"],
                                     c["reps"], c["horizon"], objective=c["spec"], bounds=BOUNDS[c["stage"]],
                                     particles=c["n"], iters=c["iters"], seed=c["seed"])
        assert st.failed == c["failed"], c["name"]
        assert [int(f.ok) for f in st.fits] == c["ok"]
        params, obj = unhex(c["params"]).reshape(-1, 6), unhex(c["objective"])
        for k, f in enumerate(st.fits):
            if f.ok:
                assert_bitwise(f.params.as_array(), params[k], f"{c['name']} rep {k}")
                assert f.objective == obj[k]
        bands = unhex(c["day_bands"])
        off = 0
        cnt = 0
        for blk in (st.beta, st.r0, st.infectious, st.recovered, st.deaths):
            n = blk.days()
            for row in (blk.median, blk.p50_lo, blk.p50_hi, blk.p90_lo, blk.p90_hi, blk.p95_lo, blk.p95_hi):
                assert_bitwise(np.array(row), bands[off:off + n], c["name"] + " bands")
                off += n
            assert blk.count == c["day_counts"][cnt:cnt + n]
            cnt += n
        sc = unhex(c["scalar_bands"])
        for k, b in enumerate((st.gamma, st.mu)):
            got = np.array([b.median, b.p50_lo, b.p50_hi, b.p90_lo, b.p90_hi, b.p95_lo, b.p95_hi])
            assert_bitwise(got, sc[7 * k:7 * k + 7], c["name"] + " scalar bands")
            assert b.count == c["scalar_counts"][k]


def test_python_surface_like_reference_smoke(sirdfit):
    """test_smoke.py:35-86 on the mirror module."""
    params = sirdfit.SirdParams(beta1=0.6, beta2=0.9, t1=15.0, t2=30.0, gamma=0.09, mu=0.012)
    init = sirdfit.SirdState(S=1e6 - 100.0, I=100.0)
    tr = sirdfit.integrate(params, init, 1e6, 60)
    assert tr.finite and tr.days() == 60 and tr.states[0].I == 100.0
    for s in tr.states:
        assert abs(s.total() - 1e6) <= 1e-9 * 1e6
    assert sirdfit.beta_at(params, 0.0) == 0.6 and sirdfit.beta_at(params, 35.0) == 0.9
    windows = sirdfit.make_windows(450, tau=35, delta=3)
    assert len(windows) == 139 and windows[-1].start == 414
    data = sirdfit.EpiSeries([s.I for s in tr.states], [s.R for s in tr.states], [s.D for s in tr.states],
                             [0.0] * 60)
    fit = sirdfit.fit_window(data, sirdfit.Window(index=0, start=0, length=21), 1e6, objective="ird-mse",
                             particles=400, iters=80, seed=2)
    assert fit.ok and fit.r2_d > 0.99 and 0.0 <= fit.params.gamma <= 1.0
    fc = sirdfit.forecast_extension(fit, 10)
    assert fc.junction_day == 20 and fc.trajectory.days() == 11
    assert fc.trajectory.states[0].D == fit.trajectory.states[20].D
    res = sirdfit.fit_all_windows(data, 10.0, tau=20, delta=10, particles=30, iters=5, seed=4)
    assert res.failed_count == len(res.fits) and all(not f.ok for f in res.fits) and math.isnan(res.mean_r2_d)


def test_cpp_objective_boundary_matches_serial(ctx, golden_costs_case):
    """make_window_objective's BatchObjective (boundary 1) through the C++ layer
    equals objective_value(integrate_euler(...)) slot by slot
    (test_calibration.cpp:139-164)."""
    I, R, D, init, N, pos, want = golden_costs_case
    import paper_2204_12346_b200 as eng
    win = eng.Window(ctx, I, R, D, init, N, "ird-mxse")
    assert_bitwise(win.eval_costs(pos), want, "boundary fixture")
    assert win.eval_costs(pos)[0] == 0.0  # the generator itself


@pytest.fixture(scope="module")
def golden_costs_case():
    from conftest import GOLDEN
    g = np.load(GOLDEN / "costs.npz")
    I, R, D = g["boundary_fixture/obs"]
    return (I, R, D, g["boundary_fixture/init"], float(g["boundary_fixture/N"][0]),
            g["boundary_fixture/special/positions"][:3], g["boundary_fixture/special/ird-mxse"][:3])


def test_device_r2_matches_reference_formula_and_flat_series(sirdfit):
    """R^2(D) is computed on the device with the reference's sequential sums
    (objectives.cpp:122-144); a constant observed series gives NaN instead of
    ConstantObservedError (calibration.cpp:183-185)."""
    import numpy as np
    from conftest import GOLDEN
    a = np.genfromtxt(GOLDEN / "poland_like.csv", delimiter=",", names=True)
    I, R, D = list(a["infectious"]), list(a["recovered_cum"]), list(a["deaths_cum"])
    D_flat = D[:]
    for k in range(200, 221):
        D_flat[k] = 1000.0  # its mean is exact, so ss_tot == 0 exactly
    for deaths, want_nan in ((D, False), (D_flat, True)):
        data = sirdfit.EpiSeries(infectious=I, recovered_cum=R, deaths_cum=deaths, new_cases=[0.0] * len(I))
        fit = sirdfit.fit_window(data, sirdfit.Window(0, 200, 21), 38e6, "ird-mse", particles=120, iters=15, seed=4)
        assert fit.ok
        if want_nan:
            assert np.isnan(fit.r2_d)
        else:
            obs = np.array(deaths[200:221])
            pred = np.array([s.D for s in fit.trajectory.states])
            mean = 0.0
            for y in obs:
                mean += float(y)
            mean /= len(obs)
            ss_res = ss_tot = 0.0
            for y, p in zip(obs, pred):
                e, c = float(y) - float(p), float(y) - mean
                ss_res += e * e
                ss_tot += c * c
            assert fit.r2_d == 1.0 - ss_res / ss_tot
