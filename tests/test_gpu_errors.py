"""Error behaviour through the C-ABI, message for message with the reference
(integrate_euler's guards model.cpp:78-80, PsoConfig/SearchBounds::validate
pso.cpp:16-34, the window objective's dimension check calibration.cpp:141-143,
forecast_extension calibration.cpp:298-303): the engine reports the
reference's exception class and text, never a CPU fallback."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

INTEGRATE_MSG = "integrate_euler needs n_days >= 1, substeps >= 1 and a positive population"


def _series(poland, a=40, n=21):
    I, R, D = (poland[k][a:a + n] for k in ("I", "R", "D"))
    N = poland["N"]
    return I, R, D, [N - I[0] - R[0] - D[0], I[0], R[0], D[0]], N


@pytest.mark.parametrize("n_days,substeps,population", [(0, 24, 1e6), (21, 0, 1e6), (21, 24, 0.0),
                                                        (21, 24, -5.0), (21, 24, float("nan"))])
def test_window_guards_match_integrate_euler(ctx, poland, n_days, substeps, population):
    import paper_2204_12346_b200 as eng
    I, R, D, init, _ = _series(poland)
    with pytest.raises(eng.errors.Error) as exc:
        eng.Window(ctx, I[:max(n_days, 1)][:n_days] if n_days else I[:0], R[:n_days], D[:n_days], init, population,
                   "ird-mxse", substeps=substeps)
    assert str(exc.value) == INTEGRATE_MSG


@pytest.mark.parametrize("field,value,msg", [
    ("n_particles", 0, "pso: n_particles and max_iters must be positive"),
    ("max_iters", 0, "pso: n_particles and max_iters must be positive"),
    ("inertia", float("inf"), "pso: coefficients must be finite"),
    ("social", float("nan"), "pso: coefficients must be finite"),
])
def test_swarm_config_errors_are_per_swarm_with_reference_text(ctx, poland, field, value, msg):
    import paper_2204_12346_b200 as eng
    from paper_2204_12346_b200 import _capi
    I, R, D, init, N = _series(poland)
    win = eng.Window(ctx, I, R, D, init, N, "d-mse")
    good = dict(window=win, lower=[0] * 6, upper=[2, 2, 13, 13, 1, 0.1], n_particles=40, max_iters=3, seed=1)
    out = ctx.fit_swarms([good, dict(good, **{field: value}), good])
    assert out[0][0] == 0 and out[2][0] == 0
    assert out[1][0] == 1
    assert _capi.lib().sg_last_error(ctx.handle).decode() == msg
    np.testing.assert_array_equal(out[0][3], out[2][3])  # the failing swarm does not disturb its neighbours


def test_bound_errors_name_the_dimension(ctx, poland):
    import paper_2204_12346_b200 as eng
    from paper_2204_12346_b200 import _capi
    I, R, D, init, N = _series(poland)
    win = eng.Window(ctx, I, R, D, init, N, "ird-mse")
    for d, (lo, hi) in enumerate([(1.0, 0.5), (0.0, float("inf")), (float("nan"), 1.0)]):
        lower, upper = [0.0] * 6, [2, 2, 13, 13, 1, 0.1]
        lower[d + 2], upper[d + 2] = lo, hi
        out = ctx.fit_swarms([dict(window=win, lower=lower, upper=upper, n_particles=8, max_iters=2, seed=3)])
        assert out[0][0] == 1
        assert _capi.lib().sg_last_error(ctx.handle).decode() == f"pso: bound {d + 2} is invalid"


def test_all_infeasible_swarm_reports_status_4(ctx, poland):
    """Every particle blows up (pso.cpp:137-139): AllInfeasibleError."""
    import paper_2204_12346_b200 as eng
    I, R, D, init, N = _series(poland)
    win = eng.Window(ctx, I, R, D, init, N, "ird-mxse")
    out = ctx.fit_swarms([dict(window=win, lower=[1e300] * 2 + [0, 0] + [1e300] * 2,
                               upper=[1e301] * 2 + [13, 13] + [1e301] * 2, n_particles=64, max_iters=4, seed=2)])
    assert out[0][0] == 4
    assert np.all(np.isinf(out[0][3]))


def test_window_objective_rejects_wrong_dimension(ctx, poland):
    import paper_2204_12346_b200 as eng
    I, R, D, init, N = _series(poland)
    win = eng.Window(ctx, I, R, D, init, N, "ird-mxse")
    with pytest.raises(eng.errors.Error) as exc:
        win.eval_costs(np.zeros((4, 5)))
    assert str(exc.value) == "window objective expects 6-dim positions"


def test_band_calls_reject_bad_arguments_without_side_effects(ctx, poland):
    """The C5 band calls validate before any device work: a bound outside
    its box names its dimension like the PSO config check (pso.cpp:16-34),
    a negative horizon and windows of two contexts are refused, and the
    context keeps working afterwards."""
    import paper_2204_12346_b200 as eng
    from paper_2204_12346_b200.errors import Error
    I, R, D, init, N = _series(poland, 0, 36)
    win = eng.Window(ctx, I, R, D, init, N, "ird-mxse")
    lo, hi = [0.0] * 6, [2.0, 2.0, 28.0, 28.0, 1.0, 0.1]
    bad_hi = list(hi)
    bad_hi[3] = -1.0
    with pytest.raises(Error, match="bound 3 is invalid"):
        ctx.forecast_ensemble_bands_batch([win, win], lo, bad_hi, [1, 2], 1000, 21)
    with pytest.raises(Error, match="bound 3 is invalid"):
        win.forecast_ensemble_bands(lo, bad_hi, 1, 1000, 21)
    with pytest.raises(Error, match="horizon"):
        ctx.forecast_ensemble_bands_batch([win], lo, hi, [1], 1000, -1)
    other = eng.Context(0)
    try:
        w2 = eng.Window(other, I, R, D, init, N, "ird-mxse")
        with pytest.raises(Error, match="share one context"):
            ctx.forecast_ensemble_bands_batch([win, w2], lo, hi, [1, 2], 1000, 21)
        del w2
    finally:
        other.close()
    bands, counts = ctx.forecast_ensemble_bands_batch([win], lo, hi, [7], 1000, 21)
    b1, c1, _ = win.forecast_ensemble_bands(lo, hi, 7, 1000, 21)
    assert counts[0].tolist() == c1.tolist() and np.array_equal(bands[0], b1, equal_nan=True)
