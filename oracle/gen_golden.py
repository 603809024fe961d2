"""Generate the golden fixtures under tests/golden/ from the REFERENCE build.

TEST INFRASTRUCTURE.  Run in the build container (needs /root/reference to
build oracle/_ref/libsirdref.so):

    python oracle/gen_golden.py

Every output value below is produced by the unmodified reference library
(oracle/_ref, kind "reference"); the inputs are generated here from fixed
seeds.  The fixtures are committed so the C restatement (oracle/) and the
CUDA path can be checked on machines without /root/reference.

Fixtures
  poland_like.csv   synthetic Poland-like series, 450 days,
                    cleaned by the reference's build_epi_series + smooth7.
  kat.json          mix_seed / mt19937_64 / uniform01 known-answer values.
  costs.npz         per-particle costs, 8 objective specs x several windows x
                    particle sets (stage-1/2 uniform, near-optimal, unrepaired
                    t1>t2, blow-ups, flat and zero windows, MAPE zeros).
  fits.json         optimize() results (best position, cost, full history).
  forecast.npz      forecast_extension trajectories.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import oracle_py as op  # noqa: E402

GOLDEN = ROOT / "tests" / "golden"

# N = 38e6, 450 days, init S=N-200, I=200, gamma 0.1,
# mu 0.0027, six chained segments (len, beta1, beta2, t1, t2).
POLAND_N = 38_000_000.0
POLAND_SEGMENTS = [(30, 0.30, 0.115, 5, 20), (150, 0.115, 0.118, 0, 0), (60, 0.118, 0.145, 5, 35),
                   (60, 0.145, 0.085, 5, 30), (90, 0.085, 0.135, 40, 70), (60, 0.135, 0.07, 5, 30)]
POLAND_DAYS = 450


def poland_truth(ref) -> np.ndarray:
    """Chained integrate_euler segments -> (450, 4) true states."""
    state = np.array([POLAND_N - 200.0, 200.0, 0.0, 0.0])
    rows = [state]
    for length, b1, b2, t1, t2 in POLAND_SEGMENTS:
        st, fin = ref.integrate([b1, b2, t1, t2, 0.1, 0.0027], state, POLAND_N, length + 1)
        assert fin
        rows.extend(st[1:])
        state = st[-1]
    return np.array(rows[:POLAND_DAYS])


def poland_series(ref) -> dict:
    """Noise on daily increments x(1+U(-0.2,0.2)) (mt19937_64 seeded 2204,
    uniform01 draws in (day, column) order) and a weekday factor 1.1 / weekend
    0.7; re-cumulate; clean with the reference's build_epi_series + smooth7."""
    truth = poland_truth(ref)
    cum = np.stack([truth[:, 1] + truth[:, 2] + truth[:, 3], truth[:, 2], truth[:, 3]], axis=1)
    inc = np.diff(cum, axis=0, prepend=0.0)
    u = ref.uniform01(2204, inc.size).reshape(inc.shape)
    factor = 1.0 + (-0.2 + 0.4 * u)
    week = np.where((np.arange(POLAND_DAYS) % 7 >= 5), 0.7, 1.1)[:, None]
    noisy = np.cumsum(np.maximum(inc * factor * week, 0.0), axis=0)
    out = {k: np.zeros(POLAND_DAYS) for k in ("I", "R", "D", "new")}
    dp = op._dp
    rc = ref.lib.ref_clean_series(np.ascontiguousarray(noisy[:, 0]).ctypes.data_as(dp),
                                  np.ascontiguousarray(noisy[:, 1]).ctypes.data_as(dp),
                                  np.ascontiguousarray(noisy[:, 2]).ctypes.data_as(dp), POLAND_DAYS, 1,
                                  out["I"].ctypes.data_as(dp), out["R"].ctypes.data_as(dp),
                                  out["D"].ctypes.data_as(dp), out["new"].ctypes.data_as(dp))
    assert rc == 0, ref.lib.ref_last_error()
    out["truth"] = truth
    return out


def write_series_csv(path: Path, s: dict) -> None:
    lines = ["day,infectious,recovered_cum,deaths_cum,new_cases"]
    for t in range(POLAND_DAYS):
        lines.append(f"{t},{float(s['I'][t])!r},{float(s['R'][t])!r},{float(s['D'][t])!r},{float(s['new'][t])!r}")
    path.write_text("\n".join(lines) + "\n")


def stage_box(stage: int, tau: int):
    if stage == 1:
        return [0, 0, 0, 0, 0, 0], [10, 10, tau, tau, 10, 10]
    return [0, 0, 0, 0, 0, 0], [2, 2, tau - 7, tau - 7, 1, 0.1]


def uniform_particles(seed: int, n: int, lo, hi, repair=False) -> np.ndarray:
    """acceptance/main.cpp:443-451 style: one engine, row-major draws."""
    ref = op.load("reference")
    u = ref.uniform01(seed, n * 6).reshape(n, 6)
    lo, hi = np.array(lo, float), np.array(hi, float)
    x = lo + u * (hi - lo)
    if repair:
        sw = x[:, 2] > x[:, 3]
        x[sw, 2], x[sw, 3] = x[sw, 3].copy(), x[sw, 2].copy()
    return x


def special_particles(tau: int) -> np.ndarray:
    rows = [
        [0.6, 0.6, 1.0, 2.0, 0.09, 0.01],
        [1.5, 1.5, 8.0, 2.0, 0.01, 0.09],        # unordered switch times
        [0.3, 0.9, 5.0, 5.0, 0.1, 0.01],         # t1 == t2: no ramp
        [0.3, 0.9, 0.0, float(tau), 0.1, 0.01],  # ramp over the whole window
        [0.0, 2.0, 3.0, 9.0, 0.0, 0.0],          # zero rates
        [2.0, 0.0, 0.0, 1e-9, 1.0, 0.1],         # razor-thin ramp at t=0
        [10.0, 10.0, 0.0, 0.0, 0.0, 0.0],        # fast growth
        [10.0, 10.0, 0.0, 0.0, 10.0, 10.0],      # stage-1 corner
        [5e3, 5e3, 0.0, 0.0, 0.0, 0.0],          # blow-up
        [1e300, 1e300, 0.0, 0.0, 1.0, 1.0],      # immediate overflow
        [0.5, 0.5, 3.0, 7.0, 1e5, 1e5],          # stiff rates -> blow-up
        [-0.5, 0.4, 2.0, 6.0, 0.1, 0.01],        # negative beta through the ramp (sign crossing)
        [0.4, 0.8, float("nan"), 6.0, 0.1, 0.01],  # NaN switch time
        [0.4, 0.8, 2.0, float("nan"), 0.1, 0.01],
        [0.4, 0.8, 2.0, float("inf"), 0.1, 0.01],  # ramp never ends
        [1e-310, 0.7, 1.0, 9.0, 0.1, 0.01],      # subnormal beta1
        [0.7, 1e-310, 1.0, 9.0, 0.1, 0.01],      # subnormal beta2
        [-0.0, 0.7, 1.0, 9.0, 0.1, 0.01],        # negative zero
        [1e-200, 3e-200, 1.0, 9.0, 0.1, 0.01],   # tiny betas
        [0.2, 0.4, 2.0, 2.0 + 2 ** -40, 0.1, 0.01],  # ramp shorter than one substep
    ]
    return np.array(rows, dtype=np.float64)


def windows_for_costs(ref, poland: dict):
    """(name, I, R, D, init, N) cases."""
    out = []
    # poland-like windows: tau=20 window 0 (config 1) and tau=35 windows 0, 60, 138
    for tau, widx in ((20, 0), (35, 0), (35, 60), (35, 138)):
        s = widx * 3
        L = tau + 1
        I, R, D = poland["I"][s:s + L], poland["R"][s:s + L], poland["D"][s:s + L]
        init = [POLAND_N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
        out.append((f"poland_tau{tau}_w{widx}", tau, I, R, D, init, POLAND_N))
    # reference test fixture (test_calibration.cpp:139-152)
    N = 1e6
    st, _ = ref.integrate([0.6, 0.6, 0.0, 0.0, 0.09, 0.01], [N - 100, 100, 0, 0], N, 25)
    out.append(("boundary_fixture", 20, st[:21, 1], st[:21, 2], st[:21, 3], st[0], N))
    # flat window (range 0 -> 1/max(1,|lo|)), zero window (MAPE +inf), MAPE zeros
    L = 15
    out.append(("flat", 14, np.full(L, 50.0), np.full(L, 20.0), np.full(L, 0.5), [1000 - 70.5, 50, 20, 0.5], 1000.0))
    out.append(("zeros", 14, np.zeros(L), np.zeros(L), np.zeros(L), [1000.0, 0, 0, 0], 1000.0))
    Dz = np.concatenate([np.zeros(5), np.linspace(1, 30, L - 5)])
    st, _ = ref.integrate([0.5, 0.3, 3, 9, 0.1, 0.02], [5e5 - 40, 40, 0, 0], 5e5, L)
    out.append(("mape_zeros", 14, st[:, 1], np.concatenate([np.zeros(3), st[3:, 2]]), Dz, st[0], 5e5))
    return out


def gen_costs(ref, poland: dict) -> dict:
    data = {}
    for name, tau, I, R, D, init, N in windows_for_costs(ref, poland):
        lo1, hi1 = stage_box(1, tau)
        lo2, hi2 = stage_box(2, max(tau, 7))
        sets = {
            "stage2": uniform_particles(10, 96, lo2, hi2),
            "stage1": uniform_particles(11, 64, lo1, hi1),
            "special": special_particles(tau),
        }
        if name.startswith("poland"):
            # near-optimal: best fit of a short swarm, jittered x(1 +- 1e-6)
            rc, best, _, _ = ref.fit_swarm("ird-mxse", I, R, D, init, N, lo2, hi2, 256, 30, seed=3)
            u = ref.uniform01(12, 32 * 6).reshape(32, 6)
            sets["near_opt"] = best[None, :] * (1.0 + (u - 0.5) * 2e-6)
        data[f"{name}/obs"] = np.stack([I, R, D])
        data[f"{name}/init"] = np.array(init, dtype=np.float64)
        data[f"{name}/N"] = np.array([N])
        for sname, pos in sets.items():
            data[f"{name}/{sname}/positions"] = pos
            for spec in op.SPECS:
                data[f"{name}/{sname}/{spec}"] = ref.eval_costs(spec, I, R, D, init, N, pos)
    return data


def gen_fits(ref, poland: dict) -> list:
    cases = []
    N = 1e6
    st, _ = ref.integrate([0.6, 0.6, 0.0, 0.0, 0.09, 0.01], [N - 100, 100, 0, 0], N, 25)
    cases.append(dict(name="appendixA", spec="ird-mxse", I=st[:21, 1], R=st[:21, 2], D=st[:21, 3], init=st[0],
                      N=N, tau=20, stage=2, n=64, iters=10, w=0.5, c1=0.5, c2=0.5, seed=1))
    s = poland
    for spec, n, iters, seed, widx, tau in (("ird-mxse", 256, 60, 1, 0, 20), ("d-mse", 200, 40, 5, 10, 35),
                                           ("ird-mape", 130, 25, 9, 100, 35), ("d-mae", 97, 30, 2, 138, 35)):
        a = widx * 3
        I, R, D = s["I"][a:a + tau + 1], s["R"][a:a + tau + 1], s["D"][a:a + tau + 1]
        cases.append(dict(name=f"poland_{spec}_w{widx}", spec=spec, I=I, R=R, D=D,
                          init=[POLAND_N - I[0] - R[0] - D[0], I[0], R[0], D[0]], N=POLAND_N, tau=tau, stage=2,
                          n=n, iters=iters, w=0.5, c1=0.5, c2=0.5, seed=seed))
    # constriction coefficients (acceptance #6) and stage-1 bounds
    a = 30
    I, R, D = s["I"][a:a + 36], s["R"][a:a + 36], s["D"][a:a + 36]
    cases.append(dict(name="poland_stage1_constriction", spec="ird-mse", I=I, R=R, D=D,
                      init=[POLAND_N - I[0] - R[0] - D[0], I[0], R[0], D[0]], N=POLAND_N, tau=35, stage=1,
                      n=150, iters=40, w=0.7298, c1=1.4962, c2=1.4962, seed=601))
    # all-zero data (test_calibration.cpp:210-224) and an all-infeasible swarm
    z = np.zeros(15)
    cases.append(dict(name="zeros", spec="d-mse", I=z, R=z, D=z, init=[1000.0, 0, 0, 0], N=1000.0, tau=14,
                      stage=2, n=50, iters=5, w=0.5, c1=0.5, c2=0.5, seed=3))
    cases.append(dict(name="all_infeasible", spec="ird-mape", I=z, R=z, D=z, init=[1000.0, 0, 0, 0], N=1000.0,
                      tau=14, stage=2, n=33, iters=4, w=0.5, c1=0.5, c2=0.5, seed=4))
    out = []
    for c in cases:
        lo, hi = stage_box(c["stage"], c["tau"])
        rc, best, cost, hist = ref.fit_swarm(c["spec"], c["I"], c["R"], c["D"], c["init"], c["N"], lo, hi, c["n"],
                                             c["iters"], c["w"], c["c1"], c["c2"], c["seed"])
        rec = {k: (np.asarray(v).tolist() if isinstance(v, (np.ndarray, list)) else v) for k, v in c.items()}
        rec.update(lower=lo, upper=hi, status=rc, best=[float(x).hex() for x in best], best_cost=float(cost).hex(),
                   history=[float(x).hex() for x in hist])
        rec["I"] = [float(x).hex() for x in c["I"]]
        rec["R"] = [float(x).hex() for x in c["R"]]
        rec["D"] = [float(x).hex() for x in c["D"]]
        rec["init"] = [float(x).hex() for x in c["init"]]
        out.append(rec)
    return out


def gen_forecast(ref, poland: dict) -> dict:
    data = {}
    pos = np.concatenate([uniform_particles(21, 24, *stage_box(2, 35), repair=True), special_particles(35)[:12]])
    a = 414
    I, R, D = poland["I"][a:a + 36], poland["R"][a:a + 36], poland["D"][a:a + 36]
    init = [POLAND_N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
    traj, fin_w, fc, fin_f = [], [], [], []
    for p in pos:
        st, fin = ref.integrate(p, init, POLAND_N, 36)
        traj.append(st)
        fin_w.append(fin)
        if fin:
            f, ff = ref.forecast(p, st[-1], POLAND_N, 21)
        else:
            f, ff = np.full((22, 4), np.nan), False
        fc.append(f)
        fin_f.append(ff)
    data.update(positions=pos, init=np.array(init), N=np.array([POLAND_N]), window=np.array(traj),
                window_finite=np.array(fin_w), forecast=np.array(fc), forecast_finite=np.array(fin_f))
    return data


def _hex(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).ravel()]


def synthetic_series(ref, params, n_days, N=1e6, i0=100.0):
    """tests/synthetic.hpp:22-49: the model's own trajectory as the series."""
    st, _ = ref.integrate(params, [N - i0, i0, 0, 0], N, n_days)
    return st[:, 1].copy(), st[:, 2].copy(), st[:, 3].copy()


STAGE_BOUNDS7 = {1: [0, 10, 0, 10, 0, 10, 0], 2: [0, 2, 0, 1, 0, 0.1, 7]}


def gen_calibration(ref, poland: dict) -> dict:
    """fit_window / fit_all_windows / stability_study / forecast_extension
    of the reference on small cases (calibration.cpp:157-436)."""
    dp = op._dp
    out = {"fit_window": [], "fit_all_windows": [], "stability": []}

    def arr(x):
        return np.ascontiguousarray(x, dtype=np.float64)

    fw_cases = []
    I, R, D = synthetic_series(ref, [0.6, 0.6, 0, 0, 0.09, 0.01], 25)
    fw_cases.append(("appendixA", I, R, D, 0, 21, "ird-mxse", 2, 1e6, 64, 10, 1, 21))
    fw_cases.append(("poland_c1_small", poland["I"], poland["R"], poland["D"], 0, 21, "ird-mxse", 2, POLAND_N, 256,
                     50, 1, 21))
    fw_cases.append(("poland_w100_dmape", poland["I"], poland["R"], poland["D"], 300, 36, "d-mape", 2, POLAND_N,
                     200, 20, 7, 21))
    fw_cases.append(("poland_stage1", poland["I"], poland["R"], poland["D"], 150, 36, "ird-mae", 1, POLAND_N, 100,
                     15, 3, 10))
    z = np.zeros(15)
    fw_cases.append(("zeros", z, z, z, 0, 15, "d-mse", 2, 1000.0, 50, 5, 3, 5))
    fw_cases.append(("too_small_population", I, R, D, 0, 21, "ird-mse", 2, 10.0, 30, 5, 4, 5))
    fw_cases.append(("window_outside", I, R, D, 10, 21, "ird-mse", 2, 1e6, 30, 5, 4, 5))
    fw_cases.append(("margin_too_big", I, R, D, 0, 5, "ird-mse", 2, 1e6, 30, 5, 4, 5))
    fw_cases.append(("all_infeasible", z, z, z, 0, 15, "ird-mape", 2, 1000.0, 33, 4, 4, 5))
    for name, I, R, D, start, length, spec, stage, N, n, iters, seed, horizon in fw_cases:
        fam, met = op.parse_spec(spec)
        I, R, D = arr(I), arr(R), arr(D)
        b7 = arr(STAGE_BOUNDS7[stage])
        best, obj, r2, fin = np.zeros(6), np.zeros(1), np.zeros(1), ctypes_int()
        traj = np.zeros((length, 4))
        rc = ref.lib.ref_fit_window(I.ctypes.data_as(dp), R.ctypes.data_as(dp), D.ctypes.data_as(dp), len(I), start,
                                    length, fam, met, b7.ctypes.data_as(dp), N, 24, 1, n, iters, 0.5, 0.5, 0.5, seed,
                                    best.ctypes.data_as(dp), obj.ctypes.data_as(dp), r2.ctypes.data_as(dp),
                                    traj.ctypes.data_as(dp), fin)
        rec = dict(name=name, I=_hex(I), R=_hex(R), D=_hex(D), start=start, length=length, spec=spec, stage=stage,
                   N=N, n=n, iters=iters, seed=seed, horizon=horizon, status=rc)
        if rc == 0:
            fc = np.zeros((horizon + 1, 4))
            frc = ref.lib.ref_fit_window_forecast(I.ctypes.data_as(dp), R.ctypes.data_as(dp), D.ctypes.data_as(dp),
                                                  len(I), start, length, fam, met, b7.ctypes.data_as(dp), N, 24, n,
                                                  iters, seed, horizon, fc.ctypes.data_as(dp))
            rec.update(params=_hex(best), objective=float(obj[0]).hex(), r2=float(r2[0]).hex(),
                       trajectory=_hex(traj), forecast_status=frc, forecast=_hex(fc) if frc == 0 else None)
        else:
            rec["error"] = ref.lib.ref_last_error().decode()
        out["fit_window"].append(rec)

    fa_cases = []
    I, R, D = synthetic_series(ref, [0.5, 0.3, 5.0, 12.0, 0.1, 0.02], 31)
    fa_cases.append(("test_calibration_seeded", I, R, D, 14, 8, "ird-mxse", 2, 1e6, 150, 40, 11))
    I2, R2, D2 = synthetic_series(ref, [0.5, 0.5, 0, 0, 0.1, 0.02], 31, i0=500.0)
    I2 = I2.copy()
    I2[14:] = 2e6  # test_calibration.cpp:255-275: the third window covers the flood
    fa_cases.append(("population_flood", I2, R2, D2, 10, 7, "ird-mxse", 2, 1e6, 60, 10, 5))
    fa_cases.append(("poland_first_120d", poland["I"][:120], poland["R"][:120], poland["D"][:120], 35, 3, "ird-mse",
                     2, POLAND_N, 64, 20, 2204))
    for name, I, R, D, tau, delta, spec, stage, N, n, iters, seed in fa_cases:
        fam, met = op.parse_spec(spec)
        I, R, D = arr(I), arr(R), arr(D)
        b7 = arr(STAGE_BOUNDS7[stage])
        mw = 64
        nw, failed = (ctypes_size(), ctypes_size())
        ok = np.zeros(mw, dtype=np.int32)
        best, obj, r2, mean = np.zeros(6 * mw), np.zeros(mw), np.zeros(mw), np.zeros(1)
        rc = ref.lib.ref_fit_all_windows(I.ctypes.data_as(dp), R.ctypes.data_as(dp), D.ctypes.data_as(dp), len(I),
                                         tau, delta, fam, met, b7.ctypes.data_as(dp), N, 24, 1, n, iters, 0.5, 0.5,
                                         0.5, seed, mw, nw, ok.ctypes.data_as(op._ip), best.ctypes.data_as(dp),
                                         obj.ctypes.data_as(dp), r2.ctypes.data_as(dp), mean.ctypes.data_as(dp), failed)
        assert rc == 0, name
        k = nw.value
        out["fit_all_windows"].append(dict(
            name=name, I=_hex(I), R=_hex(R), D=_hex(D), tau=tau, delta=delta, spec=spec, stage=stage, N=N, n=n,
            iters=iters, seed=seed, n_windows=k, ok=ok[:k].tolist(), params=_hex(best[:6 * k]), objective=_hex(obj[:k]),
            r2=_hex(r2[:k]), mean_r2=float(mean[0]).hex(), failed=failed.value))

    st_cases = []
    I, R, D = synthetic_series(ref, [0.5, 0.4, 2.0, 6.0, 0.1, 0.02], 31)
    st_cases.append(("one_repetition", I, R, D, 5, 11, "ird-mxse", 2, 1e6, 120, 30, 1, 4, 99))
    st_cases.append(("seven_repetitions", I, R, D, 5, 11, "d-mse", 2, 1e6, 80, 25, 7, 6, 901))
    I3, R3, D3 = synthetic_series(ref, [0.5, 0.5, 0, 0, 0.1, 0.02], 20)
    st_cases.append(("population_too_small", I3, R3, D3, 0, 11, "ird-mxse", 2, 1.0, 30, 5, 3, 2, 1))
    st_cases.append(("poland_last_window", poland["I"], poland["R"], poland["D"], 414, 36, "ird-mxse", 2, POLAND_N,
                     64, 15, 5, 21, 2204))
    for name, I, R, D, start, length, spec, stage, N, n, iters, reps, horizon, seed in st_cases:
        fam, met = op.parse_spec(spec)
        I, R, D = arr(I), arr(R), arr(D)
        b7 = arr(STAGE_BOUNDS7[stage])
        sizes = [length, length, length + horizon, length + horizon, length + horizon]
        ok = np.zeros(reps, dtype=np.int32)
        params, obj = np.zeros(6 * reps), np.zeros(reps)
        bands, counts = np.zeros(7 * sum(sizes)), np.zeros(sum(sizes), dtype=np.uint64)
        sc, scc, failed = np.zeros(14), np.zeros(2, dtype=np.uint64), np.zeros(1, dtype=np.uint64)
        u64 = lambda a: a.ctypes.data_as(op._u64p)  # noqa: E731
        rc = ref.lib.ref_stability_study(I.ctypes.data_as(dp), R.ctypes.data_as(dp), D.ctypes.data_as(dp), len(I),
                                         start, length, fam, met, b7.ctypes.data_as(dp), N, 24, n, iters, 0.5, 0.5,
                                         0.5, reps, horizon, seed, ok.ctypes.data_as(op._ip),
                                         params.ctypes.data_as(dp), obj.ctypes.data_as(dp), bands.ctypes.data_as(dp),
                                         u64(counts), sc.ctypes.data_as(dp), u64(scc), u64(failed))
        assert rc == 0, name
        out["stability"].append(dict(
            name=name, I=_hex(I), R=_hex(R), D=_hex(D), start=start, length=length, spec=spec, stage=stage, N=N, n=n,
            iters=iters, reps=reps, horizon=horizon, seed=seed, ok=ok.tolist(), params=_hex(params),
            objective=_hex(obj), day_bands=_hex(bands), day_counts=counts.astype(int).tolist(), scalar_bands=_hex(sc),
            scalar_counts=scc.astype(int).tolist(), failed=int(failed[0])))
    return out


def gen_ensemble_bands(ref, poland: dict) -> list:
    """Forecast-scenario ensembles reduced to build_quantile_bands by the
    reference: sample k = Swarm-init draws of mt19937_64(mix_seed(seed, k))
    (pso.cpp:55-73) + repair, integrate_euler over the window, then
    forecast_extension; blown-up samples are NaN rows (dropped)."""
    out = []
    dp = op._dp
    for name, widx, stage, seed, n, horizon in (("poland_w138_stage2", 138, 2, 2204, 3000, 21),
                                                ("poland_w33_stage1", 33, 1, 77, 2000, 21),
                                                ("poland_w90_wild", 90, 0, 13, 1500, 14),
                                                ("poland_w0_h0", 0, 2, 5, 257, 0)):
        a = 3 * widx
        I, R, D = poland["I"][a:a + 36], poland["R"][a:a + 36], poland["D"][a:a + 36]
        init = np.array([POLAND_N - I[0] - R[0] - D[0], I[0], R[0], D[0]])
        if stage == 0:  # rates up to 60/day: explicit Euler at h = 1/24 blows up for part of the box
            lo, hi = np.zeros(6), np.array([60.0, 60.0, 28.0, 28.0, 60.0, 60.0])
        else:
            lo, hi = (np.array(v, dtype=np.float64) for v in stage_box(stage, 35))
        rows = np.full((n, horizon + 1), np.nan)
        for k in range(n):
            u = ref.uniform01(ref.mix_seed(seed, k), 6)
            x = lo + u * (hi - lo)
            if x[2] > x[3]:
                x[2], x[3] = x[3], x[2]
            st, fin = ref.integrate(x, init, POLAND_N, 36)
            if not fin:
                continue
            fc, ff = ref.forecast(x, st[-1], POLAND_N, horizon)
            if ff:
                rows[k] = fc[:, 3]
        vals = np.ascontiguousarray(rows)
        bands = np.zeros(7 * (horizon + 1))
        counts = np.zeros(horizon + 1, dtype=np.uint64)
        rc = ref.lib.ref_quantile_bands(vals.ctypes.data_as(dp), n, horizon + 1, bands.ctypes.data_as(dp),
                                        counts.ctypes.data_as(op._szp))
        assert rc == 0
        out.append(dict(name=name, I=_hex(I), R=_hex(R), D=_hex(D), init=_hex(init), N=POLAND_N, stage=stage,
                        lower=_hex(lo), upper=_hex(hi), seed=seed, n=n, horizon=horizon, bands=_hex(bands),
                        counts=counts.astype(int).tolist(), blown=int(np.isnan(rows[:, -1]).sum())))
    return out


def gen_series(ref) -> dict:
    """Host data layer pins (tools/main.cpp inputs/outputs): format_double,
    build_epi_series(+smooth7) on raw series with gaps / dips / outflow caps,
    and build_envelope, all by the reference."""
    import ctypes
    dp = op._dp
    rng = np.random.default_rng(2204)
    out = {"format_double": [], "clean": [], "envelope": []}
    vals = [0.0, -0.0, 1.0, 2.5, 1e-05, 0.0001, 123456789.0, 1.2345678901234567e17, 1e16, 1e15, 1e21, 3.14159,
            -2.75, 5e-324, 1.7976931348623157e308, 1e-7, 123.456, 0.1 + 0.2, 38000000.0, 85358.31234, float("inf"),
            -float("inf"), float("nan"), 100.0, 1e22, 12345678.9, 2 ** 53, 0.5, 9.999999999999999e-5]
    vals += list(rng.standard_normal(40) * 10.0 ** rng.integers(-12, 20, 40))
    buf = ctypes.create_string_buffer(64)
    for v in vals:
        ref.lib.ref_format_double(float(v), buf)
        out["format_double"].append([float(v).hex(), buf.value.decode()])
    for case in range(6):
        n = int(rng.integers(20, 80))
        days = np.sort(rng.choice(np.arange(n + 20), size=n, replace=False)).astype(np.int32)
        days -= days[0]
        base = np.cumsum(rng.uniform(0, 50, size=(n, 3)), axis=0) * np.array([3.0, 1.5, 0.2])
        if case >= 2:  # reporting dips and outflow spikes
            base[rng.integers(1, n - 1, 4), 1] *= 0.5
            base[rng.integers(1, n - 1, 3), 2] *= 0.3
            base[rng.integers(1, n - 1, 3), 1] += 5000.0
        raw = base.copy()
        mask = rng.random((n, 3)) < (0.15 if case % 2 else 0.0)
        mask[0] = mask[-1] = False
        raw[mask] = np.nan
        for smooth in (0, 1):
            m = int(days[-1]) + 1
            I, R, D, NEW = (np.zeros(m) for _ in range(4))
            nout = ctypes.c_size_t()
            stats = np.zeros(3, dtype=np.uint64)
            c_, r_, d_ = (np.ascontiguousarray(raw[:, k]) for k in range(3))
            rc = ref.lib.ref_clean_raw(days.ctypes.data_as(op._ip), c_.ctypes.data_as(dp), r_.ctypes.data_as(dp),
                                       d_.ctypes.data_as(dp), n, smooth, m, I.ctypes.data_as(dp),
                                       R.ctypes.data_as(dp), D.ctypes.data_as(dp), NEW.ctypes.data_as(dp),
                                       ctypes.byref(nout), stats.ctypes.data_as(op._u64p))
            assert rc == 0, ref.lib.ref_last_error()
            out["clean"].append(dict(days=days.tolist(), raw=[[None if np.isnan(x) else float(x).hex() for x in row]
                                                              for row in raw], smooth=smooth, I=_hex(I), R=_hex(R),
                                     D=_hex(D), new=_hex(NEW), stats=stats.astype(int).tolist()))
    for case in range(4):
        ns, nd = int(rng.integers(1, 12)), int(rng.integers(1, 9))
        v = rng.standard_normal((ns, nd))
        v[rng.random((ns, nd)) < 0.2] = np.nan
        bands = np.zeros(7 * nd)
        cnt = np.zeros(nd, dtype=np.uint64)
        v = np.ascontiguousarray(v)
        assert ref.lib.ref_build_envelope(v.ctypes.data_as(dp), ns, nd, bands.ctypes.data_as(dp),
                                          cnt.ctypes.data_as(op._szp)) == 0
        out["envelope"].append(dict(values=[[None if np.isnan(x) else float(x).hex() for x in row] for row in v],
                                    bands=_hex(bands), counts=cnt.astype(int).tolist()))
    return out


def gen_cli(ref) -> dict:
    """acceptance/main.cpp:180-207 setup: a model trajectory reported as raw
    cumulative counts (synthetic.hpp:56-69), cleaned by build_epi_series and
    fitted by fit_all_windows with the CLI's settings; the reference's
    per-window results for `fit --tau 20 --delta 10 --objective ird-mxse
    --particles 300 --iters 40 --seed 7`."""
    import ctypes
    dp = op._dp
    N = 1e6
    st, _ = ref.integrate([0.55, 0.85, 15.0, 30.0, 0.09, 0.012], [N - 100, 100, 0, 0], N, 60)
    confirmed = st[:, 1] + st[:, 2] + st[:, 3]
    raw = np.stack([confirmed, st[:, 2], st[:, 3]], axis=1)
    n = len(raw)
    days = np.arange(n, dtype=np.int32)
    I, R, D, NEW = (np.zeros(n) for _ in range(4))
    nout = ctypes.c_size_t()
    stats = np.zeros(3, dtype=np.uint64)
    c_, r_, d_ = (np.ascontiguousarray(raw[:, k]) for k in range(3))
    assert ref.lib.ref_clean_raw(days.ctypes.data_as(op._ip), c_.ctypes.data_as(dp), r_.ctypes.data_as(dp),
                                 d_.ctypes.data_as(dp), n, 0, n, I.ctypes.data_as(dp), R.ctypes.data_as(dp),
                                 D.ctypes.data_as(dp), NEW.ctypes.data_as(dp), ctypes.byref(nout),
                                 stats.ctypes.data_as(op._u64p)) == 0
    mw = 16
    nw, failed = ctypes.c_size_t(), ctypes.c_size_t()
    ok = np.zeros(mw, dtype=np.int32)
    best, obj, r2, mean = np.zeros(6 * mw), np.zeros(mw), np.zeros(mw), np.zeros(1)
    b7 = np.ascontiguousarray(STAGE_BOUNDS7[2], dtype=np.float64)
    assert ref.lib.ref_fit_all_windows(I.ctypes.data_as(dp), R.ctypes.data_as(dp), D.ctypes.data_as(dp), n, 20, 10,
                                       1, 0, b7.ctypes.data_as(dp), N, 24, 1, 300, 40, 0.5, 0.5, 0.5, 7, mw, nw,
                                       ok.ctypes.data_as(op._ip), best.ctypes.data_as(dp), obj.ctypes.data_as(dp),
                                       r2.ctypes.data_as(dp), mean.ctypes.data_as(dp), failed) == 0
    k = nw.value
    buf = ctypes.create_string_buffer(64)
    cells = []
    for row in raw:
        out_row = []
        for v in row:
            ref.lib.ref_format_double(float(v), buf)
            out_row.append(buf.value.decode())
        cells.append(out_row)
    return dict(raw_cells=cells, start_date="2020-03-01", n_windows=k, ok=ok[:k].tolist(),
                params=_hex(best[:6 * k]), objective=_hex(obj[:k]), r2=_hex(r2[:k]), mean_r2=float(mean[0]).hex(),
                failed=failed.value)


def ctypes_int():
    import ctypes
    return ctypes.byref(ctypes.c_int(0))


def ctypes_size():
    import ctypes
    return ctypes.c_size_t(0)


def gen_kat(ref) -> dict:
    return {
        "mix_seed": [[b, i, ref.mix_seed(b, i)] for b, i in ((0, 0), (1, 0), (1, 1), (2204, 7),
                                                            (2**64 - 1, 12345), (42, 2**63))],
        "mt_default_10000th": int(ref.mt_raw(5489, 1, skip=9999)[0]),
        "mt_mix00_first_700": [int(x) for x in ref.mt_raw(ref.mix_seed(0, 0), 700)],
        "uniform01_mix10_first_3": [float(x).hex() for x in ref.uniform01(ref.mix_seed(1, 0), 3)],
    }


def main() -> None:
    op.build("ref")
    ref = op.load("reference")
    GOLDEN.mkdir(parents=True, exist_ok=True)
    poland = poland_series(ref)
    write_series_csv(GOLDEN / "poland_like.csv", poland)
    truth = poland["truth"]
    print(f"poland-like: true D[449]={truth[-1, 3]:.1f} confirmed={truth[-1, 1:].sum():.1f} "
          f"I peak={truth[:, 1].max():.1f} at day {int(truth[:, 1].argmax())}; cleaned D[449]={poland['D'][-1]:.1f}")
    (GOLDEN / "kat.json").write_text(json.dumps(gen_kat(ref), indent=1))
    np.savez_compressed(GOLDEN / "costs.npz", **gen_costs(ref, poland))
    (GOLDEN / "fits.json").write_text(json.dumps(gen_fits(ref, poland), indent=1))
    np.savez_compressed(GOLDEN / "forecast.npz", **gen_forecast(ref, poland))
    (GOLDEN / "calibration.json").write_text(json.dumps(gen_calibration(ref, poland)))
    (GOLDEN / "ensemble_bands.json").write_text(json.dumps(gen_ensemble_bands(ref, poland)))
    (GOLDEN / "series.json").write_text(json.dumps(gen_series(ref)))
    (GOLDEN / "cli_fit.json").write_text(json.dumps(gen_cli(ref)))
    print("wrote", sorted(p.name for p in GOLDEN.iterdir()))


if __name__ == "__main__":
    main()
