"""Python mirror of the reference's `sirdfit` module (proj/bindings/module.cpp,
proj/python/sirdfit/__init__.py), running on the B200 engine.

Same names, argument names, defaults and exception types as the reference's
pybind11 module, so `import paper_2204_12346_b200.sirdfit as sirdfit` is a
drop-in for the calibration path.  The functions call the C++ host layer
(csrc/host_api.cpp) through the C-ABI (include/sirdgpu.h); every SIRD
integration and cost evaluation runs on the GPU.

`load_raw_csv` runs the reference's cleaning pipeline (timeseries.cpp),
restated on the host in paper_2204_12346_b200/series.py.
"""
from __future__ import annotations

import csv
import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _capi
from .errors import (AllInfeasibleError, ConstantObservedError, DegenerateRatesError, Error, NonFiniteError,
                     SchemeError, raise_for_status)

kDefaultSubsteps = 24  # model.hpp:12

__all__ = ["EpiSeries", "FitAllResult", "FitResult", "Forecast", "SirdParams", "SirdState", "Trajectory", "Window",
           "StabilityResult", "QuantileBands", "ScalarBands", "basic_reproduction_number", "beta_at",
           "fit_all_windows", "fit_window", "forecast_extension", "integrate", "load_epi_csv", "load_raw_csv",
           "make_windows",
           "stability_study", "mix_seed", "r_squared_d"]


@dataclass
class SirdParams:  # module.cpp:52-72
    beta1: float = 0.0
    beta2: float = 0.0
    t1: float = 0.0
    t2: float = 0.0
    gamma: float = 0.0
    mu: float = 0.0

    def as_array(self) -> np.ndarray:
        return np.array([self.beta1, self.beta2, self.t1, self.t2, self.gamma, self.mu])


@dataclass
class SirdState:  # module.cpp:74-88
    S: float = 0.0
    I: float = 0.0
    R: float = 0.0
    D: float = 0.0

    def total(self) -> float:
        return self.S + self.I + self.R + self.D


@dataclass
class Trajectory:  # module.cpp:90-94
    states: list
    population: float
    finite: bool

    def days(self) -> int:
        return len(self.states)

    @staticmethod
    def from_array(a: np.ndarray, population: float, finite: bool) -> "Trajectory":
        return Trajectory([SirdState(*map(float, row)) for row in a], float(population), bool(finite))


@dataclass
class EpiSeries:  # module.cpp:96-105
    infectious: list
    recovered_cum: list
    deaths_cum: list
    new_cases: list
    start_date: str = "2020-03-18"

    def size(self) -> int:
        return len(self.infectious)

    def __len__(self) -> int:
        return self.size()


@dataclass
class Window:  # module.cpp:107-118
    index: int
    start: int
    length: int

    def last_day(self) -> int:
        return self.start + self.length - 1


@dataclass
class FitResult:  # module.cpp:120-127
    window: Window
    params: SirdParams
    objective: float
    r2_d: float
    trajectory: Optional[Trajectory]
    ok: bool
    failure: str
    population: float = 0.0
    substeps: int = kDefaultSubsteps


@dataclass
class FitAllResult:  # module.cpp:129-132
    fits: list
    mean_r2_d: float
    failed_count: int


@dataclass
class Forecast:  # module.cpp:134-137
    junction_day: int
    horizon: int
    trajectory: Trajectory


@dataclass
class QuantileBands:  # calibration.hpp:150-160
    count: list
    median: list
    p50_lo: list
    p50_hi: list
    p90_lo: list
    p90_hi: list
    p95_lo: list
    p95_hi: list

    def days(self) -> int:
        return len(self.count)


@dataclass
class ScalarBands:  # calibration.hpp:162-168
    count: int
    median: float
    p50_lo: float
    p50_hi: float
    p90_lo: float
    p90_hi: float
    p95_lo: float
    p95_hi: float


@dataclass
class StabilityResult:  # calibration.hpp:173-186
    window: Window
    horizon: int
    repetitions: int
    failed: int
    beta: QuantileBands
    r0: QuantileBands
    infectious: QuantileBands
    recovered: QuantileBands
    deaths: QuantileBands
    gamma: ScalarBands
    mu: ScalarBands
    fits: list = field(default_factory=list)


_BOUNDS = {  # ParamBounds::stage1 / stage2 (calibration.cpp:54-65)
    "stage1": dict(beta_lo=0.0, beta_hi=10.0, gamma_lo=0.0, gamma_hi=10.0, mu_lo=0.0, mu_hi=10.0, t_margin=0),
    "stage2": dict(beta_lo=0.0, beta_hi=2.0, gamma_lo=0.0, gamma_hi=1.0, mu_lo=0.0, mu_hi=0.1, t_margin=7),
}

_default_ctx: Optional[_capi.Context] = None


def context() -> _capi.Context:
    """The engine context these functions run on (device 0 unless set_context)."""
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = _capi.Context(0)
    return _default_ctx


def set_context(ctx: _capi.Context) -> None:
    global _default_ctx
    _default_ctx = ctx


def mix_seed(base: int, index: int) -> int:
    """pso.cpp:36-41 (SplitMix64 finalizer)."""
    m = 0xFFFFFFFFFFFFFFFF
    z = (base + 0x9E3779B97F4A7C15 * (index + 1)) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def beta_at(params: SirdParams, t: float) -> float:
    """model.cpp:55-64."""
    if t < params.t1:
        return params.beta1
    if t >= params.t2:
        return params.beta2
    slope = (params.beta2 - params.beta1) / (params.t2 - params.t1)
    return params.beta1 + slope * (t - params.t1)


def basic_reproduction_number(beta: float, gamma: float, mu: float) -> float:
    removal = gamma + mu
    if removal <= 0.0:
        raise DegenerateRatesError()
    return beta / removal


def r_squared_d(observed_d, predicted_d) -> float:
    """objectives.cpp:122-144 (sequential sums, same order)."""
    if len(observed_d) == 0 or len(observed_d) != len(predicted_d):
        raise Error("r_squared_d: series must be non-empty and of equal length")
    mean = 0.0
    for y in observed_d:
        mean += float(y)
    mean /= float(len(observed_d))
    ss_res = ss_tot = 0.0
    for y, p in zip(observed_d, predicted_d):
        e = float(y) - float(p)
        ss_res += e * e
        c = float(y) - mean
        ss_tot += c * c
    if ss_tot == 0.0:
        raise ConstantObservedError()
    return 1.0 - ss_res / ss_tot


def integrate(params: SirdParams, init: SirdState, population: float, n_days: int,
              substeps: int = kDefaultSubsteps) -> Trajectory:
    """integrate_euler (model.cpp:76-107) on the device."""
    if n_days < 1 or substeps < 1 or not (population > 0.0):
        raise Error("integrate_euler needs n_days >= 1, substeps >= 1 and a positive population")
    states, fin = context().integrate_batch(params.as_array()[None, :], [init.S, init.I, init.R, init.D],
                                            population, n_days, substeps)
    return Trajectory.from_array(states[0], population, fin[0])


def make_windows(n_days: int, tau: int = 35, delta: int = 3) -> list:
    """calibration.cpp:37-52."""
    if tau < 1 or delta < 1:
        raise SchemeError("window scheme needs tau >= 1 and delta >= 1")
    if n_days < tau + 1:
        raise SchemeError(f"series has {n_days} days; a window needs {tau + 1}")
    count = 1 + (n_days - 1 - tau) // delta
    return [Window(i, i * delta, tau + 1) for i in range(count)]


def load_raw_csv(path: str, smooth: bool = False) -> EpiSeries:
    """module.cpp:151-162: read date,confirmed,recovered,deaths and clean it
    (build_epi_series, optionally smooth7)."""
    from . import series as S
    epi = S.build_epi_series(S.read_raw_csv_file(path))
    if smooth:
        epi = S.smooth7(epi)
    return EpiSeries(epi.infectious, epi.recovered_cum, epi.deaths_cum, epi.new_cases, S.format_date(epi.start_date))


def load_epi_csv(path: str) -> EpiSeries:
    """Read a cleaned series (columns infectious, recovered_cum, deaths_cum[, new_cases])."""
    with open(path, newline="") as f:
        rows = list(csv.DictReader(f))
    col = lambda k: [float(r[k]) for r in rows]  # noqa: E731
    new = col("new_cases") if rows and "new_cases" in rows[0] else [0.0] * len(rows)
    return EpiSeries(col("infectious"), col("recovered_cum"), col("deaths_cum"), new)


def _settings(population, objective, bounds, particles, iters, inertia, cognitive, social, substeps):
    fam, met = _capi.parse_spec(objective)
    if bounds not in _BOUNDS:
        raise Error(f"unknown bounds preset: {bounds}")
    b = _BOUNDS[bounds]
    return _capi.sg_fit_settings(fam, met, b["beta_lo"], b["beta_hi"], b["gamma_lo"], b["gamma_hi"], b["mu_lo"],
                                 b["mu_hi"], b["t_margin"], int(particles), int(iters), float(inertia),
                                 float(cognitive), float(social), float(population), int(substeps))


def _series(data: EpiSeries):
    return tuple(np.ascontiguousarray(a, dtype=np.float64) for a in (data.infectious, data.recovered_cum,
                                                                      data.deaths_cum))


def _fit_from_record(rec, traj: Optional[np.ndarray], population: float, substeps: int) -> FitResult:
    w = Window(int(rec.index), int(rec.start), int(rec.length))
    p = SirdParams(*[float(v) for v in rec.params])
    trajectory = None
    if rec.ok and traj is not None:
        trajectory = Trajectory.from_array(traj, population, bool(np.isfinite(traj).all()))
    if not rec.ok:
        p = SirdParams()
    return FitResult(w, p, float(rec.objective) if rec.ok else math.nan, float(rec.r2_d) if rec.ok else math.nan,
                     trajectory, bool(rec.ok), rec.failure.decode(), population, substeps)


def fit_window(data: EpiSeries, window: Window, population: float, objective: str = "ird-mxse",
               bounds: str = "stage2", particles: int = 10000, iters: int = 100, inertia: float = 0.5,
               cognitive: float = 0.5, social: float = 0.5, seed: int = 0, substeps: int = kDefaultSubsteps,
               threads: int = 1) -> FitResult:
    """fit_window (calibration.cpp:157-188); module.cpp:167-180 signature."""
    s = _settings(population, objective, bounds, particles, iters, inertia, cognitive, social, substeps)
    return fit_window_settings(data, window, s, seed)


def fit_window_settings(data: EpiSeries, window: Window, s, seed: int = 0) -> FitResult:
    """fit_window with an explicit sg_fit_settings (any bounds, e.g. the CLI's custom box)."""
    ctx = context()
    population, substeps = s.population, s.substeps
    I, R, D = _series(data)
    rec = _capi.sg_fit_record()
    traj = np.empty((max(int(window.length), 1), 4))
    rc = _capi.lib().sg_fit_window_series(ctx.handle, _capi._d(I), _capi._d(R), _capi._d(D), len(I),
                                          int(window.start), int(window.length), ctypes.byref(s),
                                          int(seed) & 0xFFFFFFFFFFFFFFFF, ctypes.byref(rec), _capi._d(traj), None)
    if rc:
        raise_for_status(rc, rec.failure.decode())
    fit = _fit_from_record(rec, traj, population, substeps)
    fit.window = Window(window.index, window.start, window.length)
    return fit


def fit_all_windows(data: EpiSeries, population: float, tau: int = 35, delta: int = 3,
                    objective: str = "ird-mxse", bounds: str = "stage2", particles: int = 10000, iters: int = 100,
                    inertia: float = 0.5, cognitive: float = 0.5, social: float = 0.5, seed: int = 0,
                    substeps: int = kDefaultSubsteps, threads: int = 1) -> FitAllResult:
    """fit_all_windows (calibration.cpp:190-216); module.cpp:182-196 signature.
    All windows run as concurrent swarms on the device."""
    s = _settings(population, objective, bounds, particles, iters, inertia, cognitive, social, substeps)
    return fit_all_windows_settings(data, s, tau, delta, seed)


def fit_all_windows_settings(data: EpiSeries, s, tau: int = 35, delta: int = 3, seed: int = 0) -> FitAllResult:
    """fit_all_windows with an explicit sg_fit_settings."""
    ctx = context()
    population, substeps = s.population, s.substeps
    I, R, D = _series(data)
    n_max = max(1, 1 + (len(I) - 1 - tau) // max(delta, 1)) if len(I) > tau else 1
    recs = (_capi.sg_fit_record * n_max)()
    trajs = np.empty((n_max, tau + 1, 4))
    n_win, failed = ctypes.c_size_t(), ctypes.c_size_t()
    mean = ctypes.c_double()
    rc = _capi.lib().sg_fit_all_windows_series(ctx.handle, _capi._d(I), _capi._d(R), _capi._d(D), len(I), int(tau),
                                               int(delta), ctypes.byref(s), int(seed) & 0xFFFFFFFFFFFFFFFF, n_max,
                                               ctypes.byref(n_win), recs, _capi._d(trajs), ctypes.byref(mean),
                                               ctypes.byref(failed))
    if rc:
        raise_for_status(rc, _capi.lib().sg_last_error(ctx.handle).decode())
    fits = [_fit_from_record(recs[k], trajs[k], population, substeps) for k in range(n_win.value)]
    return FitAllResult(fits, float(mean.value), int(failed.value))


def forecast_extension(fit: FitResult, horizon: int, substeps: int = kDefaultSubsteps) -> Forecast:
    """forecast_extension (calibration.cpp:298-322) on the device."""
    if not fit.ok or fit.trajectory is None or fit.trajectory.days() == 0:
        raise Error("cannot extend a failed fit")
    if not fit.trajectory.finite:
        raise NonFiniteError()
    j = fit.trajectory.states[-1]
    states, fin = context().forecast_batch(fit.params.as_array()[None, :], [[j.S, j.I, j.R, j.D]],
                                           fit.trajectory.population, int(horizon), substeps)
    if not fin[0]:
        raise NonFiniteError()
    return Forecast(fit.window.last_day(), int(horizon),
                    Trajectory.from_array(states[0], fit.trajectory.population, True))


def stability_study(data: EpiSeries, window: Window, population: float, repetitions: int, horizon: int,
                    objective: str = "ird-mxse", bounds: str = "stage2", particles: int = 10000, iters: int = 100,
                    inertia: float = 0.5, cognitive: float = 0.5, social: float = 0.5, seed: int = 0,
                    substeps: int = kDefaultSubsteps) -> StabilityResult:
    """stability_study (calibration.cpp:378-436): repetitions run as concurrent swarms."""
    s = _settings(population, objective, bounds, particles, iters, inertia, cognitive, social, substeps)
    return stability_study_settings(data, window, s, repetitions, horizon, seed)


def stability_study_settings(data: EpiSeries, window: Window, s, repetitions: int, horizon: int,
                             seed: int = 0) -> StabilityResult:
    """stability_study with an explicit sg_fit_settings."""
    ctx = context()
    population, substeps = s.population, s.substeps
    I, R, D = _series(data)
    L, H = int(window.length), int(horizon)
    reps = max(int(repetitions), 1)
    recs = (_capi.sg_fit_record * reps)()
    sizes = [L, L, L + H, L + H, L + H]
    day_bands = np.empty(7 * sum(sizes))
    day_counts = np.empty(sum(sizes), dtype=np.uint64)
    scal = np.empty(14)
    scal_counts = np.empty(2, dtype=np.uint64)
    failed = ctypes.c_uint64()
    u64 = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))  # noqa: E731
    rc = _capi.lib().sg_stability_study_series(ctx.handle, _capi._d(I), _capi._d(R), _capi._d(D), len(I),
                                               int(window.start), L, ctypes.byref(s), int(repetitions), H,
                                               int(seed) & 0xFFFFFFFFFFFFFFFF, recs, _capi._d(day_bands),
                                               u64(day_counts), _capi._d(scal), u64(scal_counts),
                                               ctypes.byref(failed))
    if rc:
        raise_for_status(rc, _capi.lib().sg_last_error(ctx.handle).decode())
    bands, off, coff = [], 0, 0
    for n in sizes:
        rows = [day_bands[off + r * n: off + (r + 1) * n].tolist() for r in range(7)]
        bands.append(QuantileBands(day_counts[coff:coff + n].astype(int).tolist(), *rows))
        off += 7 * n
        coff += n
    sc = [ScalarBands(int(scal_counts[k]), *[float(v) for v in scal[7 * k:7 * k + 7]]) for k in range(2)]
    fits = [_fit_from_record(recs[k], None, population, substeps) for k in range(int(repetitions))]
    return StabilityResult(Window(window.index, window.start, window.length), H, int(repetitions),
                           int(failed.value), *bands, *sc, fits)
