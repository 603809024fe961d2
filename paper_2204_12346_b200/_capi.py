"""ctypes binding of the C-ABI in include/sirdgpu.h (libsirdgpu.so).

This is the Python side of the drop-in boundary; it holds no arithmetic.
The shared library is built in-tree by `paper_2204_12346_b200.build`
(`__graft_entry__.build()`); importing this module when it is missing raises
immediately — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import weakref
from pathlib import Path

import numpy as np

from .errors import NoDeviceError, raise_for_status

# SG_LIB overrides the library (tuning experiments only; the default is the in-tree build).
LIB_PATH = Path(os.environ.get("SG_LIB", Path(__file__).resolve().parent / "libsirdgpu.so"))

FAMILY = {"d": 0, "ird": 1}
METRIC = {"mxse": 0, "mse": 1, "mae": 2, "mape": 3}

_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)


class sg_state(ctypes.Structure):
    _fields_ = [("S", ctypes.c_double), ("I", ctypes.c_double), ("R", ctypes.c_double), ("D", ctypes.c_double)]


class sg_swarm_desc(ctypes.Structure):
    _fields_ = [
        ("window", ctypes.c_void_p),
        ("lower", ctypes.c_double * 6),
        ("upper", ctypes.c_double * 6),
        ("n_particles", ctypes.c_uint64),
        ("max_iters", ctypes.c_uint64),
        ("inertia", ctypes.c_double),
        ("cognitive", ctypes.c_double),
        ("social", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("repair_time_order", ctypes.c_int),
    ]


class sg_swarm_result(ctypes.Structure):
    _fields_ = [
        ("best_position", ctypes.c_double * 6),
        ("best_cost", ctypes.c_double),
        ("cost_history", _dp),
        ("status", ctypes.c_int),
    ]


class sg_fit_settings(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int), ("metric", ctypes.c_int),
                ("beta_lo", ctypes.c_double), ("beta_hi", ctypes.c_double),
                ("gamma_lo", ctypes.c_double), ("gamma_hi", ctypes.c_double),
                ("mu_lo", ctypes.c_double), ("mu_hi", ctypes.c_double),
                ("t_margin", ctypes.c_uint64), ("n_particles", ctypes.c_uint64), ("max_iters", ctypes.c_uint64),
                ("inertia", ctypes.c_double), ("cognitive", ctypes.c_double), ("social", ctypes.c_double),
                ("population", ctypes.c_double), ("substeps", ctypes.c_int)]


class sg_fit_record(ctypes.Structure):
    _fields_ = [("index", ctypes.c_uint64), ("start", ctypes.c_uint64), ("length", ctypes.c_uint64),
                ("params", ctypes.c_double * 6), ("objective", ctypes.c_double), ("r2_d", ctypes.c_double),
                ("ok", ctypes.c_int), ("status", ctypes.c_int), ("failure", ctypes.c_char * 192)]


_u64p = ctypes.POINTER(ctypes.c_uint64)
_szp = ctypes.POINTER(ctypes.c_size_t)

# Every symbol include/sirdgpu.h declares, with its ctypes signature.
SIGNATURES = {
    "sg_abi_version": (ctypes.c_int, []),
    "sg_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "sg_ctx_destroy": (None, [ctypes.c_void_p]),
    "sg_last_error": (ctypes.c_char_p, [ctypes.c_void_p]),
    "sg_ctx_launch_count": (ctypes.c_uint64, [ctypes.c_void_p]),
    "sg_ctx_stream": (ctypes.c_void_p, [ctypes.c_void_p]),
    "sg_ctx_copy_bytes": (None, [ctypes.c_void_p, _u64p, _u64p]),
    "sg_ctx_band_stats": (ctypes.c_int, [ctypes.c_void_p, _u64p, _u64p, _u64p]),
    "sg_window_create": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp, ctypes.c_int, sg_state, ctypes.c_double,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "sg_window_destroy": (None, [ctypes.c_void_p]),
    "sg_eval_costs": (ctypes.c_int, [ctypes.c_void_p, _dp, ctypes.c_size_t, ctypes.c_size_t, _dp]),
    "sg_eval_costs_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                            ctypes.c_void_p]),
    "sg_integrate_batch": (ctypes.c_int, [ctypes.c_void_p, _dp, ctypes.c_size_t, sg_state, ctypes.c_double,
                                          ctypes.c_int, ctypes.c_int, _dp, _u8p]),
    "sg_fit_swarms": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(sg_swarm_desc), ctypes.c_size_t,
                                     ctypes.POINTER(sg_swarm_result)]),
    "sg_plan_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(sg_swarm_desc), ctypes.c_size_t,
                                      ctypes.POINTER(ctypes.c_void_p)]),
    "sg_plan_run": (ctypes.c_int, [ctypes.c_void_p]),
    "sg_plan_run_timed": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp]),
    "sg_plan_step_launches": (ctypes.c_uint64, [ctypes.c_void_p]),
    "sg_plan_ramp_substeps": (ctypes.c_uint64, [ctypes.c_void_p]),
    "sg_plan_results": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(sg_swarm_result)]),
    "sg_plan_evals": (ctypes.c_uint64, [ctypes.c_void_p]),
    "sg_plan_destroy": (None, [ctypes.c_void_p]),
    "sg_probe_fp64_rate": (ctypes.c_int, [ctypes.c_void_p, _dp]),
    "sg_integrate_states": (ctypes.c_int, [ctypes.c_void_p, _dp, ctypes.POINTER(sg_state), ctypes.c_size_t,
                                           ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp, _u8p]),
    "sg_integrate_states_r2": (ctypes.c_int, [ctypes.c_void_p, _dp, ctypes.POINTER(sg_state), _dp, ctypes.c_size_t,
                                              ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp, _u8p, _dp]),
    "sg_fit_window_series": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp, ctypes.c_size_t, ctypes.c_uint64,
                                            ctypes.c_uint64, ctypes.POINTER(sg_fit_settings), ctypes.c_uint64,
                                            ctypes.POINTER(sg_fit_record), _dp, _dp]),
    "sg_fit_all_windows_series": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp, ctypes.c_size_t, ctypes.c_uint64,
                                                 ctypes.c_uint64, ctypes.POINTER(sg_fit_settings), ctypes.c_uint64,
                                                 ctypes.c_size_t, _szp, ctypes.POINTER(sg_fit_record), _dp, _dp,
                                                 _szp]),
    "sg_fit_window_range_series": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp, ctypes.c_size_t, ctypes.c_uint64,
                                                  ctypes.c_uint64, ctypes.POINTER(sg_fit_settings), ctypes.c_uint64,
                                                  ctypes.c_uint64, ctypes.c_uint64, _szp,
                                                  ctypes.POINTER(sg_fit_record), _dp]),
    "sg_stability_study_series": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, _dp, ctypes.c_size_t, ctypes.c_uint64,
                                                 ctypes.c_uint64, ctypes.POINTER(sg_fit_settings), ctypes.c_uint64,
                                                 ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(sg_fit_record),
                                                 _dp, _u64p, _dp, _u64p, _u64p]),
    "sg_gswarm_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _dp, _dp, ctypes.c_uint64, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_uint64, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_void_p)]),
    "sg_gswarm_destroy": (None, [ctypes.c_void_p]),
    "sg_gswarm_positions_device": (ctypes.c_void_p, [ctypes.c_void_p]),
    "sg_gswarm_costs_device": (ctypes.c_void_p, [ctypes.c_void_p]),
    "sg_gswarm_get_positions": (ctypes.c_int, [ctypes.c_void_p, _dp]),
    "sg_gswarm_set_positions": (ctypes.c_int, [ctypes.c_void_p, _dp]),
    "sg_gswarm_set_initial_positions": (ctypes.c_int, [ctypes.c_void_p, _dp]),
    "sg_gswarm_set_costs": (ctypes.c_int, [ctypes.c_void_p, _dp]),
    "sg_gswarm_eval_window": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "sg_gswarm_step": (ctypes.c_int, [ctypes.c_void_p, _dp]),
    "sg_gswarm_best": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp]),
    "sg_objective_values": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp,
                                           ctypes.c_size_t, _dp, _u8p, ctypes.c_size_t, _dp]),
    "sg_metric_values": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, _dp, _dp, ctypes.c_size_t, ctypes.c_size_t,
                                        _dp]),
    "sg_sird_rhs_batch": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(sg_state), _dp, _dp, _dp, ctypes.c_double,
                                         ctypes.c_size_t, ctypes.POINTER(sg_state)]),
    "sg_forecast_batch": (ctypes.c_int, [ctypes.c_void_p, _dp, ctypes.POINTER(sg_state), ctypes.c_size_t,
                                         ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp, _u8p]),
    "sg_forecast_ensemble": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, ctypes.c_uint64, ctypes.c_size_t,
                                            ctypes.c_int, _dp, _dp, _dp]),
    "sg_forecast_ensemble_bands": (ctypes.c_int, [ctypes.c_void_p, _dp, _dp, ctypes.c_uint64, ctypes.c_size_t,
                                                  ctypes.c_int, _dp, _u64p, _dp]),
    "sg_quantile_bands": (ctypes.c_int, [ctypes.c_void_p, _dp, ctypes.c_size_t, ctypes.c_int, _dp, _u64p]),
    "sg_forecast_ensemble_bands_batch": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_size_t, _dp, _dp,
                                                        _u64p, ctypes.c_size_t, ctypes.c_int, _dp, _u64p]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libsirdgpu.so (raises FileNotFoundError if it was never built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise FileNotFoundError(
                f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the engine has no CPU fallback)")
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            if "SG_LIB" in os.environ and not hasattr(handle, name):
                continue  # A/B against an older build (diagnostics only)
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    return out.reshape(shape) if shape is not None else out


def parse_spec(spec) -> tuple[int, int]:
    """'ird-mxse' -> (1, 0); parse_objective (objectives.cpp:146-170)."""
    if isinstance(spec, tuple):
        return spec
    from .errors import Error
    name = str(spec)
    if name.startswith("d-"):
        fam, met = 0, name[2:]
    elif name.startswith("ird-"):
        fam, met = 1, name[4:]
    else:
        raise Error(f"unknown objective '{name}'")
    if met not in METRIC:
        raise Error(f"unknown objective '{name}'")
    return fam, METRIC[met]


class Context:
    """One engine context on one device (sg_ctx)."""

    def __init__(self, device: int = 0):
        L = lib()
        h = ctypes.c_void_p()
        rc = L.sg_ctx_create(int(device), ctypes.byref(h))
        if rc == 7:
            raise NoDeviceError(f"no sm_100 device at index {device}")
        raise_for_status(rc, "sg_ctx_create failed")
        self._h = h
        self.device = device
        # windows and plans of this context: destroyed before it (include/sirdgpu.h rule)
        self._children = weakref.WeakSet()

    def _adopt(self, child) -> None:
        self._children.add(child)

    @property
    def handle(self):
        return self._h

    def check(self, rc: int) -> None:
        if rc:
            raise_for_status(rc, lib().sg_last_error(self._h).decode())

    @property
    def launch_count(self) -> int:
        return int(lib().sg_ctx_launch_count(self._h))

    @property
    def copy_bytes(self) -> tuple[int, int]:
        """(host->device, device->host) bytes this context has copied so far."""
        a, b = ctypes.c_uint64(), ctypes.c_uint64()
        lib().sg_ctx_copy_bytes(self._h, ctypes.byref(a), ctypes.byref(b))
        return int(a.value), int(b.value)

    @property
    def band_stats(self) -> tuple[int, int, int]:
        """(days resolved from the ensemble's fused histogram, days that took
        the histogram pass, ramp substeps evaluated) over this context's band
        calls so far."""
        a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        self.check(lib().sg_ctx_band_stats(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return int(a.value), int(b.value), int(c.value)

    @property
    def stream(self) -> int:
        return int(lib().sg_ctx_stream(self._h) or 0)

    def close(self) -> None:
        if getattr(self, "_h", None):
            for child in list(getattr(self, "_children", ())):
                child.close()
            lib().sg_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- integrator ---------------------------------------------------------------
    def integrate_batch(self, params, init, population: float, n_days: int, substeps: int = 24):
        """integrate_batch (model.cpp:116-125): -> (states n x n_days x 4, finite n)."""
        p = _f64(params).reshape(-1, 6)
        n = p.shape[0]
        states = np.empty((n, n_days, 4))
        fin = np.empty(n, dtype=np.uint8)
        s = sg_state(*[float(v) for v in init])
        self.check(lib().sg_integrate_batch(self._h, _d(p), n, s, float(population), int(n_days), int(substeps),
                                            _d(states), fin.ctypes.data_as(_u8p)))
        return states, fin.astype(bool)

    def forecast_batch(self, params, junctions, population: float, horizon: int, substeps: int = 24):
        """forecast_extension's integration (calibration.cpp:305-317), batched."""
        p = _f64(params).reshape(-1, 6)
        j = _f64(junctions).reshape(-1, 4)
        n = p.shape[0]
        states = np.empty((n, horizon + 1, 4))
        fin = np.empty(n, dtype=np.uint8)
        self.check(lib().sg_forecast_batch(self._h, _d(p), j.ctypes.data_as(ctypes.POINTER(sg_state)), n,
                                           float(population), int(horizon), int(substeps), _d(states),
                                           fin.ctypes.data_as(_u8p)))
        return states, fin.astype(bool)

    # -- swarms -------------------------------------------------------------------
    def quantile_bands(self, values):
        """build_quantile_bands on the device: values n_days x n (day-major) ->
        (bands 7 x n_days, counts n_days)."""
        v = _f64(values)
        if v.ndim != 2:
            raise ValueError("values must be 2-D (days x values)")
        n_days, n = v.shape
        bands = np.zeros((7, n_days))
        counts = np.zeros(n_days, dtype=np.uint64)
        self.check(lib().sg_quantile_bands(self._h, _d(v), n, n_days, _d(bands), counts.ctypes.data_as(_u64p)))
        return bands, counts

    def forecast_ensemble_bands_batch(self, windows, lower, upper, seeds, n: int, horizon: int):
        """sg_forecast_ensemble_bands for many windows in one pipelined call:
        -> (bands n_windows x 7 x (horizon+1), counts n_windows x (horizon+1))."""
        w = len(windows)
        handles = (ctypes.c_void_p * w)(*[x.handle.value for x in windows])
        lo, hi = _f64(lower), _f64(upper)
        sd = np.ascontiguousarray([int(x) & 0xFFFFFFFFFFFFFFFF for x in seeds], dtype=np.uint64)
        bands = np.empty((w, 7, horizon + 1))
        counts = np.empty((w, horizon + 1), dtype=np.uint64)
        self.check(lib().sg_forecast_ensemble_bands_batch(handles, w, _d(lo), _d(hi), sd.ctypes.data_as(_u64p), n,
                                                          int(horizon), _d(bands), counts.ctypes.data_as(_u64p)))
        return bands, counts

    def fit_swarms(self, swarms: list[dict]):
        """sg_fit_swarms: each dict has window, lower, upper, n_particles, max_iters,
        inertia, cognitive, social, seed, repair.  Returns list of
        (status, best[6], best_cost, history)."""
        n = len(swarms)
        descs = _descs(swarms)
        res = (sg_swarm_result * n)()
        hists = []
        for k, s in enumerate(swarms):
            h = np.zeros(max(int(s["max_iters"]), 1))
            hists.append(h)
            res[k].cost_history = _d(h)
        self.check(lib().sg_fit_swarms(self._h, descs, n, res))
        return [(int(res[k].status), np.array(res[k].best_position[:]), float(res[k].best_cost), hists[k])
                for k in range(n)]


class Window:
    """sg_window: the device-side BatchObjective of one calibration window."""

    def __init__(self, ctx: Context, infectious, recovered_cum, deaths_cum, init, population: float,
                 spec="ird-mxse", substeps: int = 24):
        self.ctx = ctx
        self.I = _f64(infectious)
        self.R = _f64(recovered_cum)
        self.D = _f64(deaths_cum)
        self.family, self.metric = parse_spec(spec)
        self.population = float(population)
        self.substeps = int(substeps)
        self.n_days = len(self.I)
        self.init = tuple(float(v) for v in init)
        h = ctypes.c_void_p()
        ctx.check(lib().sg_window_create(ctx.handle, _d(self.I), _d(self.R), _d(self.D), self.n_days,
                                         sg_state(*self.init), self.population, self.substeps, self.family,
                                         self.metric, ctypes.byref(h)))
        self._h = h
        ctx._adopt(self)

    @property
    def handle(self):
        return self._h

    def eval_costs(self, positions) -> np.ndarray:
        """The BatchObjective call (calibration.cpp:140-154) on host buffers."""
        pos = _f64(positions)
        n = pos.size // 6 if pos.ndim == 1 else pos.shape[0]
        dim = 6 if pos.ndim == 1 else pos.shape[1]
        costs = np.empty(n)
        self.ctx.check(lib().sg_eval_costs(self._h, _d(pos), n, dim, _d(costs)))
        return costs

    def eval_costs_device(self, d_positions_ptr: int, n: int, d_costs_ptr: int, stream: int = 0) -> None:
        self.ctx.check(lib().sg_eval_costs_device(self._h, ctypes.c_void_p(d_positions_ptr), n,
                                                  ctypes.c_void_p(d_costs_ptr), ctypes.c_void_p(stream or None)))

    def forecast_ensemble(self, lower, upper, seed: int, n: int, horizon: int, want_costs=True, want_params=True):
        lo, hi = _f64(lower), _f64(upper)
        costs = np.empty(n) if want_costs else None
        params = np.empty((n, 6)) if want_params else None
        deaths = np.empty((n, horizon + 1))
        self.ctx.check(lib().sg_forecast_ensemble(self._h, _d(lo), _d(hi), int(seed) & 0xFFFFFFFFFFFFFFFF, n,
                                                  int(horizon), _d(costs) if costs is not None else None,
                                                  _d(params) if params is not None else None, _d(deaths)))
        return costs, params, deaths

    def forecast_ensemble_bands(self, lower, upper, seed: int, n: int, horizon: int, want_costs=False):
        """Per-day quantile bands of the ensemble's forecast deaths, computed on the device:
        -> (bands 7 x (horizon+1): median, p50_lo, p50_hi, p90_lo, p90_hi, p95_lo, p95_hi;
            counts (horizon+1); costs or None)."""
        lo, hi = _f64(lower), _f64(upper)
        bands = np.empty((7, horizon + 1))
        counts = np.empty(horizon + 1, dtype=np.uint64)
        costs = np.empty(n) if want_costs else None
        self.ctx.check(lib().sg_forecast_ensemble_bands(self._h, _d(lo), _d(hi), int(seed) & 0xFFFFFFFFFFFFFFFF, n,
                                                        int(horizon), _d(bands), counts.ctypes.data_as(_u64p),
                                                        _d(costs) if costs is not None else None))
        return bands, counts, costs

    def close(self):
        if getattr(self, "_h", None):
            lib().sg_window_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _descs(swarms: list[dict]):
    n = len(swarms)
    descs = (sg_swarm_desc * n)()
    for k, s in enumerate(swarms):
        d = descs[k]
        d.window = s["window"].handle
        d.lower[:] = [float(v) for v in s["lower"]]
        d.upper[:] = [float(v) for v in s["upper"]]
        d.n_particles = int(s["n_particles"])
        d.max_iters = int(s["max_iters"])
        d.inertia = float(s.get("inertia", 0.5))
        d.cognitive = float(s.get("cognitive", 0.5))
        d.social = float(s.get("social", 0.5))
        d.seed = int(s.get("seed", 0)) & 0xFFFFFFFFFFFFFFFF
        d.repair_time_order = 1 if s.get("repair", True) else 0
    return descs


class Plan:
    """sg_plan: set up once, run (asynchronously, on the context stream) many times."""

    def __init__(self, ctx: Context, swarms: list[dict]):
        self.ctx = ctx
        self.swarms = swarms
        self._descs = _descs(swarms)
        h = ctypes.c_void_p()
        ctx.check(lib().sg_plan_create(ctx.handle, self._descs, len(swarms), ctypes.byref(h)))
        self._h = h
        ctx._adopt(self)

    @property
    def evals(self) -> int:
        return int(lib().sg_plan_evals(self._h))

    def run(self) -> None:
        self.ctx.check(lib().sg_plan_run(self._h))

    def run_timed(self) -> tuple[float, float]:
        """Synchronous run; returns (seed_ms, steps_ms) from CUDA events on the context stream."""
        a, b = ctypes.c_double(), ctypes.c_double()
        self.ctx.check(lib().sg_plan_run_timed(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    @property
    def ramp_substeps(self) -> int:
        """Ramp substeps evaluated by the last run (R_ramp of the algorithmic op count)."""
        return int(lib().sg_plan_ramp_substeps(self._h))

    @property
    def step_launches(self) -> int:
        return int(lib().sg_plan_step_launches(self._h))

    def results(self):
        n = len(self.swarms)
        res = (sg_swarm_result * n)()
        hists = []
        for k, s in enumerate(self.swarms):
            h = np.zeros(max(int(s["max_iters"]), 1))
            hists.append(h)
            res[k].cost_history = _d(h)
        self.ctx.check(lib().sg_plan_results(self._h, res))
        return [(int(res[k].status), np.array(res[k].best_position[:]), float(res[k].best_cost), hists[k])
                for k in range(n)]

    def close(self):
        if getattr(self, "_h", None):
            lib().sg_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def probe_fp64_rate(ctx: Context) -> float:
    out = ctypes.c_double(0.0)
    ctx.check(lib().sg_probe_fp64_rate(ctx.handle, ctypes.byref(out)))
    return float(out.value)
