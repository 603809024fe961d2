"""ctypes loader for the CPU oracles (TEST INFRASTRUCTURE — see oracle/oracle.h).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm import this module, as the checker.  The product package never does.

    load("port")       -> oracle/libsirdoracle.so (C restatement)
    load("reference")  -> oracle/_ref/libsirdref.so (the reference itself)
    load("hybrid")     -> oracle/_ref/libsirdhybrid.so: the reference's own
                          Swarm driving the GPU objective through the C-ABI
                          (the drop-in under test)

build("refcallers") also builds the reference's own callers (doctest unit
suite, acceptance harness, pybind module, CLI — the first and last against
the stand-in headers in oracle/doctest_standin and oracle/cli11_standin)
against the unmodified reference and against ref_binding/ (INTEGRATION.md
§2) into oracle/_ref/.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

ORACLE_DIR = Path(__file__).resolve().parent
PORT_SO = ORACLE_DIR / "libsirdoracle.so"
REF_SO = ORACLE_DIR / "_ref" / "libsirdref.so"
HYBRID_SO = ORACLE_DIR / "_ref" / "libsirdhybrid.so"
ENGINE_SO = ORACLE_DIR.parent / "paper_2204_12346_b200" / "libsirdgpu.so"
REFERENCE_SRC = Path("/root/reference/proj")

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_szp = ctypes.POINTER(ctypes.c_size_t)

FAMILIES = {"d": 0, "ird": 1}
METRICS = {"mxse": 0, "mse": 1, "mae": 2, "mape": 3}
SPECS = [f"{f}-{m}" for f in FAMILIES for m in METRICS]


def parse_spec(name: str) -> tuple[int, int]:
    fam, met = name.split("-")
    return FAMILIES[fam], METRICS[met]


def build(kind: str = "all") -> None:
    """Compile the oracle(s) with oracle/Makefile.  `ref` needs /root/reference."""
    targets = []
    if kind in ("all", "port"):
        targets.append("port")
    if kind in ("all", "ref", "reference") and REFERENCE_SRC.exists():
        targets.append("ref")
    if kind in ("all", "hybrid") and REFERENCE_SRC.exists() and ENGINE_SO.exists():
        targets.append("hybrid")
    if kind in ("all", "refcallers") and REFERENCE_SRC.exists() and ENGINE_SO.exists():
        targets.append("refcallers")
    if targets:
        subprocess.run(["make", "-s", "-j", str(min(16, os.cpu_count() or 1)), "-C", str(ORACLE_DIR), *targets],
                       check=True)


_FIT_SWARM_ARGS = [ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, ctypes.c_int, _dp, ctypes.c_double, ctypes.c_int,
                   ctypes.c_int, _dp, _dp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                   ctypes.c_double, ctypes.c_uint64, ctypes.c_int, _dp, _dp, _dp]


def _d(a):
    return a.ctypes.data_as(_dp)


class Oracle:
    def __init__(self, path: Path, kind: str):
        self.kind = kind
        self.path = path
        lib = ctypes.CDLL(str(path), mode=ctypes.RTLD_LOCAL)
        self.lib = lib
        if kind == "hybrid":
            lib.hybrid_fit_swarm.argtypes = _FIT_SWARM_ARGS
            self._fit_swarm = lib.hybrid_fit_swarm
            return
        self._fit_swarm = lib.oracle_fit_swarm
        lib.oracle_mix_seed.restype = ctypes.c_uint64
        lib.oracle_mix_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        lib.oracle_mt_raw.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_size_t, _u64p]
        lib.oracle_uniform01.argtypes = [ctypes.c_uint64, ctypes.c_size_t, _dp]
        lib.oracle_integrate.argtypes = [_dp, _dp, ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp, _ip]
        lib.oracle_eval_costs.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, ctypes.c_int, _dp,
                                          ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp, ctypes.c_size_t, _dp]
        lib.oracle_fit_swarm.argtypes = _FIT_SWARM_ARGS
        lib.oracle_forecast.argtypes = [_dp, _dp, ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp, _ip]
        if kind == "reference":
            lib.ref_last_error.restype = ctypes.c_char_p
            lib.ref_fit_window.argtypes = [_dp, _dp, _dp, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t,
                                           ctypes.c_int, ctypes.c_int, _dp, ctypes.c_double, ctypes.c_int,
                                           ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_uint64, _dp, _dp, _dp,
                                           _dp, _ip]
            lib.ref_fit_all_windows.argtypes = [_dp, _dp, _dp, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t,
                                                ctypes.c_int, ctypes.c_int, _dp, ctypes.c_double, ctypes.c_int,
                                                ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double,
                                                ctypes.c_double, ctypes.c_double, ctypes.c_uint64, ctypes.c_size_t,
                                                _szp, _ip, _dp, _dp, _dp, _dp, _szp]
            lib.ref_clean_series.argtypes = [_dp, _dp, _dp, ctypes.c_size_t, ctypes.c_int, _dp, _dp, _dp, _dp]
            lib.ref_quantile_bands.argtypes = [_dp, ctypes.c_size_t, ctypes.c_size_t, _dp, _szp]
            lib.ref_stability_study.argtypes = [_dp, _dp, _dp, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t,
                                                ctypes.c_int, ctypes.c_int, _dp, ctypes.c_double, ctypes.c_int,
                                                ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                                ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                                _ip, _dp, _dp, _dp, _u64p, _dp, _u64p, _u64p]
            lib.ref_format_double.argtypes = [ctypes.c_double, ctypes.c_char_p]
            lib.ref_clean_raw.argtypes = [_ip, _dp, _dp, _dp, ctypes.c_size_t, ctypes.c_int, ctypes.c_size_t, _dp,
                                          _dp, _dp, _dp, _szp, _u64p]
            lib.ref_build_envelope.argtypes = [_dp, ctypes.c_size_t, ctypes.c_size_t, _dp, _szp]
            lib.ref_fit_window_forecast.argtypes = [_dp, _dp, _dp, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t,
                                                    ctypes.c_int, ctypes.c_int, _dp, ctypes.c_double, ctypes.c_int,
                                                    ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                                    ctypes.c_uint64, _dp]

    # -- streams --------------------------------------------------------------
    def mix_seed(self, base: int, index: int) -> int:
        return int(self.lib.oracle_mix_seed(base, index))

    def mt_raw(self, seed: int, n: int, skip: int = 0) -> np.ndarray:
        out = np.zeros(n, dtype=np.uint64)
        self.lib.oracle_mt_raw(seed, skip, n, out.ctypes.data_as(_u64p))
        return out

    def uniform01(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.float64)
        self.lib.oracle_uniform01(seed, n, _d(out))
        return out

    # -- integrator / objective -------------------------------------------------
    def integrate(self, params, init, population, n_days, substeps=24):
        p = np.ascontiguousarray(params, dtype=np.float64)
        i = np.ascontiguousarray(init, dtype=np.float64)
        states = np.zeros((n_days, 4), dtype=np.float64)
        fin = ctypes.c_int(0)
        rc = self.lib.oracle_integrate(_d(p), _d(i), population, n_days, substeps, _d(states), ctypes.byref(fin))
        if rc:
            raise ValueError(f"oracle_integrate status {rc}")
        return states, bool(fin.value)

    def eval_costs(self, spec, I, R, D, init, population, positions, substeps=24, n_threads=1):
        fam, met = parse_spec(spec) if isinstance(spec, str) else spec
        I, R, D = (np.ascontiguousarray(a, dtype=np.float64) for a in (I, R, D))
        init = np.ascontiguousarray(init, dtype=np.float64)
        pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 6)
        costs = np.zeros(pos.shape[0], dtype=np.float64)
        rc = self.lib.oracle_eval_costs(fam, met, _d(I), _d(R), _d(D), len(I), _d(init), population, substeps,
                                        n_threads, _d(pos), pos.shape[0], _d(costs))
        if rc:
            raise ValueError(f"oracle_eval_costs status {rc}")
        return costs

    def fit_swarm(self, spec, I, R, D, init, population, lower, upper, n_particles, max_iters,
                  inertia=0.5, cognitive=0.5, social=0.5, seed=0, repair=True, substeps=24, n_threads=1):
        fam, met = parse_spec(spec) if isinstance(spec, str) else spec
        I, R, D = (np.ascontiguousarray(a, dtype=np.float64) for a in (I, R, D))
        init = np.ascontiguousarray(init, dtype=np.float64)
        lo = np.ascontiguousarray(lower, dtype=np.float64)
        hi = np.ascontiguousarray(upper, dtype=np.float64)
        best = np.zeros(6)
        cost = np.zeros(1)
        hist = np.zeros(max_iters)
        rc = self._fit_swarm(fam, met, _d(I), _d(R), _d(D), len(I), _d(init), population, substeps,
                                       n_threads, _d(lo), _d(hi), n_particles, max_iters, inertia, cognitive,
                                       social, seed, 1 if repair else 0, _d(best), _d(cost), _d(hist))
        return rc, best, float(cost[0]), hist

    def forecast(self, params, junction, population, horizon, substeps=24):
        p = np.ascontiguousarray(params, dtype=np.float64)
        j = np.ascontiguousarray(junction, dtype=np.float64)
        states = np.zeros((horizon + 1, 4))
        fin = ctypes.c_int(0)
        rc = self.lib.oracle_forecast(_d(p), _d(j), population, horizon, substeps, _d(states), ctypes.byref(fin))
        if rc:
            raise ValueError(f"oracle_forecast status {rc}")
        return states, bool(fin.value)


_cache: dict[str, Oracle] = {}


def load(kind: str = "port") -> Oracle:
    """Load an oracle; kind "port" (C restatement) or "reference" (oracle/_ref)."""
    if kind not in _cache:
        path = {"port": PORT_SO, "reference": REF_SO, "hybrid": HYBRID_SO}[kind]
        if not path.exists():
            build({"port": "port", "reference": "ref", "hybrid": "hybrid"}[kind])
        if not path.exists():
            raise FileNotFoundError(f"oracle library {path} is not built")
        _cache[kind] = Oracle(path, kind)
    return _cache[kind]


def reference_available() -> bool:
    return REF_SO.exists() or REFERENCE_SRC.exists()
