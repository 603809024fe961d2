"""The drop-in boundary without a GPU: libsirdgpu.so loads and exports every
symbol include/sirdgpu.h declares; argument validation and status mapping
work; compute entry points fail loudly when there is no sm_100 device (no
CPU fallback).  Host-only helpers of the Python mirror match the reference.
"""
import ctypes
import math
import re
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "sirdgpu.h"


def declared_symbols():
    text = HEADER.read_text()
    decl = r"^(?:int|void|uint64_t|const char\s*\*|void\s*\*|const double\s*\*|double\s*\*)\s*\*?\s*(sg_[a-z0-9_]+)\s*\("
    return sorted(set(re.findall(decl, text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2204_12346_b200 import _capi
    lib = _capi.lib()
    names = declared_symbols()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_capi.SIGNATURES), set(names) ^ set(_capi.SIGNATURES)
    nm = subprocess.run(["nm", "-D", "--defined-only", str(_capi.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sg_[a-z0-9_]+)$", nm, re.M))
    assert set(names) <= exported


def test_abi_version_and_null_arguments():
    from paper_2204_12346_b200 import _capi
    lib = _capi.lib()
    assert lib.sg_abi_version() == 1
    assert lib.sg_ctx_create(0, None) == 1
    assert lib.sg_eval_costs(None, None, 0, 6, None) == 1
    assert lib.sg_fit_swarms(None, None, 0, None) == 1
    assert lib.sg_ctx_launch_count(None) == 0
    assert lib.sg_last_error(None) == b"null context"
    lib.sg_ctx_destroy(None)
    lib.sg_window_destroy(None)
    lib.sg_plan_destroy(None)


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2204_12346_b200 as eng
    with pytest.raises(eng.errors.NoDeviceError):
        eng.Context(0)


def test_status_codes_map_to_reference_exceptions():
    from paper_2204_12346_b200 import errors
    cases = {1: errors.Error, 2: errors.SchemeError, 3: errors.InsufficientPopulationError,
             4: errors.AllInfeasibleError, 5: errors.NonFiniteError, 6: errors.DeviceError, 8: errors.DeviceError}
    for code, cls in cases.items():
        with pytest.raises(cls):
            errors.raise_for_status(code, "x")
    errors.raise_for_status(0)
    assert issubclass(errors.SchemeError, errors.Error) and issubclass(errors.NoDeviceError, errors.DeviceError)


def test_objective_names_parse_like_the_reference():
    from paper_2204_12346_b200 import _capi, errors
    assert _capi.parse_spec("ird-mxse") == (1, 0)
    assert _capi.parse_spec("d-mape") == (0, 3)
    for bad in ("mxse", "ird-max", "x-mse", ""):
        with pytest.raises(errors.Error):
            _capi.parse_spec(bad)


def test_make_windows_matches_brute_force():
    """acceptance/main.cpp:210-235 / test_calibration.cpp:36-75."""
    from paper_2204_12346_b200 import errors, sirdfit
    assert len(sirdfit.make_windows(450, 35, 3)) == 139
    rng = np.random.default_rng(2024)
    for _ in range(200):
        tau, delta = int(rng.integers(1, 51)), int(rng.integers(1, 11))
        n = tau + 1 + int(rng.integers(0, 150))
        starts = list(range(0, n - tau, delta))
        ws = sirdfit.make_windows(n, tau, delta)
        assert [w.start for w in ws] == starts and all(w.length == tau + 1 for w in ws)
    for args in ((35, 35, 3), (100, 0, 3), (100, 5, 0)):
        with pytest.raises(errors.SchemeError):
            sirdfit.make_windows(*args)


def test_host_helpers_match_reference(port):
    from paper_2204_12346_b200 import errors, sirdfit
    for base, idx in ((0, 0), (1, 1), (2204, 138), (2**64 - 1, 5)):
        assert sirdfit.mix_seed(base, idx) == port.mix_seed(base, idx)
    p = sirdfit.SirdParams(0.6, 0.9, 15.0, 30.0, 0.09, 0.012)
    assert sirdfit.beta_at(p, 0.0) == 0.6 and sirdfit.beta_at(p, 35.0) == 0.9
    assert sirdfit.beta_at(p, 22.5) == pytest.approx(0.75)
    assert sirdfit.basic_reproduction_number(0.5, 0.1, 0.01) == pytest.approx(0.5 / 0.11)
    with pytest.raises(errors.DegenerateRatesError):
        sirdfit.basic_reproduction_number(0.5, 0.0, 0.0)
    with pytest.raises(errors.ConstantObservedError):
        sirdfit.r_squared_d([1.0, 1.0], [1.0, 2.0])
    assert sirdfit.r_squared_d([1.0, 2.0, 4.0], [1.0, 2.0, 4.0]) == 1.0


def test_cpp_api_header_is_self_contained():
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ missing")
    src = f'#include "sirdfit_b200.hpp"\nint main() {{ sirdfit_b200::FitSettings s; return (int)s.pso.n_particles; }}\n'
    r = subprocess.run([gxx, "-std=c++20", "-fsyntax-only", f"-I{ROOT / 'include'}", "-x", "c++", "-"], input=src,
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run(["gcc", "-std=c11", "-fsyntax-only", f"-I{ROOT / 'include'}", "-x", "c", "-"],
                       input='#include "sirdgpu.h"\nint main(void) { return SG_ABI_VERSION - 1; }\n',
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
