"""CPU-side checks of the reference-side binding (ref_binding/, INTEGRATION.md
§2): the reference's own callers link against libsirdgpu.so, and the host-only
parts of the bound API answer like the reference without a GPU."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref"


def _need(*paths):
    for p in paths:
        if not p.exists():
            pytest.skip(f"{p} not built (oracle/Makefile refcallers needs /root/reference)")


@pytest.mark.parametrize("binary", ["acceptance_b200", "api_parity", "sirdfit_cli_b200", "unit_tests_b200",
                                    "py_b200/sirdfit/_core"])
def test_binding_links_the_engine(binary):
    path = REF / binary
    if binary.endswith("_core"):
        _need(REF / "py_b200" / "sirdfit")
        cands = list((REF / "py_b200" / "sirdfit").glob("_core*.so"))
        if not cands:
            pytest.skip("pybind module not built")
        path = cands[0]
    _need(path)
    ldd = subprocess.run(["ldd", str(path)], capture_output=True, text=True).stdout
    assert "libsirdgpu.so" in ldd and "not found" not in ldd, ldd


def test_acceptance_window_criterion_on_host_parts():
    """Criterion 5 (make_windows vs brute-force enumeration) needs no device:
    the bound make_windows answers on the CPU exactly like the reference."""
    _need(REF / "acceptance_ref", REF / "acceptance_b200")
    a = subprocess.run([str(REF / "acceptance_ref"), "5"], capture_output=True, text=True, timeout=300)
    b = subprocess.run([str(REF / "acceptance_b200"), "5"], capture_output=True, text=True, timeout=300)
    assert a.returncode == b.returncode == 0 and a.stdout == b.stdout, (a.stdout, b.stdout)


def test_python_module_imports_and_answers_host_calls():
    _need(REF / "py_b200" / "sirdfit" / "__init__.py")
    code = ("import sirdfit; w = sirdfit.make_windows(450, tau=35, delta=3); "
            "print(len(w), w[-1].start, sirdfit.basic_reproduction_number(0.5, 0.1, 0.01))")
    outs = []
    for pkg in ("py_b200", "py_ref"):
        env = dict(os.environ, PYTHONPATH=str(REF / pkg))
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env)
        assert r.returncode == 0, r.stderr
        outs.append(r.stdout)
    assert outs[0] == outs[1] and outs[0].startswith("139 414")


def test_reference_cli_builds_with_the_standin_and_passes_acceptance_4_and_8_on_cpu():
    """The CLI11 stand-in (oracle/cli11_standin) compiles the reference's
    unmodified tools/main.cpp; on the pure reference, acceptance #4
    (byte-identical fits.json for 1 vs max threads) and #8 (band nesting)
    pass — the baseline the engine build is compared against on the GPU."""
    _need(REF / "acceptance_ref", REF / "sirdfit_cli_ref")
    for c in ("4", "8"):
        r = subprocess.run([str(REF / "acceptance_ref"), c, "--cli", str(REF / "sirdfit_cli_ref")], capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr
    r = subprocess.run([str(REF / "sirdfit_cli_b200"), "fit", "--population", "1000"], capture_output=True, text=True)
    assert r.returncode != 0 and "--input is required" in r.stderr


def test_reference_unit_suite_builds_with_the_standin_and_passes_on_cpu():
    """The doctest stand-in (oracle/doctest_standin) compiles the reference's
    unmodified unit tests; on the pure reference all 73 test cases pass (the
    engine build of the same suite runs in tests/test_gpu_refbinding.py)."""
    exe = REF / "unit_tests_ref"
    _need(exe)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "[doctest] test cases: 73 | 73 passed | 0 failed" in r.stdout, r.stdout[-500:]
