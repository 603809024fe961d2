"""Boundary 2 driven by the reference's OWN callers (VERDICT r01 "missing 1").

ref_binding/ replaces the reference's src/model.cpp, src/objectives.cpp and
src/calibration.cpp with bindings over the B200 engine;
oracle/Makefile `refcallers` builds the reference's unmodified callers twice —
against the pure reference and against the binding:

  * tests/acceptance/main.cpp (the reference's acceptance gate)
    criteria 1-9 must PASS on the engine with the same detail
    text as the pure reference (timings stripped: every number they print —
    population drift, Euler halving ratios, R^2 of the self-consistency fits,
    8-spec bound comparison, forecast coverage — comes out bit-identical);
    criterion 10 times CPU thread scaling of the objective (4 threads vs 1)
    and cannot pass on a device that ignores n_threads, so it is checked for
    what it can show: the device objective beats the reference's 1-thread time.
  * bindings/module.cpp as the pybind module `sirdfit._core` + the reference's
    python/sirdfit/__init__.py: the reference's tests/python/test_smoke.py
    passes on the engine (its two CLI cases included), and fit/forecast
    values equal the pure-reference module's bit for bit.
  * tests/test_*.cpp, the reference's doctest unit suite (built against
    oracle/doctest_standin): 73 test cases pass on the engine as on the pure
    reference.
  * tools/main.cpp, the `sirdfit` CLI (built against oracle/cli11_standin:
    the reference does not ship its vendored CLI11): acceptance #4 and #8
    drive it, and every output file of preprocess / fit / compare / forecast
    / stability is byte-identical to the pure-reference CLI's."""
import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref"
ACC_REF, ACC_B200 = REF / "acceptance_ref", REF / "acceptance_b200"
CLI_REF, CLI_B200 = REF / "sirdfit_cli_ref", REF / "sirdfit_cli_b200"
SMOKE = REF / "proj" / "tests" / "python" / "test_smoke.py"

pytestmark = pytest.mark.gpu

CRITERIA = [1, 2, 3, 4, 5, 6, 7, 8, 9]


def _acc_args(exe, criterion):
    cli = CLI_B200 if exe == ACC_B200 else CLI_REF
    return [str(exe), str(criterion)] + (["--cli", str(cli)] if criterion in (4, 8) else [])


def _need(*paths):
    for p in paths:
        if not p.exists():
            pytest.skip(f"{p} not built (oracle/Makefile refcallers needs /root/reference)")


def _strip_times(detail):
    # ", 1.234 s" / "(0.1 s vs 0.2 s)" timings are the only run-dependent text
    return re.sub(r"[-+0-9.e]+ s\b", "<t> s", detail)


@pytest.fixture(scope="module")
def reference_outcomes():
    _need(ACC_REF, CLI_REF)
    procs = {c: subprocess.Popen(_acc_args(ACC_REF, c), stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for c in CRITERIA if c not in (4, 8)}
    procs.update({c: subprocess.Popen(_acc_args(ACC_REF, c), stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                      text=True) for c in (4, 8)})
    out = {}
    for c, p in procs.items():
        so, se = p.communicate(timeout=900)
        out[c] = (p.returncode, so.strip())
    return out


@pytest.mark.parametrize("criterion", CRITERIA)
def test_acceptance_criterion_on_engine(criterion, reference_outcomes):
    _need(ACC_B200, CLI_B200)
    got = subprocess.run(_acc_args(ACC_B200, criterion), capture_output=True, text=True, timeout=900)
    rc_ref, line_ref = reference_outcomes[criterion]
    assert got.returncode == 0, got.stdout + got.stderr
    assert got.stdout.strip().startswith(f"criterion {criterion}: PASS")
    assert rc_ref == 0, line_ref
    assert _strip_times(got.stdout.strip()) == _strip_times(line_ref)


def test_acceptance_criterion_10_device_objective():
    """#10 asserts a >= 2x CPU speedup from 4 threads; the engine ignores
    n_threads (the device decides parallelism), so its two timings are the
    same objective.  What #10 can show: 10,000 evaluations on the device take
    less time than the reference's 1-thread objective."""
    _need(ACC_REF, ACC_B200)
    pat = re.compile(r"\(([-+0-9.e]+) s vs ([-+0-9.e]+) s\)")
    ref = subprocess.run([str(ACC_REF), "10"], capture_output=True, text=True, timeout=900)
    dev = subprocess.run([str(ACC_B200), "10"], capture_output=True, text=True, timeout=900)
    r_serial, _ = (float(x) for x in pat.search(ref.stdout).groups())
    d_serial, d_parallel = (float(x) for x in pat.search(dev.stdout).groups())
    assert max(d_serial, d_parallel) < r_serial, (ref.stdout, dev.stdout)


def test_reference_unit_tests_on_engine():
    """The reference's own doctest suite (tests/test_model.cpp,
    test_objectives.cpp, test_pso.cpp, test_calibration.cpp,
    test_timeseries.cpp: 73 test cases, ~65k assertions), built unmodified
    against oracle/doctest_standin, passes on the engine exactly as it does
    on the pure reference."""
    ref, b200 = REF / "unit_tests_ref", REF / "unit_tests_b200"
    _need(ref, b200)
    r = subprocess.run([str(ref)], capture_output=True, text=True, timeout=900)
    e = subprocess.run([str(b200)], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:]
    assert e.returncode == 0, e.stdout[-3000:]
    summary = [ln for ln in e.stdout.splitlines() if ln.startswith("[doctest]")]
    assert summary == [ln for ln in r.stdout.splitlines() if ln.startswith("[doctest]")], (summary, r.stdout[-500:])
    assert "73 passed | 0 failed" in summary[0], summary


def _run_py(pkg_dir, code):
    env = dict(os.environ, PYTHONPATH=str(pkg_dir))
    return subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900, env=env)


def test_reference_python_smoke_on_engine():
    smoke = SMOKE
    _need(smoke, REF / "py_b200" / "sirdfit" / "__init__.py", CLI_B200)
    env = dict(os.environ, PYTHONPATH=str(REF / "py_b200"), SIRDFIT_CLI=str(CLI_B200))
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir",
                          str(smoke.parent), str(smoke)], capture_output=True, text=True, timeout=900, env=env,
                         cwd=smoke.parent)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "7 passed" in out.stdout, out.stdout[-2000:]
    # the module really is the engine: libsirdgpu.so is mapped into the process
    probe = _run_py(REF / "py_b200", "import sirdfit, sys; sirdfit.integrate(sirdfit.SirdParams(beta1=0.5), "
                                     "sirdfit.SirdState(S=999.0, I=1.0), 1000.0, 5);"
                                     "print(any('libsirdgpu.so' in l for l in open('/proc/self/maps')))")
    assert probe.stdout.strip() == "True", probe.stdout + probe.stderr


PY_FIT = r"""
import datetime, tempfile, sirdfit
P = dict(beta1=0.6, beta2=0.9, t1=15.0, t2=30.0, gamma=0.09, mu=0.012)
tr = sirdfit.integrate(sirdfit.SirdParams(**P), sirdfit.SirdState(S=1e6 - 100.0, I=100.0), 1e6, 60)
with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False) as f:
    f.write("date,confirmed,recovered,deaths\n")
    for t, s in enumerate(tr.states):
        day = datetime.date(2020, 3, 1) + datetime.timedelta(days=t)
        f.write(f"{day.isoformat()},{s.I + s.R + s.D!r},{s.R!r},{s.D!r}\n")
data = sirdfit.load_raw_csv(f.name)
out = [s.D for s in tr.states] + list(data.infectious)
fit = sirdfit.fit_window(data, sirdfit.Window(index=0, start=5, length=21), 1e6, objective="ird-mse",
                         particles=400, iters=80, seed=2)
p = fit.params
out += [fit.objective, fit.r2_d, p.beta1, p.beta2, p.t1, p.t2, p.gamma, p.mu]
out += [s.D for s in sirdfit.forecast_extension(fit, 10).trajectory.states]
allr = sirdfit.fit_all_windows(data, 1e6, tau=20, delta=10, objective="d-mape", particles=300, iters=30, seed=4)
out += [f.objective for f in allr.fits] + [allr.mean_r2_d, float(allr.failed_count)]
print(" ".join(float(x).hex() for x in out))
"""


def test_python_module_values_match_pure_reference():
    _need(REF / "py_b200" / "sirdfit" / "__init__.py", REF / "py_ref" / "sirdfit" / "__init__.py")
    dev = _run_py(REF / "py_b200", PY_FIT)
    ref = _run_py(REF / "py_ref", PY_FIT)
    assert dev.returncode == 0 and ref.returncode == 0, dev.stderr[-2000:] + ref.stderr[-2000:]
    assert dev.stdout.split() == ref.stdout.split()


def test_cpp_api_against_reference_in_one_process():
    """tests/cpp/api_parity.cpp: optimize/Swarm (host objectives of 1-100
    dimensions, a host repair hook, window objectives fused and stepped),
    objective_value, metric_value, sird_rhs, integrate_euler_into,
    minmax_normalize and build_envelope of sirdfit_b200 against the
    unmodified reference, bit for bit."""
    exe = REF / "api_parity"
    _need(exe)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "MISMATCH" not in out.stdout, out.stdout + out.stderr[-2000:]
    assert out.stdout.count("\nok ") + out.stdout.startswith("ok ") >= 20, out.stdout


def _write_raw_csv(path, n_days=80):
    """A reported series from the reference's own model (the smoke test's
    generator with noise-free cumulative columns)."""
    code = ("import sirdfit, datetime\n"
            "tr = sirdfit.integrate(sirdfit.SirdParams(beta1=0.6, beta2=0.3, t1=20.0, t2=45.0, gamma=0.09, mu=0.012),"
            " sirdfit.SirdState(S=1e6 - 100.0, I=100.0), 1e6, %d)\n"
            "print('date,confirmed,recovered,deaths')\n"
            "for t, s in enumerate(tr.states):\n"
            "    d = datetime.date(2020, 3, 1) + datetime.timedelta(days=t)\n"
            "    print(f'{d.isoformat()},{s.I + s.R + s.D!r},{s.R!r},{s.D!r}')\n" % n_days)
    out = _run_py(REF / "py_ref", code)
    assert out.returncode == 0, out.stderr
    path.write_text(out.stdout)


def test_cli_outputs_byte_identical_to_reference(tmp_path):
    """Every command of the reference CLI on the engine writes the same bytes
    as the pure-reference CLI (fits.json, envelopes, bands, forecasts, the
    compare table, the cleaned series) with the same exit code."""
    _need(CLI_REF, CLI_B200)
    raw = tmp_path / "raw.csv"
    _write_raw_csv(raw)
    common = ["--input", str(raw), "--population", "1000000"]
    search = ["--particles", "300", "--iters", "25", "--seed", "11"]
    commands = {
        "preprocess": ["preprocess", "--input", str(raw), "--smooth"],
        "fit": ["fit", *common, "--tau", "20", "--delta", "7", "--objective", "ird-mxse", *search, "--threads", "max"],
        "compare": ["compare", *common, "--tau", "20", "--delta", "20", "--particles", "120", "--iters", "10",
                    "--seed", "3"],
        "forecast": ["forecast", *common, "--tau", "20", "--objective", "d-mape", "--horizon", "14",
                     "--window-start", "last", *search],
        "stability": ["stability", *common, "--tau", "20", "--objective", "d-mse", "--reps", "9", "--horizon", "10",
                      "--window-start", "30", *search],
    }
    for name, args in commands.items():
        outs = {}
        for which, exe in (("ref", CLI_REF), ("b200", CLI_B200)):
            d = tmp_path / f"{name}_{which}"
            r = subprocess.run([str(exe), *args, "--out-dir", str(d)], capture_output=True, text=True, timeout=900)
            files = {p.name: p.read_bytes() for p in sorted(d.glob("*"))} if d.exists() else {}
            outs[which] = (r.returncode, files, r.stdout)
        assert outs["ref"][0] == outs["b200"][0], (name, outs["ref"][2], outs["b200"][2])
        assert outs["ref"][1] and set(outs["ref"][1]) == set(outs["b200"][1]), name
        for fname, data in outs["ref"][1].items():
            assert outs["b200"][1][fname] == data, f"{name}: {fname} differs"
