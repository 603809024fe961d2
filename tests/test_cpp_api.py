"""The C++ calibration API (include/sirdfit_b200.hpp) as a maintainer of the
reference would use it: tests/cpp/api_demo.cpp must
compile and link against libsirdgpu.so with the reference's C++20 flags
(CPU), and on a B200 print exactly what the Python API computes on the same
inputs (bit for bit)."""
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2204_12346_b200" / "libsirdgpu.so"
SRC = ROOT / "tests" / "cpp" / "api_demo.cpp"


@pytest.fixture(scope="module")
def demo(tmp_path_factory):
    if not LIB.exists():
        pytest.skip("libsirdgpu.so not built")
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    exe = tmp_path_factory.mktemp("cpp") / "api_demo"
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{ROOT / 'include'}", str(SRC), "-o", str(exe),
                    f"-L{LIB.parent}", "-lsirdgpu", f"-Wl,-rpath,{LIB.parent}"], check=True)
    return exe


def test_cpp_api_compiles_and_links(demo):
    assert demo.exists()


@pytest.mark.gpu
def test_cpp_api_matches_python_api(demo):
    import paper_2204_12346_b200 as eng
    import paper_2204_12346_b200.sirdfit as sf
    from conftest import GOLDEN
    out = subprocess.run([str(demo), str(GOLDEN / "poland_like.csv")], capture_output=True, text=True, check=True)
    got = {}
    for line in out.stdout.splitlines():
        k, v = line.split(" ", 1)
        got[k] = v if k == "all.n" else float.fromhex(v)
    a = np.genfromtxt(GOLDEN / "poland_like.csv", delimiter=",", names=True)
    data = sf.EpiSeries(infectious=list(a["infectious"]), recovered_cum=list(a["recovered_cum"]),
                        deaths_cum=list(a["deaths_cum"]), new_cases=list(a["new_cases"]))
    N = 38e6
    fit = sf.fit_window(data, sf.Window(0, 0, 21), N, "ird-mxse", particles=256, iters=60, seed=2204)
    assert got["fit.objective"] == fit.objective
    assert got["fit.r2_d"] == fit.r2_d
    assert (got["fit.beta1"], got["fit.t2"], got["fit.mu"]) == (fit.params.beta1, fit.params.t2, fit.params.mu)
    assert got["forecast.D7"] == sf.forecast_extension(fit, 7).trajectory.states[-1].D
    allr = sf.fit_all_windows(data, N, tau=35, delta=60, objective="ird-mxse", particles=300, iters=20, seed=7)
    assert int(got["all.n"]) == len(allr.fits)
    for k, f in enumerate(allr.fits):
        assert got[f"all.objective.{k}"] == f.objective
    assert got["all.mean_r2_d"] == allr.mean_r2_d
    st = sf.stability_study(data, sf.Window(0, 100, 21), N, 6, 5, objective="d-mse", particles=128, iters=15,
                            seed=11)
    assert got["stability.deaths_median_last"] == st.deaths.median[-1]
    assert got["stability.gamma_median"] == st.gamma.median
    I, R, D = (a[k][40:76] for k in ("infectious", "recovered_cum", "deaths_cum"))
    win = eng.Window(sf.context(), I, R, D, [N - I[0] - R[0] - D[0], I[0], R[0], D[0]], N, "ird-mape")
    costs = win.eval_costs(np.array([[0.3, 0.2, 5.0, 20.0, 0.1, 0.01], [1.5, 0.05, 30.0, 2.0, 0.5, 0.002]]))
    assert (got["objective.cost0"], got["objective.cost1"]) == (costs[0], costs[1])


@pytest.fixture(scope="module")
def threads_demo(tmp_path_factory):
    if not LIB.exists():
        pytest.skip("libsirdgpu.so not built")
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    exe = tmp_path_factory.mktemp("cpp") / "threads_demo"
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-pthread", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "cpp" / "threads_demo.cpp"), "-o", str(exe), f"-L{LIB.parent}", "-lsirdgpu",
                    f"-Wl,-rpath,{LIB.parent}"], check=True)
    return exe


def test_cpp_threads_demo_compiles(threads_demo):
    assert threads_demo.exists()


@pytest.mark.gpu
def test_shared_context_is_reentrant(threads_demo):
    """Four threads share objectives of one context (scratch regrowth
    included) while a fifth runs fit_window: every result equals the
    single-threaded one bit for bit (host_api.cpp:92)."""
    from conftest import GOLDEN
    out = subprocess.run([str(threads_demo), str(GOLDEN / "poland_like.csv")], capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and out.stdout.startswith("threads ok"), out.stdout + out.stderr
