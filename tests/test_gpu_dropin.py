"""The drop-in, end to end: the reference's own `Swarm` (pso.cpp, compiled
unmodified from its sources into oracle/_ref/libsirdhybrid.so) with its
objective body replaced by the engine's sg_eval_costs — the exact binding of
INTEGRATION.md §1 (oracle/hybrid_shim.cpp).  Because the GPU costs are
bit-identical, the reference optimizer must follow the pure-CPU trajectory
bit for bit: same per-iteration best, same final particle, same status
(pso.cpp:78-147 consumes costs only through `<` comparisons, so one flipped
bit anywhere would surface here).
"""
import json

import numpy as np
import pytest

from helpers import assert_bitwise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hybrid():
    from oracle import oracle_py
    if not oracle_py.HYBRID_SO.exists():
        pytest.skip("oracle/_ref/libsirdhybrid.so not built (needs the reference sources at build time)")
    return oracle_py.load("hybrid")


def _unhex(v):
    return np.array([float.fromhex(x) for x in v])


def test_reference_swarm_on_gpu_objective_matches_goldens(hybrid):
    from conftest import GOLDEN
    for c in json.loads((GOLDEN / "fits.json").read_text()):
        rc, best, cost, hist = hybrid.fit_swarm(c["spec"], _unhex(c["I"]), _unhex(c["R"]), _unhex(c["D"]),
                                                _unhex(c["init"]), c["N"], c["lower"], c["upper"], c["n"],
                                                c["iters"], inertia=c["w"], cognitive=c["c1"], social=c["c2"],
                                                seed=c["seed"])
        assert rc == c["status"], c["name"]
        assert_bitwise(hist, _unhex(c["history"]), c["name"] + " history")
        if rc == 0:
            assert_bitwise(best, _unhex(c["best"]), c["name"] + " best")
            assert cost == float.fromhex(c["best_cost"])


@pytest.mark.parametrize("spec", ["d-mse", "ird-mxse", "ird-mape"])
def test_reference_swarm_on_gpu_objective_matches_cpu_swarm(hybrid, port, poland, spec):
    a = 90
    I, R, D = poland["I"][a:a + 36], poland["R"][a:a + 36], poland["D"][a:a + 36]
    N = poland["N"]
    init = [N - I[0] - R[0] - D[0], I[0], R[0], D[0]]
    lo, hi = [0] * 6, [2, 2, 28, 28, 1, 0.1]
    got = hybrid.fit_swarm(spec, I, R, D, init, N, lo, hi, 1500, 25, seed=31)
    want = port.fit_swarm(spec, I, R, D, init, N, lo, hi, 1500, 25, seed=31)
    assert got[0] == want[0] == 0
    assert_bitwise(got[3], want[3], spec + " history")
    assert_bitwise(got[1], want[1], spec + " best")
