"""Extended version of tests/test_gpu_fuzz.py: many more seeded batches (plans vs the C oracle, bit for bit)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

import paper_2204_12346_b200 as eng  # noqa: E402
from oracle import oracle_py  # noqa: E402
from test_gpu_fuzz import _case  # noqa: E402


def main():
    n_batches = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    seed_base = int(sys.argv[2]) if len(sys.argv) > 2 else 900000  # batch b uses default_rng(seed_base + b)
    ctx = eng.Context(0)
    port = oracle_py.load("port")
    bad = 0
    for batch in range(n_batches):
        rng = np.random.default_rng(seed_base + batch)
        cases = [_case(rng) for _ in range(16)]
        wins, swarms = [], []
        for c in cases:
            w = eng.Window(ctx, c["I"], c["R"], c["D"], c["init"], c["N"], c["spec"], substeps=c["sub"])
            wins.append(w)
            swarms.append(dict(window=w, lower=c["lo"], upper=c["hi"], n_particles=c["n"], max_iters=c["iters"],
                               seed=c["seed"], repair=c["repair"], **c["coeffs"]))
        try:
            out = ctx.fit_swarms(swarms)
        except Exception as e:  # noqa: BLE001 - report the batch that failed, then stop
            print("ERROR batch", batch, repr(e), flush=True)
            for k, c in enumerate(cases):
                print("  case", k, c["spec"], "days", len(c["I"]), "sub", c["sub"], "n", c["n"], "iters", c["iters"],
                      flush=True)
            return 2
        for k, c in enumerate(cases):
            rc, best, cost, hist = port.fit_swarm(c["spec"], c["I"], c["R"], c["D"], c["init"], c["N"], c["lo"],
                                                  c["hi"], c["n"], c["iters"], seed=c["seed"], repair=c["repair"],
                                                  substeps=c["sub"], **c["coeffs"])
            ok = out[k][0] == rc and np.array_equal(out[k][3].view(np.uint64), hist.view(np.uint64))
            if rc == 0:
                ok = ok and np.array_equal(out[k][1].view(np.uint64), best.view(np.uint64))
            if not ok:
                bad += 1
                print("MISMATCH batch", batch, "case", k, c["spec"], c["sub"], flush=True)
    print(f"fuzz_long: {n_batches * 16} swarms (seeds {seed_base}..{seed_base + n_batches - 1}), {bad} mismatches", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
