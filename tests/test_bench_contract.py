"""bench.py keeps the driver's contract: one JSON line with the required keys,
for the reference arm on the CPU (oracle/_ref) and for the engine on a B200."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _line(args, timeout):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_reference_arm_line():
    from oracle import oracle_py
    if not (oracle_py.REF_SO.exists() or oracle_py.PORT_SO.exists()):
        pytest.skip("no CPU oracle built")
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-budget", "0.5"], 300)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert {"value", "unit", "cores", "kind", "sample"} <= set(d["cpu_baseline"])
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_engine_line():
    d = _line(["--steps", "3", "--warmup", "3", "--iters", "5", "--no-cpu"], 600)
    assert BASE_KEYS <= set(d)
    assert {"e2e", "roofline", "clocks", "gpu_launches"} <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["scaling"] == "strong"
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert 0.0 < r["frac"] < 1.0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["e2e"]["matches_device_run"] is True
    assert d["gpu_launches"] > 0


def test_reference_arm_under_torchrun():
    """N>1 launch of the reference arm (the driver's scaling run): rank 0
    alone prints the line, the other rank exits 0 without work."""
    from oracle import oracle_py
    if not (oracle_py.REF_SO.exists() or oracle_py.PORT_SO.exists()):
        pytest.skip("no CPU oracle built")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29537", str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
           "--steps", "1", "--warmup", "0", "--ref-budget", "0.5"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


@pytest.mark.gpu
def test_engine_line_carries_parity_and_one_thread_baseline():
    """The cpu_baseline leg's whole-window reference fits are compared bit for
    bit with the device plan; short iterations keep the
    CPU leg to seconds."""
    d = _line(["--steps", "3", "--warmup", "3", "--iters", "20", "--cpu-budget", "2", "--cpu1-budget", "0.5"], 900)
    assert d["parity"]["bit_exact"] is True and len(d["parity"]["windows"]) >= 1
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["value_1thread"] > 0
    assert d["roofline"]["frac"] == pytest.approx(d["roofline"]["achieved"] / d["roofline"]["peak"])


@pytest.mark.gpu
@pytest.mark.parametrize("split", ["windows", "restarts"])
def test_engine_arm_under_torchrun(split):
    """The ours arm's N>1 path: two ranks share cuda:0
    over gloo (functional only — value is the shared GPU's throughput); rank 0
    prints one line with n_gpus == 2, the other rank prints nothing."""
    import os
    env = dict(os.environ, SG_BENCH_BACKEND="gloo")
    port = 29541 if split == "windows" else 29543
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--iters", "10", "--split", split, "--cpu-budget", "1", "--cpu1-budget", "0.3"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["split"] == split
    assert d["scaling"] == ("strong" if split == "windows" else "weak")
    assert d["cpu_baseline"]["value"] > 0 and d["parity"]["bit_exact"] is True
