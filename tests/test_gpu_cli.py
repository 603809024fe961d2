"""The `sirdfit` CLI on the B200 engine (paper_2204_12346_b200/cli.py) —
SURVEY §8f rank 2.  Mirrors the reference's acceptance criteria #4
(fits.json byte-identical for --threads 1 and max, acceptance/main.cpp:180-207)
and #8 (every band file nests per day, 362-398), test_smoke.py:89-120 (the
fits.json document shape of docs/fits.schema.json), and checks the fitted
windows bit for bit against the reference pipeline (read raw CSV ->
build_epi_series -> fit_all_windows; tests/golden/cli_fit.json).
"""
import json

import pytest

from paper_2204_12346_b200 import cli

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden():
    from conftest import GOLDEN
    return json.loads((GOLDEN / "cli_fit.json").read_text())


@pytest.fixture(scope="module")
def raw_csv(tmp_path_factory, golden):
    import datetime as dt
    p = tmp_path_factory.mktemp("cli") / "input.csv"
    start = dt.date.fromisoformat(golden["start_date"])
    lines = ["date,confirmed,recovered,deaths"]
    for k, row in enumerate(golden["raw_cells"]):
        lines.append(f"{(start + dt.timedelta(days=k)).isoformat()},{','.join(row)}")
    p.write_text("\n".join(lines) + "\n")
    return p


FIT_ARGS = ["--population", "1000000", "--tau", "20", "--delta", "10", "--objective", "ird-mxse", "--particles",
            "300", "--iters", "40", "--seed", "7"]


def _check_fits_document(doc):
    """docs/fits.schema.json, restated."""
    assert set(doc) == {"config", "failed_count", "mean_r2_d", "n_windows", "windows"}
    cfg = doc["config"]
    assert set(cfg) == {"bounds", "bounds_preset", "cognitive", "delta", "inertia", "input", "iters", "objective",
                        "particles", "population", "seed", "smooth", "social", "substeps", "tau"}
    assert set(cfg["bounds"]) == {"beta", "gamma", "mu", "t_margin"}
    assert all(len(cfg["bounds"][k]) == 2 for k in ("beta", "gamma", "mu"))
    assert isinstance(doc["n_windows"], int) and doc["n_windows"] == len(doc["windows"]) >= 1
    for w in doc["windows"]:
        assert set(w) == {"end_day", "failure", "index", "objective_value", "ok", "params", "r2_d", "start_date",
                          "start_day"}
        assert len(w["start_date"]) == 10 and w["start_date"][4] == "-"
        if w["ok"]:
            assert set(w["params"]) == {"beta1", "beta2", "gamma", "mu", "t1", "t2"} and w["failure"] is None
        else:
            assert w["params"] is None and isinstance(w["failure"], str)


def test_fit_matches_reference_and_is_thread_invariant(raw_csv, golden, tmp_path):
    assert cli.main(["fit", "--input", str(raw_csv), *FIT_ARGS, "--threads", "1", "--out-dir",
                     str(tmp_path / "one")]) == 0
    assert cli.main(["fit", "--input", str(raw_csv), *FIT_ARGS, "--threads", "max", "--out-dir",
                     str(tmp_path / "many")]) == 0
    a = (tmp_path / "one" / "fits.json").read_bytes()
    assert a and a == (tmp_path / "many" / "fits.json").read_bytes()  # acceptance #4
    doc = json.loads(a)
    _check_fits_document(doc)
    assert doc["n_windows"] == golden["n_windows"] == 4 and doc["failed_count"] == golden["failed"]
    params = [float.fromhex(x) for x in golden["params"]]
    for k, w in enumerate(doc["windows"]):
        p = params[6 * k:6 * k + 6]
        st = float(w["start_day"])
        assert [w["params"][n] for n in ("beta1", "beta2", "gamma", "mu")] == [p[0], p[1], p[4], p[5]]
        assert w["params"]["t1"] == st + p[2] and w["params"]["t2"] == st + p[3]
        assert w["objective_value"] == float.fromhex(golden["objective"][k])
        assert w["r2_d"] == float.fromhex(golden["r2"][k])
    assert doc["mean_r2_d"] == float.fromhex(golden["mean_r2"])


def _nested(path):
    rows = 0
    for line in path.read_text().splitlines()[1:]:
        cells = line.split(",")
        assert len(cells) == 11
        prev = -float("inf")
        for c in cells[4:]:
            if c == "":
                continue
            v = float(c)
            assert v >= prev, (path.name, line)
            prev = v
        rows += 1
    return rows


def test_band_files_nest(raw_csv, tmp_path):
    """acceptance #8."""
    assert cli.main(["fit", "--input", str(raw_csv), "--population", "1000000", "--tau", "20", "--delta", "5",
                     "--objective", "ird-mxse", "--particles", "250", "--iters", "40", "--seed", "8", "--out-dir",
                     str(tmp_path / "fit")]) == 0
    assert cli.main(["stability", "--input", str(raw_csv), "--population", "1000000", "--tau", "20", "--objective",
                     "d-mse", "--particles", "200", "--iters", "30", "--seed", "9", "--reps", "12", "--horizon", "10",
                     "--window-start", "last", "--out-dir", str(tmp_path / "stab")]) == 0
    rows = sum(_nested(p) for p in (tmp_path / "fit" / "envelopes_params.csv",
                                    tmp_path / "fit" / "envelopes_compartments.csv",
                                    tmp_path / "stab" / "stability_bands.csv"))
    assert rows > 0
    summary = json.loads((tmp_path / "stab" / "stability_summary.json").read_text())
    assert summary["repetitions"] == 12 and summary["failed"] == 0 and summary["horizon"] == 10


def test_forecast_and_compare(raw_csv, tmp_path):
    assert cli.main(["forecast", "--input", str(raw_csv), "--population", "1000000", "--tau", "20", "--particles",
                     "100", "--iters", "10", "--horizon", "7", "--window-start", "5", "--out-dir",
                     str(tmp_path / "fc")]) == 0
    lines = (tmp_path / "fc" / "forecast.csv").read_text().splitlines()
    assert lines[0].startswith("day,date,S,I,R,D") and len(lines) == 1 + 8
    assert cli.main(["compare", "--input", str(raw_csv), "--population", "1000000", "--tau", "20", "--delta", "20",
                     "--particles", "40", "--iters", "4", "--out-dir", str(tmp_path / "cmp")]) == 0
    rows = (tmp_path / "cmp" / "comparison.csv").read_text().splitlines()
    assert rows[0] == "bounds,family,mxse,mse,mae,mape" and len(rows) == 5


def test_failed_windows_exit_1(raw_csv, tmp_path):
    # a population far below the reported counts cannot seed any window
    assert cli.main(["fit", "--input", str(raw_csv), "--population", "10", "--tau", "20", "--delta", "10",
                     "--particles", "30", "--iters", "5", "--out-dir", str(tmp_path / "f")]) == 1
    doc = json.loads((tmp_path / "f" / "fits.json").read_text())
    assert doc["failed_count"] == doc["n_windows"] and doc["mean_r2_d"] is None


def test_python_cli_byte_identical_to_reference_cli(tmp_path):
    """`python -m paper_2204_12346_b200.cli` against the reference's own
    `sirdfit` CLI (oracle/_ref/sirdfit_cli_ref: tools/main.cpp over the pure
    reference, built with the CLI11 stand-in): every output file of every
    command is byte-identical (JSON layout and number formatting included)
    and the exit codes agree."""
    import subprocess
    import sys
    from pathlib import Path
    ROOT = Path(__file__).resolve().parents[1]
    ref_cli = ROOT / "oracle" / "_ref" / "sirdfit_cli_ref"
    if not ref_cli.exists():
        pytest.skip("reference CLI not built (oracle/Makefile refcallers)")
    raw = tmp_path / "raw.csv"
    lines = ["date,confirmed,recovered,deaths"]
    import datetime
    from oracle import oracle_py
    port = oracle_py.load("port")
    st, _ = port.integrate([0.6, 0.3, 20.0, 45.0, 0.09, 0.012], [1e6 - 100, 100, 0, 0], 1e6, 80)
    st = st.tolist()
    for t, (S_, I_, R_, D_) in enumerate(st):
        d = datetime.date(2020, 3, 1) + datetime.timedelta(days=t)
        lines.append(f"{d.isoformat()},{I_ + R_ + D_!r},{R_!r},{D_!r}")
    raw.write_text("\n".join(lines) + "\n")
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
    mismatches = []
    for name, args in commands.items():
        d_ref, d_eng = tmp_path / f"{name}_ref", tmp_path / f"{name}_eng"
        r = subprocess.run([str(ref_cli), *args, "--out-dir", str(d_ref)], capture_output=True, text=True,
                           timeout=600)
        e = subprocess.run([sys.executable, "-m", "paper_2204_12346_b200.cli", *args, "--out-dir", str(d_eng)],
                           capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert r.returncode == e.returncode, (name, r.stderr, e.stderr)
        ref_files = {p.name: p.read_bytes() for p in sorted(d_ref.glob("*"))}
        eng_files = {p.name: p.read_bytes() for p in sorted(d_eng.glob("*"))}
        assert ref_files and set(ref_files) == set(eng_files), (name, sorted(ref_files), sorted(eng_files))
        for fname, data in ref_files.items():
            if eng_files[fname] != data:
                a, b = data.decode().splitlines(), eng_files[fname].decode().splitlines()
                diff = [(i, x, y) for i, (x, y) in enumerate(zip(a, b)) if x != y][:3]
                mismatches.append((name, fname, len(a), len(b), diff))
    assert not mismatches, mismatches
