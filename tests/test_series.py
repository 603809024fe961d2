"""Host data layer (paper_2204_12346_b200/series.py) vs the reference:
format_double (csv.cpp:84-94), build_epi_series + smooth7
(timeseries.cpp:50-179) on raw series with gaps, dips and outflow caps, and
build_envelope (calibration.cpp:218-245).  Golden values from the reference
(tests/golden/series.json); CPU only."""
import json
import math

import pytest

from paper_2204_12346_b200 import series as S


@pytest.fixture(scope="module")
def golden():
    from conftest import GOLDEN
    return json.loads((GOLDEN / "series.json").read_text())


def _unhex(v):
    return None if v is None else float.fromhex(v)


def _same(a, b):
    return (math.isnan(a) and math.isnan(b)) or (a == b and math.copysign(1, a) == math.copysign(1, b))


def test_format_double_matches_to_chars(golden):
    for h, want in golden["format_double"]:
        assert S.format_double(float.fromhex(h)) == want, (h, want)


def test_cleaning_matches_reference(golden):
    import datetime as dt
    for case in golden["clean"]:
        start = dt.date(2020, 3, 18)
        records = [S.RawRecord(start + dt.timedelta(days=d), *[_unhex(x) for x in row])
                   for d, row in zip(case["days"], case["raw"])]
        stats = S.CleaningStats()
        epi = S.build_epi_series(records, stats)
        if case["smooth"]:
            epi = S.smooth7(epi)
        for name, key in (("infectious", "I"), ("recovered_cum", "R"), ("deaths_cum", "D"), ("new_cases", "new")):
            want = [float.fromhex(x) for x in case[key]]
            got = getattr(epi, name)
            assert len(got) == len(want)
            assert all(_same(a, b) for a, b in zip(got, want)), name
        assert [stats.interpolated_cells, stats.negative_corrections, stats.outflow_corrections] == case["stats"]


def test_envelopes_match_reference(golden):
    for case in golden["envelope"]:
        rows = [[math.nan if x is None else float.fromhex(x) for x in row] for row in case["values"]]
        n_days = len(rows[0])
        env = S.build_envelope([[r[d] for r in rows] for d in range(n_days)])
        want = [float.fromhex(x) for x in case["bands"]]
        got = env.outer_lo + env.band1_lo + env.band2_lo + env.median + env.band2_hi + env.band1_hi + env.outer_hi
        assert all(_same(a, b) for a, b in zip(got, want))
        assert env.count == case["counts"]


def test_raw_csv_parsing_and_errors(tmp_path):
    p = tmp_path / "in.csv"
    p.write_text("date,confirmed,recovered,deaths\n2020-03-01,10,1,0\n2020-03-03,,2,0\n2020-03-04,30,3,1\n")
    recs = S.read_raw_csv_file(str(p))
    assert len(recs) == 3 and recs[1].confirmed_cum is None
    epi = S.build_epi_series(recs)
    assert epi.size() == 4 and S.format_date(epi.start_date) == "2020-03-01"
    for text, msg in (("date,c,r,d\n", "expected header"),
                      ("date,confirmed,recovered,deaths\n2020-03-01,1,2\n", "expected 4 fields"),
                      ("date,confirmed,recovered,deaths\n2020-02-30,1,2,3\n", "invalid calendar day"),
                      ("date,confirmed,recovered,deaths\n2020-03-02,1,2,3\n2020-03-01,1,2,3\n", "strictly increasing"),
                      ("date,confirmed,recovered,deaths\n2020-03-01,-1,2,3\n", "negative or not finite")):
        with pytest.raises(S.Error, match=msg):
            S.read_raw_csv(text)
    with pytest.raises(S.MissingEndpointError):
        S.build_epi_series(S.read_raw_csv("date,confirmed,recovered,deaths\n2020-03-01,,1,1\n2020-03-02,1,1,1\n"))


def test_cli_reports_errors_as_json(tmp_path, capsys):
    from paper_2204_12346_b200 import cli
    assert cli.main(["fit", "--input", str(tmp_path / "missing.csv"), "--population", "1000"]) == 2
    err = capsys.readouterr().err
    assert json.loads(err)["error"].startswith("cannot open")
    p = tmp_path / "in.csv"
    p.write_text("date,confirmed,recovered,deaths\n2020-03-01,10,1,0\n2020-03-02,20,2,0\n")
    assert cli.main(["preprocess", "--input", str(p), "--out-dir", str(tmp_path / "o")]) == 0
    lines = (tmp_path / "o" / "preprocessed.csv").read_text().splitlines()
    assert lines[0] == "date,infectious,recovered_cum,deaths_cum,new_cases"
    assert lines[1] == "2020-03-01,9,1,0,10"
