"""`sirdfit`-compatible command line driver on the B200 engine.

    python -m paper_2204_12346_b200.cli {preprocess,fit,compare,forecast,stability} ...

Same subcommands, options, defaults, output files and exit codes as the
reference CLI (tools/main.cpp:24-498): preprocessed.csv; fits.json (the
docs/fits.schema.json document) with envelopes_params.csv and
envelopes_compartments.csv; comparison.csv; forecast.csv;
stability_bands.csv and stability_summary.json; errors as a JSON object on
stderr with exit code 2, failed windows/repetitions with exit code 1.
Every calibration runs through the C++ host layer and the CUDA kernels
(paper_2204_12346_b200.sirdfit); this module only parses, cleans (host O(days)
work, series.py) and writes.  `--threads` is accepted and ignored: results
never depend on it (README.md:16-19 of the reference).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from pathlib import Path

from . import series as S
from .errors import Error, SchemeError

OBJECTIVES = ["d-mxse", "d-mse", "d-mae", "d-mape", "ird-mxse", "ird-mse", "ird-mae", "ird-mape"]
DEFAULTS = dict(out_dir=".", smooth=False, tau=35, delta=3, objective="ird-mxse", bounds="stage2", beta_lo=0.0,
                beta_hi=2.0, gamma_lo=0.0, gamma_hi=1.0, mu_lo=0.0, mu_hi=0.1, t_margin=7, particles=10000,
                iters=100, inertia=0.5, cognitive=0.5, social=0.5, seed=0, substeps=24, threads="auto", horizon=21,
                reps=1000, window_start="last")
PRESETS = {  # ParamBounds::stage1 / stage2 (calibration.cpp:54-65)
    "stage1": dict(beta_lo=0.0, beta_hi=10.0, gamma_lo=0.0, gamma_hi=10.0, mu_lo=0.0, mu_hi=10.0, t_margin=0),
    "stage2": dict(beta_lo=0.0, beta_hi=2.0, gamma_lo=0.0, gamma_hi=1.0, mu_lo=0.0, mu_hi=0.1, t_margin=7),
}


def _parse_threads(s: str) -> int:  # tools/main.cpp:54-63
    if s in ("auto", "max"):
        return 0
    if not s.isdigit():
        raise Error("--threads expects a non-negative integer, 'auto' or 'max'")
    return int(s)


def _bounds(o) -> dict:  # resolve_bounds, tools/main.cpp:66-82
    if o.bounds in PRESETS:
        return PRESETS[o.bounds]
    return dict(beta_lo=o.beta_lo, beta_hi=o.beta_hi, gamma_lo=o.gamma_lo, gamma_hi=o.gamma_hi, mu_lo=o.mu_lo,
                mu_hi=o.mu_hi, t_margin=o.t_margin)


def _settings(o, objective=None, preset=None):
    from . import _capi
    if preset is not None:
        o = argparse.Namespace(**{**vars(o), "bounds": preset})
    fam, met = _capi.parse_spec(objective or o.objective)
    b = _bounds(o)
    _parse_threads(o.threads)
    return _capi.sg_fit_settings(fam, met, b["beta_lo"], b["beta_hi"], b["gamma_lo"], b["gamma_hi"], b["mu_lo"],
                                 b["mu_hi"], int(b["t_margin"]), int(o.particles), int(o.iters), float(o.inertia),
                                 float(o.cognitive), float(o.social), float(o.population), int(o.substeps))


def _load(o, stats=None) -> S.Series:  # load_series, tools/main.cpp:99-106
    raw = S.read_raw_csv_file(o.input)
    epi = S.build_epi_series(raw, stats)
    return S.smooth7(epi) if o.smooth else epi


def _jsonable(v):
    if isinstance(v, float) and not math.isfinite(v):
        return None if math.isnan(v) else v
    if isinstance(v, dict):
        return {k: _jsonable(x) for k, x in v.items()}
    if isinstance(v, (list, tuple)):
        return [_jsonable(x) for x in v]
    return v


def _dump(path: Path, doc: dict) -> None:
    # nlohmann::json objects are key-sorted; NaN prints as null
    path.write_text(json.dumps(_jsonable(doc), indent=2, sort_keys=True, allow_nan=False) + "\n")


def _config_json(o) -> dict:  # tools/main.cpp:145-163
    b = _bounds(o)
    return {"input": o.input, "population": o.population, "tau": o.tau, "delta": o.delta, "objective": o.objective,
            "bounds_preset": o.bounds,
            "bounds": {"beta": [b["beta_lo"], b["beta_hi"]], "gamma": [b["gamma_lo"], b["gamma_hi"]],
                       "mu": [b["mu_lo"], b["mu_hi"]], "t_margin": int(b["t_margin"])},
            "particles": o.particles, "iters": o.iters, "inertia": o.inertia, "cognitive": o.cognitive,
            "social": o.social, "seed": o.seed, "substeps": o.substeps, "smooth": o.smooth}


def _to_mirror(epi: S.Series):
    from . import sirdfit
    return sirdfit.EpiSeries(epi.infectious, epi.recovered_cum, epi.deaths_cum, epi.new_cases,
                             S.format_date(epi.start_date))


def _resolve_window_start(text: str, epi: S.Series, tau: int) -> int:  # tools/main.cpp:110-132
    if epi.size() < tau + 1:
        raise SchemeError(f"series has {epi.size()} days; a window needs {tau + 1}")
    max_start = epi.size() - 1 - tau
    if text == "last":
        return max_start
    if text.isdigit():
        day = int(text)
        if day > max_start:
            raise SchemeError(f"window starting at day {day} runs past the data")
        return day
    offset = (S.parse_date(text) - epi.start_date).days
    if offset < 0 or offset > max_start:
        raise SchemeError(f"window starting at {text} runs past the data")
    return offset


# ---- subcommands ----------------------------------------------------------------------

def run_preprocess(o) -> int:
    stats = S.CleaningStats()
    raw = S.read_raw_csv_file(o.input)
    epi = S.build_epi_series(raw, stats)
    if o.smooth:
        epi = S.smooth7(epi)
    out = Path(o.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    S.write_epi_csv(str(out / "preprocessed.csv"), epi)
    print(f"rows in: {len(raw)}\ndays out: {epi.size()}\ninterpolated cells: {stats.interpolated_cells}\n"
          f"negative daily corrections: {stats.negative_corrections}\noutflow caps: {stats.outflow_corrections}")
    return 0


def _fit_all(o, epi, objective=None, preset=None):
    from . import sirdfit
    s = _settings(o, objective, preset)
    return sirdfit.fit_all_windows_settings(_to_mirror(epi), s, o.tau, o.delta, o.seed)


def _envelope_rows(rows, name, env, epi):  # tools/main.cpp:210-219
    for day in range(env.days()):
        rows.append([name, str(day), S.format_date(epi.date_at(day)), str(env.count[day]),
                     S.format_double(env.outer_lo[day]), S.format_double(env.band1_lo[day]),
                     S.format_double(env.band2_lo[day]), S.format_double(env.median[day]),
                     S.format_double(env.band2_hi[day]), S.format_double(env.band1_hi[day]),
                     S.format_double(env.outer_hi[day])])


ENVELOPE_HEADER = "series,day,date,count,outer_lo,band1_lo,band2_lo,median,band2_hi,band1_hi,outer_hi"
BAND_HEADER = "series,day,date,count,p95_lo,p90_lo,p50_lo,median,p50_hi,p90_hi,p95_hi"


def run_fit(o) -> int:  # tools/main.cpp:257-285
    epi = _load(o)
    result = _fit_all(o, epi)
    out = Path(o.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    windows = []
    for fit in result.fits:
        params = None
        if fit.ok:
            st = float(fit.window.start)
            params = {"beta1": fit.params.beta1, "beta2": fit.params.beta2, "t1": st + fit.params.t1,
                      "t2": st + fit.params.t2, "gamma": fit.params.gamma, "mu": fit.params.mu}
        windows.append({"index": fit.window.index, "start_day": fit.window.start,
                        "start_date": S.format_date(epi.date_at(fit.window.start)), "end_day": fit.window.last_day(),
                        "ok": fit.ok, "objective_value": fit.objective, "r2_d": fit.r2_d, "params": params,
                        "failure": None if fit.ok else fit.failure})
    _dump(out / "fits.json", {"config": _config_json(o), "n_windows": len(result.fits),
                              "failed_count": result.failed_count, "mean_r2_d": result.mean_r2_d,
                              "windows": windows})
    p = S.parameter_envelopes(result.fits, epi.size())
    rows = []
    for name in ("beta", "gamma", "mu", "r0"):
        _envelope_rows(rows, name, p[name], epi)
    S.write_table(str(out / "envelopes_params.csv"), ENVELOPE_HEADER, rows)
    c = S.compartment_envelopes(result.fits, epi.size())
    rows = []
    for name in ("infectious", "recovered", "deaths"):
        _envelope_rows(rows, name, c[name], epi)
    S.write_table(str(out / "envelopes_compartments.csv"), ENVELOPE_HEADER, rows)
    print(f"windows: {len(result.fits)} ({result.failed_count} failed)\n"
          f"mean R2(D): {S.format_double(result.mean_r2_d)}")
    return 1 if result.failed_count > 0 else 0


def run_compare(o) -> int:  # tools/main.cpp:287-321
    epi = _load(o)
    any_failed = False
    rows = []
    for preset, family in (("stage1", "d"), ("stage1", "ird"), ("stage2", "d"), ("stage2", "ird")):
        row = [preset, family]
        for metric in ("mxse", "mse", "mae", "mape"):
            res = _fit_all(o, epi, objective=f"{family}-{metric}", preset=preset)
            any_failed = any_failed or res.failed_count > 0
            row.append(S.format_double(res.mean_r2_d))
        rows.append(row)
    out = Path(o.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    header = "bounds,family,mxse,mse,mae,mape"
    S.write_table(str(out / "comparison.csv"), header, rows)
    print(header)
    for row in rows:
        print(",".join(row))
    return 1 if any_failed else 0


def run_forecast(o) -> int:  # tools/main.cpp:323-361
    from . import sirdfit
    epi = _load(o)
    start = _resolve_window_start(o.window_start, epi, o.tau)
    window = sirdfit.Window(0, start, o.tau + 1)
    fit = sirdfit.fit_window_settings(_to_mirror(epi), window, _settings(o), o.seed)
    fc = sirdfit.forecast_extension(fit, o.horizon, o.substeps)
    rows = []
    for k in range(o.horizon + 1):
        day = fc.junction_day + k
        s = fc.trajectory.states[k]
        row = [str(k), S.format_date(epi.date_at(day)), S.format_double(s.S), S.format_double(s.I),
               S.format_double(s.R), S.format_double(s.D)]
        if day < epi.size():
            row += [S.format_double(epi.infectious[day]), S.format_double(epi.recovered_cum[day]),
                    S.format_double(epi.deaths_cum[day])]
        else:
            row += ["", "", ""]
        rows.append(row)
    out = Path(o.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    S.write_table(str(out / "forecast.csv"),
                  "day,date,S,I,R,D,reported_infectious,reported_recovered_cum,reported_deaths_cum", rows)
    p = fit.params
    print(f"window: days {window.start}..{window.last_day()} ({S.format_date(epi.date_at(window.start))})\n"
          f"objective {o.objective} = {S.format_double(fit.objective)}, R2(D) = {S.format_double(fit.r2_d)}\n"
          f"params: beta1={S.format_double(p.beta1)} beta2={S.format_double(p.beta2)} "
          f"t1={S.format_double(float(start) + p.t1)} t2={S.format_double(float(start) + p.t2)} "
          f"gamma={S.format_double(p.gamma)} mu={S.format_double(p.mu)}")
    return 0


def run_stability(o) -> int:  # tools/main.cpp:363-397
    from . import sirdfit
    epi = _load(o)
    start = _resolve_window_start(o.window_start, epi, o.tau)
    window = sirdfit.Window(0, start, o.tau + 1)
    st = sirdfit.stability_study_settings(_to_mirror(epi), window, _settings(o), o.reps, o.horizon, o.seed)
    rows = []
    for name in ("beta", "r0", "infectious", "recovered", "deaths"):
        b = getattr(st, name)
        for k in range(b.days()):
            day = window.start + k
            rows.append([name, str(day), S.format_date(epi.date_at(day)), str(b.count[k]),
                         S.format_double(b.p95_lo[k]), S.format_double(b.p90_lo[k]), S.format_double(b.p50_lo[k]),
                         S.format_double(b.median[k]), S.format_double(b.p50_hi[k]), S.format_double(b.p90_hi[k]),
                         S.format_double(b.p95_hi[k])])
    out = Path(o.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    S.write_table(str(out / "stability_bands.csv"), BAND_HEADER, rows)

    def sb(b):
        return {"count": b.count, "median": b.median, "p50": [b.p50_lo, b.p50_hi], "p90": [b.p90_lo, b.p90_hi],
                "p95": [b.p95_lo, b.p95_hi]}
    _dump(out / "stability_summary.json",
          {"window": {"start_day": window.start, "start_date": S.format_date(epi.date_at(window.start)),
                      "end_day": window.last_day()},
           "horizon": st.horizon, "repetitions": st.repetitions, "failed": st.failed, "gamma": sb(st.gamma),
           "mu": sb(st.mu), "config": _config_json(o)})
    print(f"repetitions: {st.repetitions} ({st.failed} failed)")
    return 1 if st.failed > 0 else 0


# ---- argument parsing (tools/main.cpp:400-478) ----------------------------------------------

def _read_config(path: str) -> dict:
    """--config FILE: `key = value` lines (CLI11's INI/TOML subset); flags on
    the command line take precedence, then the file, then the defaults."""
    out = {}
    for line in Path(path).read_text().splitlines():
        line = line.split("#", 1)[0].strip()
        if not line or line.startswith("["):
            continue
        if "=" not in line:
            raise Error(f"config line '{line}' is not key = value")
        k, v = (x.strip() for x in line.split("=", 1))
        out[k.replace("-", "_")] = v.strip('"').strip("'")
    return out


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="sirdfit",
                                 description="SIRD model calibration on overlapping windows with particle swarm "
                                             "search (B200 engine)")
    ap.add_argument("--config", help="config file with key = value lines")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def data(p):
        p.add_argument("--input", required=True, help="Input CSV: date,confirmed,recovered,deaths")
        p.add_argument("--out-dir", dest="out_dir", default=argparse.SUPPRESS)
        p.add_argument("--smooth", action="store_true", default=argparse.SUPPRESS)

    def search(p):
        p.add_argument("--population", type=float, required=True)
        for name, typ in (("tau", int), ("delta", int), ("beta-lo", float), ("beta-hi", float), ("gamma-lo", float),
                          ("gamma-hi", float), ("mu-lo", float), ("mu-hi", float), ("t-margin", int),
                          ("particles", int), ("iters", int), ("inertia", float), ("cognitive", float),
                          ("social", float), ("seed", int), ("substeps", int)):
            p.add_argument(f"--{name}", dest=name.replace("-", "_"), type=typ, default=argparse.SUPPRESS)
        p.add_argument("--bounds", choices=["stage1", "stage2", "custom"], default=argparse.SUPPRESS)
        p.add_argument("--threads", default=argparse.SUPPRESS)

    def objective(p):
        p.add_argument("--objective", choices=OBJECTIVES, default=argparse.SUPPRESS)

    data(sub.add_parser("preprocess", help="Clean a reported series into the daily model inputs"))
    p = sub.add_parser("fit", help="Calibrate every window and write fits and envelopes")
    data(p), search(p), objective(p)
    p = sub.add_parser("compare", help="Mean R2(D) for every objective spec and bounds preset")
    data(p), search(p)
    for name, extra in (("forecast", False), ("stability", True)):
        p = sub.add_parser(name)
        data(p), search(p), objective(p)
        p.add_argument("--horizon", type=int, default=argparse.SUPPRESS)
        p.add_argument("--window-start", dest="window_start", default=argparse.SUPPRESS)
        if extra:
            p.add_argument("--reps", type=int, default=argparse.SUPPRESS)
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    args = ap.parse_args(argv)
    opts = dict(DEFAULTS)
    try:
        if args.config:
            typed = {k: type(DEFAULTS[k])(v) if k in DEFAULTS and not isinstance(DEFAULTS[k], bool) else v
                     for k, v in _read_config(args.config).items()}
            for k, v in list(typed.items()):
                if k in DEFAULTS and isinstance(DEFAULTS[k], bool):
                    typed[k] = str(v).lower() in ("1", "true", "yes", "on")
            opts.update(typed)
        opts.update({k: v for k, v in vars(args).items() if k not in ("config",)})
        o = argparse.Namespace(**opts)
        if not hasattr(o, "population") and o.cmd != "preprocess":
            raise Error("--population is required")
        if getattr(o, "population", 1.0) <= 0:
            raise Error("--population: value must be positive")
        run = {"preprocess": run_preprocess, "fit": run_fit, "compare": run_compare, "forecast": run_forecast,
               "stability": run_stability}[o.cmd]
        return run(o)
    except Exception as e:  # tools/main.cpp:493-496
        sys.stderr.write(json.dumps({"error": str(e)}) + "\n")
        return 2


if __name__ == "__main__":
    sys.exit(main())
