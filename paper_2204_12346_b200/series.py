"""Host-side data layer of the calibration driver: raw CSV ingest and the
cleaning pipeline (timeseries.cpp), dates (dates.cpp), number formatting and
tables (csv.cpp), and the rank envelopes of a window sweep
(calibration.cpp:17-35, 218-296).

O(days) post-/pre-processing that the reference also runs on the host
(SURVEY.md §2, §8f ranks 2 and 4); restated here in plain Python with the
reference's operation order, so the CLI (paper_2204_12346_b200/cli.py)
accepts the same inputs and writes the same tables as `sirdfit`
(tools/main.cpp).  No SIRD arithmetic happens here.
"""
from __future__ import annotations

import datetime as _dt
import math
from dataclasses import dataclass, field
from decimal import Decimal
from typing import Optional

from .errors import Error

SMOOTHING_WINDOW = 7  # timeseries.hpp:48


class ParseError(Error):
    """sirdfit::ParseError (errors.hpp:20-22)."""


class EmptySeriesError(Error):
    def __init__(self, msg: str = "series has no records"):
        super().__init__(msg)


class MissingEndpointError(Error):
    """sirdfit::MissingEndpointError (errors.hpp:16-18)."""


# ---- dates (dates.cpp) -------------------------------------------------------------

def parse_date(text: str) -> _dt.date:
    if len(text) != 10 or text[4] != "-" or text[7] != "-":
        raise ParseError(f"bad date '{text}': expected YYYY-MM-DD")
    try:
        y, m, d = int(text[0:4]), int(text[5:7]), int(text[8:10])
    except ValueError:
        raise ParseError(f"bad date '{text}': expected YYYY-MM-DD") from None
    if not (text[0:4].isdigit() and text[5:7].isdigit() and text[8:10].isdigit()):
        raise ParseError(f"bad date '{text}': expected YYYY-MM-DD")
    try:
        return _dt.date(y, m, d)
    except ValueError:
        raise ParseError(f"invalid calendar day '{text}'") from None


def format_date(day: _dt.date) -> str:
    return f"{day.year:04d}-{day.month:02d}-{day.day:02d}"


# ---- numbers (csv.cpp:84-94) ---------------------------------------------------------

def format_double(value: float) -> str:
    """std::to_chars(double) with no format: the shortest round-trip digits,
    printed as %f or %e style, whichever is shorter (fixed on ties); NaN is an
    empty field, infinities 'inf' / '-inf'."""
    if math.isnan(value):
        return ""
    if math.isinf(value):
        return "inf" if value > 0 else "-inf"
    if value == 0.0:
        return "-0" if math.copysign(1.0, value) < 0 else "0"
    sign, digits, exp = Decimal(repr(value)).normalize().as_tuple()
    ds = "".join(map(str, digits))
    n = len(ds)
    point = n + exp  # decimal point position relative to the digit string
    if exp >= 0:
        # integral value: of the equally long digit strings, to_chars prints
        # the one closest to the value, i.e. the exact integer
        fixed = str(int(abs(value)))
    elif point > 0:
        fixed = ds[:point] + "." + ds[point:]
    else:
        fixed = "0." + "0" * (-point) + ds
    e10 = point - 1
    mant = ds[0] + ("." + ds[1:] if n > 1 else "")
    sci = f"{mant}e{'-' if e10 < 0 else '+'}{abs(e10):02d}"
    out = fixed if len(fixed) <= len(sci) else sci
    return ("-" if sign else "") + out


def parse_number(field_text: str, line_no: int, column: str) -> float:
    try:
        if field_text.strip() != field_text or field_text.lower() in ("nan", "inf", "-inf", "+inf", "infinity"):
            raise ValueError
        if field_text.startswith("+"):
            raise ValueError  # from_chars rejects a leading '+'
        return float(field_text)
    except ValueError:
        raise ParseError(f"line {line_no}: bad {column} value '{field_text}'") from None


# ---- raw series and cleaning (timeseries.cpp) ---------------------------------------------

@dataclass
class RawRecord:
    date: _dt.date
    confirmed_cum: Optional[float] = None
    recovered_cum: Optional[float] = None
    deaths_cum: Optional[float] = None


@dataclass
class CleaningStats:
    interpolated_cells: int = 0
    negative_corrections: int = 0
    outflow_corrections: int = 0


@dataclass
class Series:
    """EpiSeries (timeseries.hpp:37-46) with its calendar start."""
    start_date: _dt.date
    infectious: list
    recovered_cum: list
    deaths_cum: list
    new_cases: list

    def size(self) -> int:
        return len(self.infectious)

    def date_at(self, day: int) -> _dt.date:
        return self.start_date + _dt.timedelta(days=day)


_COLUMNS = ("confirmed_cum", "recovered_cum", "deaths_cum")
_COLUMN_NAMES = ("confirmed", "recovered", "deaths")


def _strip(s: str) -> str:
    return s.strip(" \t\r")


def read_raw_csv(text: str) -> list:
    """read_raw_csv (csv.cpp:96-128): header date,confirmed,recovered,deaths."""
    lines = text.split("\n")
    if text == "" or not lines:
        raise ParseError("line 1: empty input")
    header = lines[0].rstrip("\r")
    want = ["date", "confirmed", "recovered", "deaths"]
    got = header.split(",")
    if len(got) != len(want) or any(_strip(g) != w for g, w in zip(got, want)):
        raise ParseError("line 1: expected header 'date,confirmed,recovered,deaths'")
    records = []
    if text.endswith("\n"):
        lines = lines[:-1]
    for line_no, line in enumerate(lines[1:], start=2):
        line = line[:-1] if line.endswith("\r") else line
        if _strip(line) == "":
            continue
        fields = line.split(",")
        if len(fields) != 4:
            raise ParseError(f"line {line_no}: expected 4 fields, got {len(fields)}")
        try:
            date = parse_date(_strip(fields[0]))
        except ParseError as e:
            raise ParseError(f"line {line_no}: {e}") from None
        vals = []
        for f, name in zip(fields[1:], _COLUMN_NAMES):
            f = _strip(f)
            vals.append(None if f == "" else parse_number(f, line_no, name))
        records.append(RawRecord(date, *vals))
    validate_raw(records)
    return records


def read_raw_csv_file(path: str) -> list:
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise Error(f"cannot open '{path}'") from None
    try:
        return read_raw_csv(text)
    except ParseError as e:
        raise ParseError(f"{path}: {e}") from None


def validate_raw(records: list) -> None:
    """RawSeries::validate (timeseries.cpp:31-48)."""
    if not records:
        raise EmptySeriesError()
    for k, rec in enumerate(records):
        if k > 0 and rec.date <= records[k - 1].date:
            raise ParseError(f"dates must be strictly increasing (violated at {format_date(rec.date)})")
        for col, name in zip(_COLUMNS, _COLUMN_NAMES):
            v = getattr(rec, col)
            if v is not None and (not math.isfinite(v) or v < 0.0):
                raise ParseError(f"{name} at {format_date(rec.date)} is negative or not finite")


def interpolate_missing(records: list, stats: Optional[CleaningStats] = None) -> list:
    """timeseries.cpp:50-90: daily grid, linear interpolation of interior gaps."""
    validate_raw(records)
    first, last = records[0].date, records[-1].date
    n = (last - first).days + 1
    grid = [RawRecord(first + _dt.timedelta(days=d)) for d in range(n)]
    for rec in records:
        grid[(rec.date - first).days] = RawRecord(rec.date, rec.confirmed_cum, rec.recovered_cum, rec.deaths_cum)
    for col, name in zip(_COLUMNS, _COLUMN_NAMES):
        if getattr(grid[0], col) is None or getattr(grid[-1], col) is None:
            raise MissingEndpointError(f"column '{name}' has no value at the first or last date")
        prev = 0
        for day in range(1, n):
            if getattr(grid[day], col) is None:
                continue
            if day > prev + 1:
                lo = getattr(grid[prev], col)
                hi = getattr(grid[day], col)
                slope = (hi - lo) / float(day - prev)
                for k in range(prev + 1, day):
                    setattr(grid[k], col, lo + slope * float(k - prev))
                    if stats:
                        stats.interpolated_cells += 1
            prev = day
    return grid


def daily_from_cumulative(cumulative: list, stats: Optional[CleaningStats] = None) -> list:
    """timeseries.cpp:92-109."""
    daily = [0.0] * len(cumulative)
    if not cumulative:
        return daily
    daily[0] = cumulative[0]
    for k in range(1, len(cumulative)):
        daily[k] = cumulative[k] - cumulative[k - 1]
    for k in range(len(daily)):
        if daily[k] < 0.0:
            daily[k] = daily[k - 1] if k > 0 else 0.0
            if stats:
                stats.negative_corrections += 1
    return daily


def moving_average7(values: list) -> list:
    """timeseries.cpp:111-123 (trailing window, running sum in this order)."""
    out = [0.0] * len(values)
    window_sum = 0.0
    for k, v in enumerate(values):
        window_sum += v
        if k >= SMOOTHING_WINDOW:
            window_sum -= values[k - SMOOTHING_WINDOW]
        out[k] = window_sum / float(min(k + 1, SMOOTHING_WINDOW))
    return out


def build_epi_series(records: list, stats: Optional[CleaningStats] = None) -> Series:
    """timeseries.cpp:125-169."""
    grid = interpolate_missing(records, stats)
    n = len(grid)
    confirmed = [r.confirmed_cum for r in grid]
    recovered = [r.recovered_cum for r in grid]
    deaths = [r.deaths_cum for r in grid]
    new_cases = daily_from_cumulative(confirmed, stats)
    recovered_daily = daily_from_cumulative(recovered, stats)
    deaths_daily = daily_from_cumulative(deaths, stats)
    infectious = [0.0] * n
    first = new_cases[0] - recovered_daily[0] - deaths_daily[0]
    infectious[0] = first if 0.0 < first else 0.0  # std::max(0.0, x)
    for t in range(1, n):
        nxt = infectious[t - 1] + new_cases[t] - recovered_daily[t] - deaths_daily[t]
        if nxt < 0.0:
            deficit = -nxt
            from_recovered = deficit if deficit < recovered_daily[t] else recovered_daily[t]  # std::min
            recovered_daily[t] -= from_recovered
            deficit -= from_recovered
            deaths_daily[t] -= deficit if deficit < deaths_daily[t] else deaths_daily[t]
            nxt = 0.0
            if stats:
                stats.outflow_corrections += 1
        infectious[t] = nxt
    rec_cum, dea_cum = [0.0] * n, [0.0] * n
    acc_r = acc_d = 0.0
    for t in range(n):  # std::partial_sum
        acc_r = recovered_daily[t] if t == 0 else acc_r + recovered_daily[t]
        acc_d = deaths_daily[t] if t == 0 else acc_d + deaths_daily[t]
        rec_cum[t], dea_cum[t] = acc_r, acc_d
    return Series(grid[0].date, infectious, rec_cum, dea_cum, new_cases)


def smooth7(s: Series) -> Series:
    """timeseries.cpp:171-179."""
    return Series(s.start_date, moving_average7(s.infectious), moving_average7(s.recovered_cum),
                  moving_average7(s.deaths_cum), moving_average7(s.new_cases))


def write_epi_csv(path: str, s: Series) -> None:
    """csv.cpp:142-149."""
    with open(path, "w") as f:
        f.write("date,infectious,recovered_cum,deaths_cum,new_cases\n")
        for t in range(s.size()):
            f.write(f"{format_date(s.date_at(t))},{format_double(s.infectious[t])},"
                    f"{format_double(s.recovered_cum[t])},{format_double(s.deaths_cum[t])},"
                    f"{format_double(s.new_cases[t])}\n")


def write_table(path: str, header: str, rows: list) -> None:
    """csv.cpp:203-217."""
    with open(path, "w") as f:
        f.write(header + "\n")
        for row in rows:
            f.write(",".join(row) + "\n")


# ---- envelopes (calibration.cpp:17-35, 218-296) ---------------------------------------------

def _finite_sorted(values: list) -> list:
    return sorted(v for v in values if math.isfinite(v))


def _median_sorted(s: list) -> float:
    k = len(s)
    if k % 2 == 1:
        return s[k // 2]
    return 0.5 * (s[k // 2 - 1] + s[k // 2])


@dataclass
class Envelope:
    count: list = field(default_factory=list)
    outer_lo: list = field(default_factory=list)
    outer_hi: list = field(default_factory=list)
    band1_lo: list = field(default_factory=list)
    band1_hi: list = field(default_factory=list)
    band2_lo: list = field(default_factory=list)
    band2_hi: list = field(default_factory=list)
    median: list = field(default_factory=list)

    def days(self) -> int:
        return len(self.count)


def build_envelope(values_per_day: list) -> Envelope:
    n = len(values_per_day)
    nan = math.nan
    env = Envelope([0] * n, *([nan] * n for _ in range(7)))
    for day, values in enumerate(values_per_day):
        s = _finite_sorted(values)
        k = len(s)
        env.count[day] = k
        if k == 0:
            continue
        env.outer_lo[day], env.outer_hi[day] = s[0], s[-1]
        env.band1_lo[day] = s[1] if k >= 3 else s[0]
        env.band1_hi[day] = s[k - 2] if k >= 3 else s[-1]
        if k >= 5:
            env.band2_lo[day], env.band2_hi[day] = s[2], s[k - 3]
        env.median[day] = _median_sorted(s)
    return env


def beta_at(p, t: float) -> float:
    """model.cpp:55-64 (host helper for the envelopes)."""
    if t < p.t1:
        return p.beta1
    if t >= p.t2:
        return p.beta2
    slope = (p.beta2 - p.beta1) / (p.t2 - p.t1)
    return p.beta1 + slope * (t - p.t1)


def parameter_envelopes(fits: list, n_days: int) -> dict:
    beta, gamma, mu, r0 = ([[] for _ in range(n_days)] for _ in range(4))
    for fit in fits:
        if not fit.ok:
            continue
        rate = fit.params.gamma + fit.params.mu
        for local in range(fit.window.length):
            day = fit.window.start + local
            if day >= n_days:
                break
            b = beta_at(fit.params, float(local))
            beta[day].append(b)
            gamma[day].append(fit.params.gamma)
            mu[day].append(fit.params.mu)
            r0[day].append(b / rate if rate > 0.0 else math.nan)
    return {"beta": build_envelope(beta), "gamma": build_envelope(gamma), "mu": build_envelope(mu),
            "r0": build_envelope(r0)}


def compartment_envelopes(fits: list, n_days: int) -> dict:
    I, R, D = ([[] for _ in range(n_days)] for _ in range(3))
    for fit in fits:
        if not fit.ok or fit.trajectory is None:
            continue
        for local in range(min(fit.window.length, fit.trajectory.days())):
            day = fit.window.start + local
            if day >= n_days:
                break
            s = fit.trajectory.states[local]
            I[day].append(s.I)
            R[day].append(s.R)
            D[day].append(s.D)
    return {"infectious": build_envelope(I), "recovered": build_envelope(R), "deaths": build_envelope(D)}
