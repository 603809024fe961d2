"""Device timeline of the C5 band pipeline (sg_forecast_ensemble_bands_batch).

CUPTI (through torch.profiler) records every kernel of the process with its
stream and device start/end, concurrent streams included, so this shows what
the serialised ncu launch list cannot: how much of the evaluation stream's
time the ordering / selection stream steals, and where the evaluation stream
idles.

    python tools/c5_timeline.py [n_windows] [--json out.json]
"""
import argparse
import collections
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_2204_12346_b200 as eng  # noqa: E402

I, R, D = bench.load_series()
N = bench.POPULATION


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("windows", type=int, nargs="?", default=24)
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--json", default="")
    args = ap.parse_args()
    ctx = eng.Context(0)
    wins = []
    for w in range(args.windows):
        a = w * bench.DELTA
        sl = slice(a, a + 36)
        wins.append(eng.Window(ctx, I[sl], R[sl], D[sl], [N - I[a] - R[a] - D[a], I[a], R[a], D[a]], N, bench.SPEC))
    upper = [2.0, 2.0, 28.0, 28.0, 1.0, 0.1]
    seeds = [bench.mix_seed(2204, w) for w in range(args.windows)]
    ctx.forecast_ensemble_bands_batch(wins[:2], [0] * 6, upper, seeds[:2], args.n, 21)  # warm (pool growth)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        ctx.forecast_ensemble_bands_batch(wins, [0] * 6, upper, seeds, args.n, 21)
        torch.cuda.synchronize()
    ev = _kernels(prof)
    # the same windows one call at a time on one stream: standalone durations
    with profile(activities=[ProfilerActivity.CUDA]) as prof1:
        for w in range(args.windows):
            wins[w].forecast_ensemble_bands([0] * 6, upper, seed=seeds[w], n=args.n, horizon=21)
        torch.cuda.synchronize()
    serial = collections.defaultdict(list)
    for x in _kernels(prof1):
        serial[x["name"]].append(x["end"] - x["start"])
    report(ev, args, {k: round(sum(v) / len(v), 1) for k, v in sorted(serial.items())})


def _kernels(prof):
    ev = []
    for e in prof.events():
        if e.device_type.name != "CUDA" or e.time_range.elapsed_us() <= 0:
            continue
        ev.append(dict(name=e.name.split("(")[0].split("<")[0].replace("void ", "").strip().split("::")[-1],
                       stream=getattr(e, "device_resource_id", None) or e.thread, start=e.time_range.start,
                       end=e.time_range.end))
    ev.sort(key=lambda x: x["start"])
    return ev


def report(ev, args, serial_us):
    t0, t1 = ev[0]["start"], max(x["end"] for x in ev)
    span = t1 - t0
    by = collections.defaultdict(lambda: [0, 0.0])
    streams = collections.defaultdict(float)
    for x in ev:
        by[(x["stream"], x["name"])][0] += 1
        by[(x["stream"], x["name"])][1] += x["end"] - x["start"]
        streams[x["stream"]] += x["end"] - x["start"]
    ens = [x for x in ev if x["name"] == "ensemble_kernel"]
    gaps = [b["start"] - a["end"] for a, b in zip(ens, ens[1:])]
    # time during which an ensemble kernel runs alone vs with another kernel
    edges = sorted([(x["start"], 1, x["name"] == "ensemble_kernel") for x in ev] +
                   [(x["end"], -1, x["name"] == "ensemble_kernel") for x in ev])
    alone = shared = other_only = idle = 0.0
    n_ens = n_oth = 0
    last = t0
    for t, d, is_ens in edges:
        dt = t - last
        if n_ens and n_oth:
            shared += dt
        elif n_ens:
            alone += dt
        elif n_oth:
            other_only += dt
        else:
            idle += dt
        last = t
        if is_ens:
            n_ens += d
        else:
            n_oth += d
    out = {"windows": args.windows, "n": args.n, "span_us": span, "per_window_us": span / args.windows,
           "ensemble_us_mean": sum(x["end"] - x["start"] for x in ens) / len(ens),
           "ensemble_gap_us_mean": sum(gaps) / max(1, len(gaps)), "ensemble_alone_us": alone,
           "ensemble_with_other_us": shared, "other_only_us": other_only, "idle_us": idle,
           "serial_mean_us": serial_us,
           "kernels": {f"{s}:{n}": {"launches": c, "us": round(t, 1)} for (s, n), (c, t) in sorted(by.items())}}
    print(json.dumps(out, indent=1))
    if args.json:
        Path(args.json).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
