"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, agg = None, collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
                name = d["Kernel Name"].split("(")[0][:60]
                agg[name][0] += 1
                agg[name][1] += v
    tot = sum(v for _, v in agg.values())
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {c} | {v:.1f} | {100 * v / tot:.1f}% |")


if __name__ == "__main__":
    main()
