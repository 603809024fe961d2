"""Summaries of the ncu captures for profiles/ (run here, on the .ncu-rep / CSV the GPU box wrote).

    python tools/summarize_profiles.py launches gpurun_out/X_launches.csv --tag r01b --cmd "..."
        -> profiles/<tag>_launches_summary.md (per-kernel launch counts, total time, share)
    python tools/summarize_profiles.py step gpurun_out/X.ncu-rep --tag r01b --cmd "..." --note "..."
        -> profiles/ncu_step_kernel_<tag>.json (time, DRAM bytes, pipe %, stalls, per-particle bytes)
"""
import argparse
import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"


def launches(path, tag, cmd):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in data:
        name = r[ik].split("(")[0]
        tot[name] += float(r[iv]) / 1e3
        cnt[name] += 1
    s = sum(tot.values())
    out = [f"# {tag} launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
           f"Command: `{cmd}` (per-launch, serialised, cold).", f"Raw list: `profiles/{Path(path).name}`.", "",
           "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for name, us in tot.most_common():
        out.append(f"| `{name}` | {cnt[name]} | {us:.1f} | {100 * us / s:.1f}% |")
    (PROF / f"{tag}_launches_summary.md").write_text("\n".join(out) + "\n")
    print("\n".join(out))


def raw_metrics(rep):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
             "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0, "hz": 1.0, "Khz": 1e3,
             "Mhz": 1e6, "Ghz": 1e9}
    out = {}
    for k, unit, v in zip(rows[0], rows[1], rows[2]):
        try:
            out[k] = float(v.replace(",", "")) * scale.get(unit, 1.0)
        except ValueError:
            out[k] = None
    return out  # SI units (bytes, seconds, Hz)


def opcode_mix(rep):
    """Executed warp-level instructions per opcode from the SASS source page."""
    import re
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[1]
    ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    ops = collections.Counter()
    for r in rows[2:]:
        n = int(r[ia] or 0)
        mt = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[isrc].strip())
        if n and mt:
            ops[mt.group(2)] += n
    return ops


def step(rep, tag, cmd, note, kernel, prefix="ncu_step_kernel"):
    m = raw_metrics(rep)
    ops = opcode_mix(rep)

    def f(k):
        return m.get(k)

    grid = int(f("launch__grid_size"))
    block = int(f("launch__block_size"))
    particles = grid * block
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(f(k)) for k in m
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and f(k)}
    d = {"round": 1, "tag": tag, "command": cmd, "kernel": kernel, "grid_ctas": grid,
         "particles_in_launch": particles, "gpu_time_s": f("gpu__time_duration.sum"),
         "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
         "fp64_pipe_active_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
         "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
         "warps_active_per_sm": f("sm__warps_active.avg.per_cycle_active"),
         "registers_per_thread": f("launch__registers_per_thread"),
         "instructions_executed": f("smsp__inst_executed.sum"),
         "sm_clock_ghz": (f("smsp__cycles_elapsed.avg.per_second") or 0) / 1e9,
         "stall_samples": dict(sorted(stalls.items())),
         "dram_bytes_per_particle": (rd + wr) / particles,
         # each warp instruction is one op per lane: per-particle op counts
         "fp64_ops_per_particle_executed": 32.0 * sum(ops[k] for k in ("DADD", "DMUL", "DFMA", "DSETP")) / particles,
         "other_ops_per_particle_executed": 32.0 * sum(v for k, v in ops.items()
                                                       if k not in ("DADD", "DMUL", "DFMA", "DSETP")) / particles,
         "note": note}
    out = PROF / f"{prefix}_{tag}.json"
    out.write_text(json.dumps(d, indent=1) + "\n")
    print(json.dumps(d, indent=1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["launches", "step", "ensemble"])
    ap.add_argument("path")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--cmd", default="")
    ap.add_argument("--note", default="")
    ap.add_argument("--kernel", default="pso_step_kernel<1,0,24> (ird-mxse, 24 substeps)")
    a = ap.parse_args()
    if a.what == "launches":
        launches(a.path, a.tag, a.cmd)
    else:
        step(a.path, a.tag, a.cmd, a.note, a.kernel,
             prefix="ncu_ensemble_kernel" if a.what == "ensemble" else "ncu_step_kernel")


if __name__ == "__main__":
    sys.exit(main())
