"""Summaries of an ncu report: per-launch key metrics, and the SASS lines with
the most warp-stall samples for one launch.

    python scripts/ncu_summary.py REPORT [--id N] [--top K]
"""
import argparse
import csv
import io
import subprocess

KEYS = ("Duration", "Grid Size", "Block Size", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Executed Ipc Active", "Issue Slots Busy",
        "Achieved Occupancy", "L2 Hit Rate", "DRAM Throughput", "Memory Throughput")


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def details(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "details", "--csv"))))
    hdr = rows[0]
    ii, ki, mi, vi, ui = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name",
                                                 "Metric Value", "Metric Unit"))
    out = {}
    for r in rows[1:]:
        d = out.setdefault(int(r[ii]), {"name": r[ki].split("(")[0].split("::")[-1]})
        if r[mi] in KEYS:
            d[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    return out


def sass_hotspots(rep, launch, top):
    text = ncu("-i", rep, "--page", "source", "--csv", "--print-source=sass", "--launch-skip",
               str(launch), "--launch-count", "1")
    rows = list(csv.reader(io.StringIO(text)))
    hdr = rows[1]
    ai, si = hdr.index("Address"), hdr.index("Source")
    ws, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")

    def f(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    seen, out = set(), []
    for r in rows[2:]:
        if len(r) <= ie or not r[ai].startswith("0x") or r[ai] in seen:
            continue
        seen.add(r[ai])
        out.append((int(r[ai], 16), f(r[ie]), f(r[ws]), r[si].strip()))
    out.sort()
    base = out[0][0]
    tot = sum(x[2] for x in out) or 1.0
    print(f"  samples {tot:.0f}, warp-instructions {sum(x[1] for x in out):.0f}")
    for a, c, s, src in sorted(out, key=lambda x: -x[2])[:top]:
        print(f"  {a - base:#7x} exec {c:9.0f} stall {s / tot * 100:5.1f}%  {src[:80]}")


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--id", type=int, default=None)
    ap.add_argument("--top", type=int, default=12)
    a = ap.parse_args()
    d = details(a.report)
    for k in sorted(d):
        print(k, d[k].pop("name"), "|", "; ".join(f"{m}={v}" for m, v in d[k].items()))
    if a.id is not None:
        sass_hotspots(a.report, a.id, a.top)
