"""Turn ncu output fetched from the GPU box into the committed summaries under profiles/.

    python scripts/make_profiles.py --round r01 \
        --launches gpurun_out/launches.csv      # ncu --metrics gpu__time_duration.sum,... --csv
        --full gpurun_out/prof_full.ncu-rep     # ncu --set full capture

Writes profiles/<round>_launches.txt (per-kernel launch counts, time and share of the
profiled step), profiles/<round>_ncu_full.txt (key metrics of every launch of the full
capture) and profiles/traffic.json (DRAM bytes per launch by kernel, read by bench.py for
roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
        "us": 1.0, "msecond": 1e3, "ms": 1e3, "ns": 1e-3}
FULL_KEYS = ("gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
             "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
             "sm__inst_executed.sum", "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
             "smsp__issue_active.avg.pct_of_peak_sustained_active",
             "sm__warps_active.avg.pct_of_peak_sustained_active",
             "lts__t_sector_hit_rate.pct", "dram__bytes_read.sum", "dram__bytes_write.sum",
             "dram__throughput.avg.pct_of_peak_sustained_elapsed",
             "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed")


def short(name):
    return name.split("(")[0].split("::")[-1]


def launches(path):
    """Rows of an ncu --csv --metrics log: one row per (launch, metric)."""
    text = open(path).read()
    text = text[text.index('"ID"'):]
    per = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO(text)):
        d = per.setdefault(int(r["ID"]), {"name": short(r["Kernel Name"]),
                                          "grid": r["Grid Size"], "block": r["Block Size"]})
        v = float(r["Metric Value"].replace(",", "") or 0) * UNIT.get(r["Metric Unit"], 1.0)
        d[r["Metric Name"]] = v
    return per


def launch_table(per, title):
    agg = collections.OrderedDict()
    for d in per.values():
        grid = d["grid"].strip("()").replace(", 1, 1", "").replace(" ", "")
        a = agg.setdefault(f"{d['name']} [{grid}]", {"n": 0, "us": 0.0, "rd": 0.0, "wr": 0.0})
        a["n"] += 1
        a["us"] += d.get("gpu__time_duration.sum", 0.0)
        a["rd"] += d.get("dram__bytes_read.sum", 0.0)
        a["wr"] += d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["us"] for a in agg.values()) or 1.0
    lines = [title, "", f"{'kernel (grid)':40s} {'launches':>8s} {'total us':>11s} {'mean us':>9s} "
             f"{'share':>6s} {'DRAM rd MB/launch':>18s} {'DRAM wr MB/launch':>18s}"]
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        lines.append(f"{k:40s} {a['n']:8d} {a['us']:11.1f} {a['us'] / a['n']:9.2f} "
                     f"{a['us'] / tot * 100:5.1f}% {a['rd'] / a['n'] / 1e6:18.3f} "
                     f"{a['wr'] / a['n'] / 1e6:18.3f}")
    lines.append(f"{'total':40s} {sum(a['n'] for a in agg.values()):8d} {tot:11.1f}")
    return "\n".join(lines) + "\n"


def full_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"name": short(r[hdr.index("Kernel Name")])}
        for k in FULL_KEYS:
            if k in hdr:
                i = hdr.index(k)
                try:
                    d[k] = float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0)
                except ValueError:
                    d[k] = r[i]
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--launches-title", default="")
    ap.add_argument("--full")
    ap.add_argument("--full-title", default="")
    ap.add_argument("--kc-metrics", help="ncu --csv --metrics log of the KC update launches "
                    "(sm__inst_executed.sum, dram bytes, time) -> profiles/kc_update_ncu.json")
    ap.add_argument("--kc-neurons", type=int, default=100_000)
    ap.add_argument("--kc-steps", type=int, default=256)
    ap.add_argument("--kc-source", default="")
    a = ap.parse_args()
    pdir = os.path.join(ROOT, "profiles")
    os.makedirs(pdir, exist_ok=True)
    if a.launches:
        per = launches(a.launches)
        with open(os.path.join(pdir, f"{a.round}_launches.txt"), "w") as f:
            f.write(launch_table(per, a.launches_title or f"ncu launch list ({a.launches})"))
    if a.kc_metrics:
        per = launches(a.kc_metrics)
        kc = [d for d in per.values() if d["name"].startswith("condlif_")
              and int(d["grid"].strip("()").split(",")[0]) > 1]
        inst = sorted(d["sm__inst_executed.sum"] for d in kc)
        med = inst[len(inst) // 2]
        rw = sorted(d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
                    for d in kc)
        us = sorted(d.get("gpu__time_duration.sum", 0.0) for d in kc)
        clk = [d.get("sm__cycles_elapsed.avg.per_second", 0.0) for d in kc]
        out = {"round": a.round, "source": a.kc_source or os.path.basename(a.kc_metrics),
               "kernel": f"{kc[0]['name']} (KC update, multi-block)", "launches": len(kc),
               "neurons": a.kc_neurons, "steps_per_launch": a.kc_steps,
               "warp_inst_per_launch_median": med,
               "warp_inst_per_neuron_step": med / (a.kc_neurons * a.kc_steps),
               "dram_bytes_per_launch": rw[len(rw) // 2],
               "us_per_launch_median_cold_serialised": us[len(us) // 2],
               "sm_mhz": (sum(clk) / len(clk) / 1e6) if clk and clk[0] else None,
               "note": "sm__inst_executed.sum = warp instructions issued; bench.py's issue "
                       "roofline scales warp_inst_per_neuron_step by the live launch's "
                       "neuron-steps"}
        with open(os.path.join(pdir, "kc_update_ncu.json"), "w") as f:
            json.dump(out, f, indent=1)
    if a.full:
        rows = full_rows(a.full)
        lines = [a.full_title or f"ncu --set full ({a.full})", ""]
        traffic = {}
        for i, d in enumerate(rows):
            lines.append(f"[{i}] {d['name']}")
            for k in FULL_KEYS:
                if k in d:
                    v = d[k]
                    lines.append(f"    {k:62s} {v:.6g}" if isinstance(v, float) else
                                 f"    {k:62s} {v}")
            rw = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
            traffic.setdefault(d["name"], []).append(rw)
        with open(os.path.join(pdir, f"{a.round}_ncu_full.txt"), "w") as f:
            f.write("\n".join(lines) + "\n")
        tpath = os.path.join(pdir, "traffic.json")
        tj, src = {}, []
        if os.path.exists(tpath):  # merge: later captures override earlier ones per kernel
            with open(tpath) as f:
                old = json.load(f)
            tj, src = old.get("bytes_per_launch", {}), old.get("sources", [])
        tj.update({k: max(v) for k, v in traffic.items()})
        src.append(os.path.basename(a.full))
        with open(tpath, "w") as f:
            json.dump({"sources": src, "round": a.round,
                       "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch "
                               "(max over captured launches of the kernel), ncu --set full",
                       "bytes_per_launch": tj}, f, indent=1)


if __name__ == "__main__":
    main()
