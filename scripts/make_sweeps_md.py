"""profiles/<round>_sweeps.{md,jsonl} from the JSON lines of scripts/sweeps.py."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd, src = sys.argv[1], sys.argv[2]
rows = [json.loads(l) for l in open(src) if l.startswith("{")]
out = [f"# Sweeps ({rnd}, B200, `python scripts/sweeps.py density model blocks`)", "",
       "## Config 5, kernel level: propagate with all 100 rows spiking (100 x 100k, U(0, 0.02), seed 1234)",
       "",
       "Standalone `ssb_propagate_dense_dev` / `ssb_propagate_crs_dev` (tile bitmap fold) / "
       "`ssb_propagate_crs_sliced_dev` (column slices, r02) -- the reference's `propagate`, "
       "engine.cpp:53-80 -- CUDA events around one launch after a 256 MiB read that evicts the inputs "
       "from L2 (event resolution on this box is ~2 us).  Algorithmic bytes: dense = every weight once "
       "+ acc read/write; CRS = nnz x 8 (value + index) + segment table + acc; sliced = the slices "
       "(8 B per entry incl. padding) + acc.  All results are bit-identical to the row-ordered fold.", "",
       "| pn_kc density | nnz | dense us | dense GB/s (frac of peak) | CRS tile us | CRS tile GB/s (frac) "
       "| CRS sliced us | CRS sliced GB/s (frac) |",
       "|---|---|---|---|---|---|---|---|"]
by = {}
for r in rows:
    if r["sweep"] == "density_kernel":
        by.setdefault(r["frac"], {})[r["kernel"]] = r
for f, d in sorted(by.items()):
    D, S, Q = d["dense"], d["sparse"], d.get("sparse_sliced")
    assert D["bit_exact_vs_fold"] and S["bit_exact_vs_fold"]
    q = f"{Q['us']} | {Q['achieved_gbs']} ({Q['frac_of_peak']})" if Q else "- | -"
    out.append(f"| {f} | {D['nnz']} | {D['us']} | {D['achieved_gbs']} ({D['frac_of_peak']}) | "
               f"{S['us']} | {S['achieved_gbs']} ({S['frac_of_peak']}) | {q} |")
out += ["", "## Config 5, model level: 100k KC at pn_kc density f, 0.2 s simulated (W = 256)", "",
        "| f | KC rate Hz | ForceSparse us/step | ForceDense us/step | Auto us/step (layout) | sparse ev/s | dense ev/s |",
        "|---|---|---|---|---|---|---|"]
m = {}
for r in rows:
    if r["sweep"] == "density_model":
        m.setdefault(r["frac"], {})[r["mode"]] = r
for f, d in sorted(m.items()):
    S, D, A = d["ForceSparse"], d["ForceDense"], d.get("Auto")
    a = f"{A['us_per_step']} ({A.get('pn_kc_layout', '')})" if A else "-"
    out.append(f"| {f} | {S['kc_rate_hz']:.1f} | {S['us_per_step']} | {D['us_per_step']} | {a} | "
               f"{S['synaptic_events_per_s']:.3g} | {D['synaptic_events_per_s']:.3g} |")
out += ["", "All-to-all groups stored sparse (lhi_kc, kc_dn under ForceSparse) are detected "
        "(nnz = rows x posts) and use the dense kernels on the CRS values, which are the dense rows "
        "entry for entry; pn_kc uses the CRS tile pack inline.", "",
        "## Config 3: occupancy-chosen vs swept KC block sizes (0.23 s simulated, W = 256)", "",
        "| policy | KC block | us/step |", "|---|---|---|"]
for r in rows:
    if r["sweep"] == "blocks":
        out.append(f"| {r['policy']} | {r.get('kc_block', '-')} | {r.get('us_per_step', r.get('error'))} |")
with open(os.path.join(ROOT, "profiles", f"{rnd}_sweeps.md"), "w") as f:
    f.write("\n".join(out) + "\n")
with open(os.path.join(ROOT, "profiles", f"{rnd}_sweeps.jsonl"), "w") as f:
    for r in rows:
        f.write(json.dumps(r) + "\n")
