"""Markdown table of the bench lines under profiles/<round>/ (for DESIGN.md / README)."""
import glob
import json
import os
import sys

rd = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01"
rows = []
for f in sorted(glob.glob(os.path.join(rd, "bench_c*.json"))):
    d = json.load(open(f))
    r, s, e = d["roofline"], d["roofline_select"], d["e2e"]
    rows.append((d["config"]["workload"].split(":")[0], d["value"], d["ms_per_chunk"], e["value"],
                 e.get("ms_per_chunk"), e.get("pcie_bound_ms_per_chunk"),
                 r["kernel"].split("<")[0], r["achieved"], r["frac"], r["attn_ms_per_call"] * 1e3,
                 s["achieved"], s["frac"], s["select_plan_ms_per_call"] * 1e3,
                 d["config"].get("query_tiles", "128-row").split(" (")[0]))
print("| config | headline TFLOP/s | ms/chunk | e2e TFLOP/s (ms/chunk, PCIe bound) | query tiles | attn TFLOP/s (frac) | attn µs/call | pool GB/s (frac) | select+plan µs/call |")
print("|---|---|---|---|---|---|---|---|---|")
for c, v, ms, ev, ems, pb, k, a, fr, au, pg, pf, su, qt in rows:
    print(f"| {c} | {v:.0f} | {ms:.3f} | {ev:.0f} ({ems:.2f}, {pb:.2f}) | {qt} | {a:.0f} ({fr:.3f}) | {au:.0f} | "
          f"{pg:.0f} ({pf:.2f}) | {su:.0f} |")
