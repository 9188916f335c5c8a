"""Fills k_fold's entries of dram_traffic.json / dataflow_ncu.json from a
targeted-metric ncu capture (tools/final_profiles_r2b.sh: k_fold_metrics.csv),
because k_fold's `ncu --set full` replay returns nan for its counters.
    python tools/fold_traffic.py OUTDIR    (reads OUTDIR/k_fold_metrics.csv)"""
import csv
import json
import math
import os
import sys

o = sys.argv[1]
rows = [r for r in csv.reader(open(os.path.join(o, "k_fold_metrics.csv"), errors="replace")) if len(r) > 10]
hdr = rows[0]
ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value")}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1, "%": 1, "": 1}
first = None
vals = {}
for r in rows[1:]:
    if "k_fold" not in r[ix["Kernel Name"]]:
        continue
    if first is None:
        first = r[ix["ID"]]
    if r[ix["ID"]] != first:
        continue
    try:
        vals[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1)
    except ValueError:
        vals[r[ix["Metric Name"]]] = float("nan")
tp = os.path.join(o, "dram_traffic.json")
t = json.load(open(tp))
base = t.get("k_lower") or next(iter(t.values()))
ninstr = base["sample_instructions"]
b = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
t["k_fold"] = {"dram_bytes": b, "dram_bytes_per_instr": b / ninstr, "algorithmic_bytes": base["algorithmic_bytes"],
               "sample_instructions": ninstr, "ncu_duration_s": vals["gpu__time_duration.sum"],
               "source": "k_fold_metrics.csv (ncu --metrics, C4 sample, first launch; --set full returns nan)"}
json.dump(t, open(tp, "w"), indent=1)
dp = os.path.join(o, "dataflow_ncu.json")
if os.path.exists(dp):
    d = json.load(open(dp))
    c4 = next((v for k, v in d.items() if k.startswith("C4") and isinstance(v, dict)), None)
    if c4 is not None:
        c4["k_fold"] = {"achieved_occupancy_pct": vals.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
                        "active_threads_per_warp": vals.get("smsp__thread_inst_executed_per_inst_executed.ratio"),
                        "branch_efficiency_pct": vals.get("smsp__sass_average_branch_targets_threads_uniform.pct"),
                        "issue_slots_busy_pct": None, "duration_ms": vals["gpu__time_duration.sum"] * 1e3}
        json.dump({k: v for k, v in d.items()}, open(dp, "w"), indent=1)
print(json.dumps(t["k_fold"]))
