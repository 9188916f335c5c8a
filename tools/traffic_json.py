"""Writes profiles/dram_traffic.json from one `ncu --set full` capture of the
decompile phase kernels on a C4 sample (tools/final_profiles.sh): DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) per GCN instruction for each
kernel, so bench.py can report the measured traffic of the dominant kernel
per launch beside its algorithmic bytes.  Developer aid:
    python tools/traffic_json.py gpurun_out/final/phases.ncu-rep gpurun_out/final/ncu_phases.log"""
import csv
import io
import json
import os
import subprocess
import math
import sys

def _clean(o):
    """NaN (a counter ncu could not collect) as null: the files stay strict JSON."""
    if isinstance(o, float) and math.isnan(o):
        return None
    if isinstance(o, dict):
        return {k: _clean(v) for k, v in o.items()}
    return o


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, log = sys.argv[1], sys.argv[2]
ninstr = None
for line in open(log, errors="replace"):
    if line.startswith("{") and '"instructions_per_gpu"' in line:
        d = json.loads(line)
        ninstr = d["config"]["instructions_per_gpu"]
        in_b, out_b = d["config"]["in_bytes"], d["config"]["out_bytes"]
assert ninstr, "no bench line in the log"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
units = rows[1]
res = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
ki = hdr.index("Kernel Name")
for r in rows[2:]:
    name = r[ki].split("(")[0].split("::")[-1].strip()
    vals = {}
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        j = hdr.index(m)
        if units[j] not in scale:
            raise SystemExit(f"unknown ncu unit {units[j]!r} for {m}")
        try:
            vals[m] = float(r[j].replace(",", "")) * scale[units[j]]
        except ValueError:  # ncu reports n/a when a counter could not be collected
            vals[m] = None
    rd, wr = vals["dram__bytes_read.sum"], vals["dram__bytes_write.sum"]
    b = rd + wr if rd is not None and wr is not None else None
    res[name] = {"dram_bytes": b, "dram_bytes_per_instr": b / ninstr if b is not None else None,
                 "algorithmic_bytes": in_b + out_b, "sample_instructions": ninstr,
                 "ncu_duration_s": vals["gpu__time_duration.sum"],
                 "source": os.path.basename(rep) + " (ncu --set full, C4 sample, one launch)"}
dst = os.environ.get("OUT") or os.path.join(ROOT, "profiles", "dram_traffic.json")
json.dump(_clean(res), open(dst, "w"), indent=1)
print(json.dumps(_clean(res), indent=1))
