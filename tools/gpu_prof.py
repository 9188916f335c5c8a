"""Phase profile of the decompile kernel (OCLDEC_B200_PROF=1): SM cycles per
phase summed over all kernels, plus pass timings.  Developer aid."""
import json
import os
import sys
import time

os.environ["OCLDEC_B200_PROF"] = "1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2107_07809_b200 as P  # noqa: E402
import bench  # noqa: E402

cfg = sys.argv[1]
nk = int(sys.argv[2])
s = P.Session(0)
d_buf, n, d_offs, ni = s.generate(cfg, nk, seed=bench.SEEDS[cfg])
offs = np.empty(nk + 1, dtype=np.uint64)
P.copy(offs.ctypes.data, d_offs, (nk + 1) * 8)
starts = bench.chunk_starts_from(offs)
for i in range(2):
    t = time.time()
    s.run(d_buf, n, starts)
    dt = time.time() - t
st = s.stats()
names = ["config+abi", "cfg", "normalize", "regions+reduce", "liveness", "pools", "lowering", "emit", "fold"]
tot = sum(st["prof_cycles"][:9]) or 1
print(json.dumps({"cfg": cfg, "kernels": nk, "instr": ni, "wall_s": dt, "instr_per_s": ni / dt,
                  "ms": {k: st[k] for k in ("ms_parse", "ms_decompile", "ms_emit", "ms_front", "ms_lower", "ms_fold", "ms_render")},
                  "launches": st["decompile_launches"], "retried": st["retried"],
                  "phase_share": {names[i]: round(st["prof_cycles"][i] / tot, 4) for i in range(9)},
                  "cycles_per_instr": tot / ni}))
