"""Where the e2e (host-buffer) step loses time against the device step: C4 1M.
Prints wall of run_host, its pass-event sums, the device-resident run, and the
bare PCIe copy rates of the same bytes."""
import json, time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2107_07809_b200 as P
import bench as B
nk = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
s = P.Session(0)
s.set_records(False)
d_buf, nbytes, d_offs, ninstr = s.generate("C4", nk, seed=B.SEEDS["C4"])
ho = np.empty(nk + 1, dtype=np.uint64)
P.copy(ho.ctypes.data, d_offs, (nk + 1) * 8)
starts = B.chunk_starts_from(ho)
host_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
P.copy(host_in.data_ptr(), d_buf, nbytes)
res = {}
for _ in range(2):
    s.run(d_buf, nbytes, starts, sync=True)
t0 = time.perf_counter(); s.run(d_buf, nbytes, starts, sync=True); res["dev_wall"] = time.perf_counter() - t0
st = s.stats(); res["dev_pass_sum_ms"] = st["ms_parse"] + st["ms_decompile"] + st["ms_emit"]
out_b = st["out_bytes"]
host_out = torch.empty(out_b + (1 << 24), dtype=torch.uint8, pin_memory=True)
s.run_host(host_in.data_ptr(), nbytes, host_out.data_ptr(), host_out.numel())
for i in range(2):
    t0 = time.perf_counter(); s.run_host(host_in.data_ptr(), nbytes, host_out.data_ptr(), host_out.numel())
    res[f"host_wall_{i}"] = time.perf_counter() - t0
st = s.stats(); res["host_pass_sum_ms"] = st["ms_parse"] + st["ms_decompile"] + st["ms_emit"]
res["host_stats"] = {k: v for k, v in st.items() if k.startswith("ms_")}
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); dev.copy_(host_in, non_blocking=True); torch.cuda.synchronize()
res["h2d_gbs"] = nbytes / (time.perf_counter() - t0) / 1e9
t0 = time.perf_counter(); host_out[:out_b].copy_(dev[:out_b], non_blocking=True); torch.cuda.synchronize()
res["d2h_gbs"] = out_b / (time.perf_counter() - t0) / 1e9
res["in_bytes"], res["out_bytes"] = nbytes, out_b
print(json.dumps(res))
