#!/usr/bin/env python
"""Benchmark: GCN instructions decompiled/sec (device-timed) on B200, next to
the reference CPU path on the box's host cores.

Workload (BASELINE.json configs[3], the single-GPU HBM-roofline config):
C4 = 1,000,000 synthetic GCN kernels (~500 instrs avg), generated on the
device by the counter-based generator (od_gen.cuh), resident in HBM.
A step = one decompilation pass over the whole corpus (parse -> CFG ->
structuring -> lowering -> emit -> combined_source gather).  The corpus
(~16 GB) is far larger than L2 (126 MB), so no flush is needed between steps.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N   (weak scaling: each rank
  decompiles its own 1M-kernel shard; one all_gather of offsets per step)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEEDS = {"C1": 1, "C2": 0x210707809C2, "C3": 0x210707809C3, "C4": 0x210707809C4, "C5": 0x210707809C5}
DEFAULT_KERNELS = {"C1": 1, "C2": 10_000, "C3": 10_000, "C4": 1_000_000, "C5": 1_000_000}
# Largest chunk the device run is cut into, at .kernel boundaries, in equal
# parts (OCLDEC_B200_CHUNK_BYTES overrides).  Each phase launch ends in a
# tail, so fewer, fuller chunks are faster (measured: 8 chunks 117, 6 chunks
# 121 M instr/s; 6 -> 5 chunks at 3.6 GiB: 136.1 -> 137.0).  The synthetic
# corpus has no comment-stripped lines; the library's limit is 3.75 GiB.
CHUNK_BYTES = int(os.environ.get("OCLDEC_B200_CHUNK_BYTES", 0) or 0) or 0xE6666666
METRIC = "GCN instructions decompiled/sec (device-timed) at 1/2/4/8 B200 vs host CPU"


SEMANTIC_SEED = 0x5E3A171C


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=list(SEEDS))
    ap.add_argument("--kernels", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--semantic", action="store_true",
                    help="also time the decompile step with the batched semantic check (SURVEY §8(f) rank 4)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--stream", action="store_true",
                    help="generate-and-decompile chunk by chunk (default for C5, whose corpus exceeds HBM)")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(int(float(s[0])) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((int(float(s[1])) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


def dataflow_profile():
    """the dataflow pass is judged on occupancy and branch
    efficiency.  ncu numbers of the phase kernels (tools/dataflow_json.py,
    from the final build's --set full captures), never measured in this run."""
    p = os.path.join(ROOT, "profiles", "dataflow_ncu.json")
    if not os.path.exists(p):
        return None
    def clean(o):  # NaN (a counter ncu could not collect) as null: the line stays strict JSON
        if isinstance(o, float) and o != o:
            return None
        return {k: clean(v) for k, v in o.items()} if isinstance(o, dict) else o
    d = clean(json.load(open(p)))
    d["source"] = "profiles/dataflow_ncu.json (ncu --set full of the phase kernels, C4 / C5 samples)"
    return d


def pass_roof(nbytes, ms, peak):
    """Achieved GB/s of a byte-stream pass (algorithmic bytes / device time)."""
    gbs = nbytes / (ms / 1000.0) / 1e9 if ms else None
    return {"achieved": gbs, "unit": "GB/s", "peak": peak, "frac": gbs / peak if gbs else None,
            "bytes_per_step": nbytes, "ms_per_step": ms}


def chunk_starts_from(offsets, target=CHUNK_BYTES):
    """Chunk starts at kernel offsets: as few chunks of at most `target`
    bytes as fit, of about equal size."""
    import numpy as np
    offs = np.asarray(offsets, dtype=np.int64)
    total = int(offs[-1]) if len(offs) else 0
    nch = max(1, -(-total // target))
    target = -(-total // nch)
    starts = [0]
    nxt = target
    while True:
        k = int(np.searchsorted(offs, nxt, side="left"))
        if k >= len(offs) - 1:
            break
        if offs[k] <= starts[-1]:
            k += 1
            if k >= len(offs) - 1:
                break
        starts.append(int(offs[k]))
        nxt = starts[-1] + target
    return starts


def cpu_model():
    """CPU model string of this host (/proc/cpuinfo)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _ref_sample(cfg, seconds, nthreads, cap):
    """A deterministic sample (kernels 0..n-1 of the config's corpus at its
    bench seed) sized for about `seconds` of reference work on nthreads.
    Inputs come from the oracle library's host build of the generator, so
    the CPU arms never load the product library."""
    from oracle import oracle as O
    n = 64 if cfg in ("C2", "C3", "C4") else 2
    listing, offs, ni = O.generate_corpus(cfg, n, seed=SEEDS[cfg])
    secs, instrs, _, _ = O.decompile_batch(listing, offs, nthreads)
    per = max(ni / n, 1)
    n2 = max(n, min(int(instrs / max(secs, 1e-6) * seconds / per), cap))
    listing, offs, ni = O.generate_corpus(cfg, n2, seed=SEEDS[cfg])
    return listing, offs, ni, n2


def cpu_baseline(cfg, seconds, nthreads):
    """The reference (oracle/_ref, built from its sources) on host cores over a
    bounded deterministic sample of the same corpus: all host threads, then
    one thread on a smaller sample (SURVEY §8(d) CPU-baseline recipe)."""
    from oracle import oracle as O
    listing, offs, ni, n2 = _ref_sample(cfg, seconds, nthreads, 400_000)
    secs, instrs, _, _ = O.decompile_batch(listing, offs, nthreads)
    l1, o1, _, n1 = _ref_sample(cfg, max(2.0, seconds / 4), 1, 20_000)
    s1, i1, _, _ = O.decompile_batch(l1, o1, 1)
    return {"value": instrs / secs, "unit": "instr/s", "cores": nthreads, "kind": "reference",
            "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "sample": f"{n2} kernels of {cfg} (k=0..{n2 - 1}), {instrs} instrs, {len(listing)} bytes, "
                      f"{secs:.1f} s wall, decompile_listing per kernel on {nthreads} pthreads",
            "seconds": secs, "instructions": instrs, "in_bytes": len(listing),
            "one_thread": {"value": i1 / s1, "unit": "instr/s", "cores": 1,
                           "sample": f"{n1} kernels of {cfg} (k=0..{n1 - 1}), {i1} instrs, {s1:.1f} s wall"}}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation timed on the
    host cores, same metric/config; rank 0 only.  Loads only
    oracle/_ref/libocldec_ref.so (the reference compiled from its sources,
    plus the host build of the input generator): never the product."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    nthreads = os.cpu_count() or 1
    cfg = args.config
    # one step = a bounded sample (~6 s on the box's cores) of the config
    secs_step = float(os.environ.get("OCLDEC_BENCH_REF_SECONDS", "6.0"))
    listing, offs, ni, n_step = _ref_sample(cfg, secs_step, nthreads, 200_000)
    for _ in range(args.warmup):
        O.decompile_batch(listing, offs, nthreads)
    tot_s = tot_i = 0.0
    for _ in range(args.steps):
        secs, instrs, _, _ = O.decompile_batch(listing, offs, nthreads)
        tot_s += secs
        tot_i += instrs
    value = tot_i / tot_s
    sample = f"{n_step} kernels of {cfg} per step ({int(tot_i / args.steps)} instrs), {nthreads} pthreads"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "instr/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (counter-based generator)",
        "config": {"workload": f"{cfg} sample on host cores", "kernels_per_step": n_step},
        "cpu_baseline": {"value": value, "unit": "instr/s", "cores": nthreads, "kind": "reference",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": "instr/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-launch this command as N
    ranks (one process per GPU) under torch.distributed.run, rendezvous on
    127.0.0.1.  Returns only when no re-launch is needed."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def run_stream(args, P, torch, dist, world, rank, local, nk, cdev="cuda"):
    """Streaming mode (C5: 1M kernels x ~10k instructions, ~320 GB of
    listing, more than HBM): the fixed corpus [0, nk) is split across ranks by
    kernel index (strong scaling); each rank generates a chunk of its range
    on the device, decompiles it, and moves on (ocldec_b200_session_run_
    generated), so no whole-corpus buffer exists.  `value` counts the
    decompile passes' device time (parse + decompile + gather, CUDA events
    on the session stream, summed over chunks); the generator's time, which
    stands in for reading the input, is reported beside it
    (`value_incl_generation`).  Warm-up steps run on the rank's first 2,000
    kernels.  Every (nk/100)-th kernel's source hash is sampled for the CPU
    leg's parity check against the reference."""
    import numpy as np
    cfg = args.config
    k0 = nk * rank // world
    k1 = nk * (rank + 1) // world
    sess = P.Session(local)
    stride = max(1, nk // 100)  # (run_generated keeps only the sampled kernels' hashes)
    for _ in range(max(args.warmup, 3)):
        sess.run_generated(cfg, min(k1 - k0, 2000), seed=SEEDS[cfg], k0=k0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    acc = {"ms_decompile": 0.0, "ms_generate": 0.0, "ms_wall": 0.0}
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            st, hs, ls = sess.run_generated(cfg, k1 - k0, seed=SEEDS[cfg], k0=k0, sample_stride=stride)
            for key in ("ms_decompile", "ms_generate", "ms_wall"):
                acc[key] += st[key]
            ss = sess.stats()
            for key in ("ms_parse", "ms_front", "ms_lower", "ms_fold", "ms_render", "ms_emit"):
                acc[key] = acc.get(key, 0.0) + ss[key]
    torch.cuda.synchronize()
    tot = np.array([acc["ms_decompile"], acc["ms_wall"], st["instructions"], st["in_bytes"], st["out_bytes"],
                    st["kernels"]], dtype=np.float64)
    if world > 1:
        t = torch.tensor(tot[:2], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        u = torch.tensor(tot[2:], dtype=torch.float64, device=cdev)
        dist.all_reduce(u, op=dist.ReduceOp.SUM)
        tot = np.concatenate([t.cpu().numpy(), u.cpu().numpy()])
    ms_dec, ms_wall, ninstr, in_b, out_b, nker = tot
    peak, peak_src = measured_peaks()
    dec_s = ms_dec / 1000.0 / args.steps
    line = {
        "metric": METRIC, "value": ninstr * args.steps / (ms_dec / 1000.0), "unit": "instr/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_dec / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (counter-based GCN corpus generated on the device chunk by chunk)",
        "value_incl_generation": ninstr * args.steps / (ms_wall / 1000.0),
        "ms_per_step_incl_generation": ms_wall / args.steps,
        "config": {"workload": f"{cfg}: {int(nker)} kernels split over {world} GPU(s), {int(ninstr)} instrs, "
                               f"{int(in_b)} B in, {int(out_b)} B out, streamed in chunks of <= 3 GiB",
                   "kernels": int(nker), "instructions": int(ninstr), "in_bytes": int(in_b), "out_bytes": int(out_b),
                   "chunks_rank0": st["chunks"], "warmup_kernels_per_rank": min(k1 - k0, 2000),
                   "l2": "inputs (hundreds of GB) >> L2 (126 MB); no flush", "parallelism": f"dp{world} (kernel shards)"},
        "roofline": {"bound": "hbm", "achieved": (in_b + out_b) / dec_s / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": (in_b + out_b) / dec_s / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                     "kernel": "whole decompile pipeline (all passes)",
                     "algorithmic_bytes": "in+out text bytes of the corpus"},
        "clocks": clk.summary(),
        "stats": {k: st[k] for k in ("failed", "goto_form", "fallbacks")},
        "passes_ms_per_step_rank0": {name: acc[k] / args.steps for k, name in (
            ("ms_parse", "parse"), ("ms_front", "k_front"), ("ms_lower", "k_lower"), ("ms_fold", "k_fold"),
            ("ms_render", "k_emit"), ("ms_emit", "gather"))},
    }
    if rank == 0 and world == 1 and not args.no_e2e:
        # e2e on a bounded resident sample: the whole C5 listing does not fit
        # in host memory either
        ns = min(k1 - k0, 10_000)
        d_buf, nbytes, _, ni_s = sess.generate(cfg, ns, seed=SEEDS[cfg], k0=k0)
        host_in = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
        P.copy(host_in.data_ptr(), d_buf, nbytes)
        out_cap = int(nbytes * 1.5) + (1 << 20)
        host_out = torch.empty(out_cap, dtype=torch.uint8, pin_memory=True)
        sess.run_host(host_in.data_ptr(), nbytes, host_out.data_ptr(), out_cap)
        t0 = time.perf_counter()
        n_out = sess.run_host(host_in.data_ptr(), nbytes, host_out.data_ptr(), out_cap)
        t_e = time.perf_counter() - t0
        line["e2e"] = {"value": ni_s / t_e, "unit": "instr/s", "h2d_bytes_per_step": int(nbytes),
                       "d2h_bytes_per_step": int(n_out), "seconds_per_step": t_e,
                       "sample": f"first {ns} kernels of the rank's range (host-resident sample)",
                       "path": "ocldec_b200_session_run_host (pinned host in/out)"}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            from oracle import oracle as O
            ks = [k for k in range(k0, k1) if k % stride == 0]
            parts = [O.generate_corpus(cfg, 1, seed=SEEDS[cfg], k0=k) for k in ks]
            listing = b"".join(p_[0] for p_ in parts)
            offs = np.cumsum([0] + [len(p_[0]) for p_ in parts]).astype(np.uint64)
            nth = os.cpu_count() or 1
            secs, instrs, rh, rl = O.decompile_batch(listing, offs, nth, want_hashes=True)
            line["cpu_baseline"] = {
                "value": instrs / secs, "unit": "instr/s", "cores": nth, "kind": "reference",
                "cpu_model": cpu_model(), "sample": f"{len(ks)} kernels of {cfg} (every {stride}th), {instrs} instrs, "
                                                    f"{secs:.1f} s wall on {nth} pthreads"}
            line["parity_sample"] = {"kernels": len(ks), "source_hashes_equal": bool(np.array_equal(hs, rh)),
                                     "lengths_equal": bool(np.array_equal(ls, rl)),
                                     "checked_against": "oracle/_ref (the reference) per-kernel FNV-1a of source"}
        except Exception as ex:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    if rank == 0:
        print(json.dumps(line))
    sess.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    spawn_ranks(args)
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2107_07809_b200 as P
    from paper_2107_07809_b200 import dist as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU over NCCL; OCLDEC_BENCH_DIST=gloo runs the ranks'
    # exchange over gloo instead (several ranks on one GPU: a test of the
    # multi-rank path on a one-GPU box)
    backend = os.environ.get("OCLDEC_BENCH_DIST", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    cdev = "cuda" if backend == "nccl" else "cpu"  # the collectives' tensors
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = args.config
    nk = args.kernels or DEFAULT_KERNELS[cfg]
    if args.stream or cfg == "C5":
        run_stream(args, P, torch, dist, world, rank, local, nk, cdev)
        return
    sess = P.Session(local)
    # outputs of interest: combined_source (device; pinned host for e2e) and
    # the run's totals; per-kernel records stay on the device
    sess.set_records(False)
    stream = torch.cuda.ExternalStream(sess.stream_ptr, device=torch.device("cuda", local))
    # weak scaling: rank r decompiles kernels [r*nk, (r+1)*nk)
    d_buf, nbytes, d_offs, ninstr = sess.generate(cfg, nk, seed=SEEDS[cfg], k0=rank * nk)
    offs = torch.empty(nk + 1, dtype=torch.int64, device="cuda")
    host_offs = np.empty(nk + 1, dtype=np.uint64)
    # device offsets -> host (chunk boundaries at .kernel starts every ~1 GiB)
    P.copy(host_offs.ctypes.data, d_offs, (nk + 1) * 8)
    starts = chunk_starts_from(host_offs)

    def step():
        sess.run(d_buf, nbytes, starts, sync=False)
        st = sess.stats()
        if world > 1:
            # the one exchange step: every rank's {out_bytes, lines, split
            # error, kernels} -> its offset in the job's combined output
            st["placement"] = D.place(D.exchange(st["out_bytes"], st["lines"], 0, st["kernels"], device=cdev),
                                      rank)
        return st

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    ms_dec = 0.0
    ms_parse = 0.0
    ms_emit = 0.0
    ms_ph = {"k_front": 0.0, "k_lower": 0.0, "k_fold": 0.0, "k_emit": 0.0}
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            st = step()
            launches += st["total_launches"]
            ms_dec += st["ms_decompile"]
            ms_parse += st["ms_parse"]
            ms_emit += st["ms_emit"]
            ms_ph["k_front"] += st["ms_front"]
            ms_ph["k_lower"] += st["ms_lower"]
            ms_ph["k_fold"] += st["ms_fold"]
            ms_ph["k_emit"] += st["ms_render"]
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    ms_step = ms / args.steps
    total_instr = ninstr * world
    value = total_instr * args.steps / (ms / 1000.0)
    in_b, out_b = st["in_bytes"], st["out_bytes"]
    assert st["instructions"] == ninstr, (st["instructions"], ninstr)

    # ---- e2e through the C-ABI host-buffer call: H2D + pipeline + D2H
    e2e = None
    if not args.no_e2e:
        try:
            # N > 1: each rank's first 250k kernels (~4.8 GB of listing) keep
            # the job's pinned host memory bounded (N x 28 GB otherwise)
            e_nk = nk if world == 1 else min(nk, 250_000)
            e_bytes = int(host_offs[e_nk])
            e_instr = ninstr if e_nk == nk else None
            host_in = torch.empty(e_bytes, dtype=torch.uint8, pin_memory=True)
            P.copy(host_in.data_ptr(), d_buf, e_bytes)
            out_cap = int(out_b * (e_bytes / nbytes) * 1.1) + (1 << 20)
            host_out = torch.empty(out_cap, dtype=torch.uint8, pin_memory=True)
            e_steps = max(1, min(args.steps, 3))
            sess.run_host(host_in.data_ptr(), e_bytes, host_out.data_ptr(), out_cap)  # warm
            if e_instr is None:
                e_instr = sess.stats()["instructions"]
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(e_steps):
                n_out = sess.run_host(host_in.data_ptr(), e_bytes, host_out.data_ptr(), out_cap)
            t_e = (time.perf_counter() - t0) / e_steps
            e_total = e_instr
            if world > 1:
                t = torch.tensor([t_e], dtype=torch.float64, device=cdev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                t_e = float(t.item())
                u = torch.tensor([float(e_instr)], dtype=torch.float64, device=cdev)
                dist.all_reduce(u, op=dist.ReduceOp.SUM)
                e_total = float(u.item())
            e2e = {"value": e_total / t_e, "unit": "instr/s", "h2d_bytes_per_step": int(e_bytes),
                   "d2h_bytes_per_step": int(n_out), "seconds_per_step": t_e,
                   "path": "ocldec_b200_session_run_host (pinned host in/out)",
                   "kernels_per_gpu": e_nk}
            del host_in, host_out
        except Exception as ex:  # pragma: no cover
            e2e = {"value": None, "unit": "instr/s", "error": str(ex)[:200]}

    # ---- optional: the same step with the batched semantic check (8
    # environments per kernel, the reference's interpret_asm vs
    # evaluate_decompiled restated on the device), reported beside the line
    semantic = None
    if args.semantic:
        sess.set_semantic(True, SEMANTIC_SEED)
        step()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms_sem = e0.elapsed_time(e1) / args.steps
        counts = sess.semantic_counts()
        sess.set_semantic(False)
        extra = ms_sem - ms_step
        semantic = {"ms_per_step_with_check": ms_sem, "ms_per_step_check": extra,
                    "kernels_per_s_check": nk / (extra / 1000.0) if extra > 0 else None,
                    "envs_per_kernel": 8, "seed": SEMANTIC_SEED, "counts_last_step": counts}

    peak, peak_src = measured_peaks()
    # dominant kernel: the decompile phase launch with the most device time
    # (CUDA events around each launch on the session stream)
    dom = max(ms_ph, key=ms_ph.get)
    dom_s = ms_ph[dom] / 1000.0 / args.steps
    alg_bytes = in_b + out_b  # text in + text out of the kernels one launch set processes
    achieved = alg_bytes / dom_s / 1e9 if dom_s > 0 else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(prof):
        try:
            # per launch, like achieved: the step's instructions over the
            # dominant kernel's launches in the step
            per = json.load(open(prof)).get(dom, {}).get("dram_bytes_per_instr")
            traffic = per * ninstr / max(1, len(starts)) if per else None
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "instr/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (device-generated counter-based GCN corpus; byte-identical to the host generator)",
        "config": {"workload": f"{cfg}: {nk} kernels/GPU, {ninstr} instrs, {nbytes} B in, {out_b} B out",
                   "kernels_per_gpu": nk, "instructions_per_gpu": ninstr, "in_bytes": in_b,
                   "out_bytes": out_b, "chunks": len(starts), "l2": "inputs (16+ GB) >> L2 (126 MB); no flush",
                   "parallelism": f"dp{world} (kernel shards)"},
        "passes_ms_per_step": {"parse": ms_parse / args.steps, "decompile": ms_dec / args.steps,
                               "gather": ms_emit / args.steps,
                               **{k: v / args.steps for k, v in ms_ph.items()}},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "kernel": dom, "kernel_ms_per_step": ms_ph[dom] / args.steps, "peak_source": peak_src,
                     "algorithmic_bytes": "in+out text bytes of the kernels the launches process",
                     "algorithmic_bytes_per_launch": alg_bytes / max(1, len(starts)),
                     "traffic_source": "profiles/dram_traffic.json (ncu --set full dram__bytes per instruction "
                                       "on a C4 sample, scaled to one launch)" if traffic else None},
        # the byte-stream passes the north star judges against HBM: parse
        # (P1: listing text read once) and the combined_source gather (P4b:
        # staged text read + written once)
        "passes_roofline": {"parse": pass_roof(in_b, ms_parse / args.steps, peak),
                            # the emitter itself: k_emit renders out_bytes of OpenCL text
                            "emit": pass_roof(out_b, ms_ph["k_emit"] / args.steps, peak),
                            "gather": pass_roof(2 * out_b, ms_emit / args.steps, peak)},
        "dataflow": dataflow_profile(),
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": e2e,
        "stats": {k: st[k] for k in ("failed", "goto_form", "fallbacks", "retried", "lines")},
        "job_out_bytes": st["placement"].total_bytes if world > 1 else out_b,
    }
    if semantic:
        line["semantic"] = semantic
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_seconds, os.cpu_count() or 1)
        except Exception as ex:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": str(ex)[:200]}
    if rank == 0:
        print(json.dumps(line))
    sess.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
