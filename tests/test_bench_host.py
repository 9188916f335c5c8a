"""CPU tests of bench.py's host logic: the chunking of the device run (equal
chunks at kernel boundaries, as few as fit under the cap) and the reference
arm's JSON line contract."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


@pytest.mark.parametrize("total,cap,want", [(19_160_000_000, 3 << 30, 6), (10_000, 3 << 30, 1),
                                            (7_000_000, 1_000_000, 7), (7_000_001, 1_000_000, 8)])
def test_chunks_equal_and_capped(total, cap, want):
    offs = np.linspace(0, total, 4001).astype(np.int64)  # 4000 kernels of equal size
    starts = bench.chunk_starts_from(offs, cap)
    assert starts[0] == 0 and len(starts) == want
    assert all(s in set(offs.tolist()) for s in starts)  # kernel boundaries only
    sizes = np.diff(starts + [total])
    kernel = total // 4000 + 1
    assert sizes.max() <= cap + kernel
    assert sizes.max() - sizes.min() <= 2 * kernel + (total // want) // 50


def test_reference_arm_line(tmp_path):
    """--impl reference prints one JSON line with the contract's keys (a tiny
    sample; the full arm runs for minutes)."""
    from oracle import oracle as O
    if not O.available():
        pytest.skip("oracle not built")
    code = ("import sys, bench; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','0'];"
            "args = bench.parse(); orig = bench._ref_sample;"
            "bench._ref_sample = lambda cfg, s, n, cap: orig(cfg, 0.01, min(n, 2), 64);"
            "bench.run_reference(args);"
            "maps = open('/proc/self/maps').read();"
            "print('PRODUCT_LOADED' if 'libocldec_b200' in maps else 'PRODUCT_NOT_LOADED',"
            " 'ORACLE_LOADED' if 'libocldec_ref' in maps else 'ORACLE_NOT_LOADED', file=sys.stderr)")
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    # the reference arm times the reference alone: the product library is
    # never loaded into that process
    assert "PRODUCT_NOT_LOADED" in p.stderr and "ORACLE_LOADED" in p.stderr, p.stderr[-500:]
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks
    (torch.distributed.run, 127.0.0.1): the reference arm prints one line from
    rank 0 and both ranks exit 0."""
    from oracle import oracle as O
    if not O.available():
        pytest.skip("oracle not built")
    env = dict(os.environ, OCLDEC_BENCH_REF_SECONDS="0.02")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "0", "--config", "C3"], cwd=ROOT, capture_output=True, text=True,
                       timeout=600, env=env)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(x) for x in p.stdout.strip().splitlines() if x.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


def test_stream_mode_accumulates_steps(capsys):
    """run_stream (the C5 streamed bench) over several steps: the per-step
    totals add up and the line reports them per step (a fake session: the
    host logic only)."""
    import types

    class FakeSession:
        def __init__(self, dev):
            self.n = 0

        def run_generated(self, cfg, count, seed=1, k0=0, sample_stride=0, **kw):
            self.n += 1
            st = {"ms_decompile": 100.0, "ms_generate": 50.0, "ms_wall": 160.0, "instructions": 1000 * count,
                  "in_bytes": 30000 * count, "out_bytes": 15000 * count, "kernels": count, "chunks": 1,
                  "failed": 0, "goto_form": 0, "fallbacks": 0}
            return st, np.zeros(1, dtype=np.uint64), np.zeros(1, dtype=np.uint64)

        def close(self):
            pass

        def stats(self):
            return {"ms_parse": 10.0, "ms_front": 20.0, "ms_lower": 40.0, "ms_fold": 5.0, "ms_render": 20.0,
                    "ms_emit": 1.0}

    fake_p = types.SimpleNamespace(Session=FakeSession)
    fake_torch = types.SimpleNamespace(cuda=types.SimpleNamespace(synchronize=lambda: None))
    args = types.SimpleNamespace(config="C5", steps=3, warmup=0, no_e2e=True, no_cpu=True)
    bench.run_stream(args, fake_p, fake_torch, None, 1, 0, 0, 5000)
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["steps"] == 3 and line["ms_per_step"] == 100.0
    assert line["passes_ms_per_step_rank0"]["k_lower"] == 40.0
    assert line["value"] == 5000 * 1000 / 0.1
