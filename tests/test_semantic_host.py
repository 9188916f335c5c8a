"""The device's semantic check, compiled for the host, against the reference.

tools/devhost.cpp builds the device pipeline headers (od_kernel.cuh ...
od_oracle.cuh) with g++ and, under OD_SEMCHECK, runs the batched semantic
check's per-environment interpreters (SemMachine: the listing, SemEval: the
decompiled body) on one lane at a time.  The reference's own interpret_asm /
evaluate_decompiled (proj/core/src/oracle.cpp, through oracle/ref_driver.cpp
ref_semcheck under OCLDEC_SEM_DEBUG) print the same environments' write
traces.  Every environment both sides ran must produce identical traces,
address by address and value by value.  Environments the device flags as
NaN-payload choices (SEM_INDETERMINATE, od_oracle.cuh sem_nan) are skipped:
there the host build follows x86 and the reference follows its compiler's
operand order.  No GPU needed; the GPU verdicts are pinned by
test_gpu_semantic.py.
"""
import os
import re
import subprocess
import sys

import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = "0x5E3A171C"
_LINE = re.compile(r"S (\d+) (\d+) asm (.*?)n=(\d+) \[(.*?)\] body (.*?)n=(\d+) \[(.*?)\]")

pytestmark = pytest.mark.skipif(not O.available(), reason="oracle not built")


@pytest.fixture(scope="module")
def devhost(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("devhost") / "devhost")
    subprocess.run(["g++", "-O1", "-std=c++17", "-o", exe, os.path.join(ROOT, "tools", "devhost.cpp")],
                   check=True, cwd=ROOT)
    return exe


def _traces(text):
    out = {}
    for ln in text.splitlines():
        m = _LINE.match(ln)
        if m:
            out[(int(m[1]), int(m[2]))] = (m[3], m[5].split(), m[6], m[8].split())
    return out


def _reference(listing):
    code = ("import sys; sys.path.insert(0, %r); from oracle import oracle as O; "
            "O.semcheck(sys.stdin.buffer.read(), %s)" % (ROOT, SEED))
    r = subprocess.run([sys.executable, "-c", code], input=listing, capture_output=True,
                       env=dict(os.environ, OCLDEC_SEM_DEBUG="1"), check=True)
    return _traces(r.stderr.decode())


def _device_on_host(exe, listing):
    r = subprocess.run([exe], input=listing, capture_output=True, env=dict(os.environ, OD_SEMCHECK=SEED),
                       check=True)
    return _traces(r.stderr.decode())


def _compare(exe, listing, min_compared):
    ref, dev = _reference(listing), _device_on_host(exe, listing)
    compared = 0
    for key, (asm_flags, asm, body_flags, body) in dev.items():
        if "nan=1" in asm_flags or "bad=1" in asm_flags or "bad=1" in body_flags or "full=1" in body_flags:
            continue
        if key not in ref:  # the reference stopped early (unsupported) in an earlier environment
            continue
        assert (asm, body) == (ref[key][1], ref[key][3]), key
        compared += 1
    assert compared >= min_compared, compared
    return compared


def test_reference_corpus(devhost):
    _compare(devhost, b"".join(x[1] for x in O.corpus()), 150)


def test_nests(devhost):
    _compare(devhost, b"".join(O.make_nest(s) for s in range(1, 101)), 800)


@pytest.mark.parametrize("shape,stress,count", [("C1", 0, 50), ("C3", 1, 100), ("C4", 0, 100)])
def test_generated(devhost, shape, stress, count):
    listing, _, _ = O.generate_corpus(shape, count, seed=4321 + count, stress=bool(stress))
    _compare(devhost, listing, 4 * count)


def test_reference_semcheck_slices_equal_whole():
    """The threaded reference check (slices keyed by their kernels' listing
    ordinals) equals the single pass: the named-size GPU tests rely on it."""
    listing, _, _ = O.generate_corpus("C3", 200, seed=5, stress=True)
    assert O.semcheck(listing, int(SEED, 16), nthreads=8) == O.semcheck(listing, int(SEED, 16))
