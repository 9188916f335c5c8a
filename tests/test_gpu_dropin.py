"""The drop-in proof (Option A).

The reference's own release-gate harness, proj/tests/acceptance/
acceptance_main.cpp, is linked from the reference's sources twice by
oracle/dropin.mk: once as shipped (acceptance_ref, CPU) and once with the
reference's decompiler.cpp replaced by integration/ocldec_b200_dropin.cpp
(acceptance_b200), so every decompile_listing call it makes runs on the GPU
through libocldec_b200.so while all other reference objects are unchanged.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_ref")
B200_BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")


def _checks(out):
    return {int(m.group(2)): m.group(1) for m in re.finditer(r"^\[(PASS|FAIL)\] (\d+)\.", out, re.M)}


@pytest.mark.skipif(not os.path.exists(REF_BIN), reason="drop-in harness not built (make -C oracle -f dropin.mk)")
def test_reference_harness_as_shipped_passes():
    p = subprocess.run([REF_BIN], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout
    assert _checks(p.stdout) == {i: "PASS" for i in range(1, 9)}


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(B200_BIN), reason="drop-in harness not built (make -C oracle -f dropin.mk)")
def test_reference_harness_on_the_gpu():
    """The decompile_listing gates (2 builtin slots, 4 the 1000-nest shape
    sweep through the rebuilt region tree, 5 differential execution of the
    listing against the GPU's lowered body, 6 grammar + fallback counts,
    7 determinism incl. diagnostics, 8 the golden copy kernel) pass with the
    GPU behind the reference's front door; 1 and 3 do not call it."""
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_2107_07809_b200"))
    p = subprocess.run([B200_BIN], capture_output=True, text=True, timeout=900, env=env)
    checks = _checks(p.stdout)
    print(p.stdout)
    for gate in range(1, 9):
        assert checks.get(gate) == "PASS", p.stdout
    assert re.search(r"5\. .*\((2\d) kernels x 100 environments, \1\d\d trace pairs equal\)", p.stdout), p.stdout
    assert p.returncode == 0


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(B200_BIN), reason="drop-in harness not built (make -C oracle -f dropin.mk)")
def test_differential_gate_sees_the_gpu_body():
    """Negative control: with the GPU's body withheld from the binding
    (OCLDEC_B200_DROPIN_NO_BODY=1) the differential gate fails, so its pass
    above is a comparison of the GPU's lowered bodies, not of empty traces."""
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_2107_07809_b200"),
               OCLDEC_B200_DROPIN_NO_BODY="1")
    p = subprocess.run([B200_BIN], capture_output=True, text=True, timeout=900, env=env)
    checks = _checks(p.stdout)
    assert checks.get(5) == "FAIL", p.stdout
    assert p.returncode != 0


CFG_BIN = os.path.join(ROOT, "oracle", "_ref", "cfg_check_b200")


def _cfg_listings():
    from oracle import oracle as O
    yield "corpus", b"".join(x[1] for x in O.corpus())
    yield "nests", b"".join(O.make_nest(s) for s in range(1, 301))
    for shape, stress, count in (("C2", 1, 300), ("C3", 0, 300), ("C3", 1, 300), ("C4", 0, 100)):
        yield f"{shape}-{stress}", O.generate_corpus(shape, count, seed=91 + count, stress=bool(stress))[0]


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(CFG_BIN), reason="drop-in harness not built (make -C oracle -f dropin.mk)")
def test_cfg_matches_reference(tmp_path):
    """DecompiledKernel::cfg through the drop-in (the device's step -4 flow
    graph export) equals the reference's own build_cfg / annotate_exec /
    normalize_if_else result for every kernel, field by field: blocks,
    labels, instruction copies, suppressed marks, terminators (masked source
    operands included), preds, succs, exec ops, reachability, absorption."""
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_2107_07809_b200"))
    for name, listing in _cfg_listings():
        f = tmp_path / f"{name}.s"
        f.write_bytes(listing)
        p = subprocess.run([CFG_BIN, str(f)], capture_output=True, text=True, timeout=600, env=env)
        m = re.search(r"cfg_check kernels=(\d+) compared=(\d+) mismatches=(\d+)", p.stdout)
        assert m and p.returncode == 0, (name, p.stdout[-3000:], p.stderr[-2000:])
        assert int(m.group(3)) == 0 and int(m.group(2)) >= 0.9 * int(m.group(1)), (name, p.stdout[-3000:])
