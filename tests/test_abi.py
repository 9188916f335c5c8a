"""CPU tests of the C-ABI library: it loads, exports every symbol the header
declares, carries sm_100a device code, and its host-side corpus generator is
deterministic.  No decompilation without a GPU."""
import ctypes
import os
import re
import shutil
import subprocess

import pytest

import paper_2107_07809_b200 as P
from paper_2107_07809_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ocldec_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ocldec_b200_\w+)\s*\(", src)))


def test_library_exports_header_symbols():
    L = _lib.load()
    names = header_functions()
    assert len(names) >= 12
    for n in names:
        assert hasattr(L, n), n
    assert set(_lib.EXPORTS) <= set(names)
    assert L.ocldec_b200_version() == 5


def test_library_has_sm100a_code():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_generator_deterministic_and_counted():
    a, offs_a, na = P.generate_corpus("C2", 8, seed=3)
    b, offs_b, nb = P.generate_corpus("C2", 8, seed=3)
    assert a == b and na == nb and list(offs_a) == list(offs_b)
    c, _, _ = P.generate_corpus("C2", 8, seed=4)
    assert c != a
    # kernel k is independent of the batch it is generated in
    one, _, _ = P.generate_corpus("C2", 1, seed=3, k0=5)
    assert a[int(offs_a[5]):int(offs_a[6])] == one
    # every kernel section starts with ".kernel"
    for k in range(8):
        assert a[int(offs_a[k]):int(offs_a[k]) + 8] == b".kernel "
    # instruction count = non-label .text lines (C2 never ends on a label)
    assert na == sum(1 for ln in a.decode().splitlines()
                     if ln.startswith("        ") and not ln.strip().startswith("."))


def test_shapes_sizes():
    for shape, lo, hi in (("C1", 30, 60), ("C2", 150, 260)):
        _, offs, ni = P.generate_corpus(shape, 16, seed=9)
        per = ni / 16
        assert lo <= per <= hi, (shape, per)


def test_ctypes_mirror_matches_header_layout(tmp_path):
    """The ctypes structs the Python front door uses (_lib.py) have the C
    header's sizes and field offsets (no silent ABI drift)."""
    structs = {"ocldec_b200_options": _lib.Options, "ocldec_b200_kernel": _lib.Kernel,
               "ocldec_b200_diag": _lib.Diag, "ocldec_b200_dump": _lib.Dump,
               "ocldec_b200_result": _lib.Result, "ocldec_b200_stats": _lib.Stats}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "ocldec_b200.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append("  return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    for line in filter(None, out):
        cname, field, value = line.split()
        py = structs[cname]
        got = ctypes.sizeof(py) if field == "size" else getattr(py, field).offset
        assert got == int(value), (cname, field, got, value)
