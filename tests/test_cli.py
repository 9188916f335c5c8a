"""The reference-shaped host front ends over the C ABI: the CLI
(tools/ocldec_b200_cli.cpp, reference proj/tools/ocldec.cpp:81-177) and the
header-only C++ shim include/ocldec_b200.hpp (reference decompiler.hpp:62).

CPU tests check that they build and that the CLI parses its arguments
without touching the GPU; the gpu test runs the reference's own CLI
round-trip (proj/tests/cli_roundtrip.cmake:10-27: copy.asm -> copy.cl,
byte-compare)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2107_07809_b200", "ocldec-b200")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _need_cli():
    if not os.path.exists(CLI):
        pytest.skip("CLI not built (make -C paper_2107_07809_b200/csrc)")


def test_cli_version_and_usage():
    _need_cli()
    p = subprocess.run([CLI, "--version"], capture_output=True, text=True)
    assert p.returncode == 0 and "ocldec-b200" in p.stdout
    p = subprocess.run([CLI], capture_output=True, text=True)
    assert p.returncode == 1 and "Usage" in p.stderr
    p = subprocess.run([CLI, "x.asm", "--no-such-flag"], capture_output=True, text=True)
    assert p.returncode == 1 and "Usage" in p.stderr


def test_cli_missing_input(tmp_path):
    _need_cli()
    p = subprocess.run([CLI, str(tmp_path / "nope.asm")], capture_output=True, text=True)
    assert p.returncode == 1
    assert "cannot open" in p.stderr


def test_cpp_shim_parses_reduction(tmp_path):
    src = tmp_path / "red.cpp"
    src.write_text('#include "ocldec_b200.hpp"\n'
                   'int main() {\n'
                   '  auto r = ocldec_b200::parse_reduction("merge 3 5 1 2 3\\nmerge 1 6 5 4\\nroot 6\\n");\n'
                   '  auto g = ocldec_b200::parse_reduction("merge 2 4 1 2\\nresidue 3 4\\n");\n'
                   '  bool ok = r.merges.size() == 2 && r.merges[0].kind == 3 && r.merges[0].result == 5 &&\n'
                   '            r.merges[0].absorbed == std::vector<int>{1, 2, 3} && r.reduced && r.root == 6 &&\n'
                   '            !g.reduced && g.residue == std::vector<int>{3, 4} && g.merges[0].absorbed.size() == 2;\n'
                   '  return ok ? 0 : 1; }\n')
    exe = tmp_path / "red"
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    assert subprocess.run([str(exe)]).returncode == 0


def test_cpp_shim_compiles(tmp_path):
    src = tmp_path / "shim.cpp"
    src.write_text('#include "ocldec_b200.hpp"\n'
                   'int main() { ocldec_b200::DecompileResult r; r.kernels.resize(2);\n'
                   '  r.kernels[0].source = "a"; r.kernels[1].source = "b";\n'
                   '  return r.combined_source() == "a\\nb" ? 0 : 1; }\n')
    exe = tmp_path / "shim"
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    assert subprocess.run([str(exe)]).returncode == 0


@pytest.mark.gpu
def test_cli_roundtrip_golden(tmp_path):
    _need_cli()
    inp = tmp_path / "copy.asm"
    inp.write_bytes(open(os.path.join(GOLDEN, "copy.asm"), "rb").read())
    p = subprocess.run([CLI, str(inp)], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    out = tmp_path / "copy.cl"  # default output: input stem + ".cl"
    assert out.read_bytes() == open(os.path.join(GOLDEN, "copy.cl"), "rb").read()


@pytest.mark.gpu
def test_cli_split_error_and_failed_kernel(tmp_path):
    _need_cli()
    bad = tmp_path / "bad.asm"
    bad.write_text(".text\n    s_endpgm\n")
    p = subprocess.run([CLI, str(bad), "-o", str(tmp_path / "o.cl")], capture_output=True, text=True)
    assert p.returncode == 1
    assert p.stderr.strip() == f"{bad}:1: error: .text outside of a .kernel section"
    # a kernel-level ParseError (undefined label): failed kernel, exit 1, empty output
    failk = tmp_path / "f.asm"
    failk.write_text(".kernel k\n.text\n    s_branch L_nowhere\n    s_endpgm\n")
    p = subprocess.run([CLI, str(failk), "-o", str(tmp_path / "f.cl")], capture_output=True, text=True)
    assert p.returncode == 1
    assert (tmp_path / "f.cl").read_bytes() == b""
