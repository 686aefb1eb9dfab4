"""The C-ABI library builds, loads without a GPU and exports every symbol
include/infuser_b200.h declares (CPU-only; no compute calls)."""

import re
from pathlib import Path

import pytest

from conftest import ROOT


def header_symbols():
    text = (ROOT / "include" / "infuser_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(imx_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2008_03095_b200 import _lib
    lib = _lib.load()
    declared = header_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in the header but not exported"
    assert sorted(_lib.EXPORTED) == declared


def test_library_is_sm100a_only():
    import subprocess
    from paper_2008_03095_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.library_path())],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    arches = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert arches == {"100a"}, arches


def test_no_gpu_means_loud_failure():
    from paper_2008_03095_b200 import _lib
    lib = _lib.load()
    if lib.imx_device_count() > 0:
        pytest.skip("a GPU is visible")
    import paper_2008_03095_b200 as imx
    with pytest.raises(RuntimeError, match="no CUDA device|no sm_100"):
        imx.Graph.from_edges(3, [(0, 1), (1, 2)])


def test_product_package_never_imports_the_oracle():
    pkg = ROOT / "paper_2008_03095_b200"
    for py in pkg.rglob("*.py"):
        src = py.read_text()
        assert "import oracle" not in src and "from oracle" not in src, py


def test_header_is_plain_c(tmp_path):
    """include/infuser_b200.h compiles as C99 (no C++ or torch types at the
    boundary) and a C program links against the library's symbols."""
    import shutil
    import subprocess
    from paper_2008_03095_b200 import _lib
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc unavailable")
    src = tmp_path / "abi.c"
    src.write_text('#include "infuser_b200.h"\n'
                   "int main(void) {\n"
                   "    const char *(*err)(void) = imx_last_error;\n"
                   "    imx_allreduce_fn f = 0;\n"
                   "    (void)f;\n"
                   "    return err == 0;\n"
                   "}\n")
    lib = _lib.library_path()
    out = subprocess.run([gcc, "-std=c99", "-Wall", "-Werror", "-I", str(ROOT / "include"), str(src),
                          "-o", str(tmp_path / "abi"), str(lib), f"-Wl,-rpath,{lib.parent}"],
                         capture_output=True, text=True)
    assert out.returncode == 0, out.stderr


def test_source_stamp_ignores_comments_and_layout():
    """The stamp that ties the ncu summaries under profiles/ to the library
    code (build.source_hash) hashes code only: comments and whitespace do not
    invalidate a measurement, string literals and code do."""
    from paper_2008_03095_b200 import build
    a = 'int f(int x) { // add\n  return x + 1; /* one\n more */ }\nconst char *s = "// kept /* too */";\n'
    b = 'int f(int x) {\n\n   return x + 1;   }\n  const char *s = "// kept /* too */";'
    c = b.replace("x + 1", "x + 2")
    d = b.replace("// kept", "// changed")
    assert build._code_only(a) == build._code_only(b)
    assert build._code_only(c) != build._code_only(b)
    assert build._code_only(d) != build._code_only(b)
    h = build.source_hash()
    assert len(h) == 16 and int(h, 16) >= 0
