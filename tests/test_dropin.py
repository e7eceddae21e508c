"""The C++ drop-in (include/zinpaint_b200.hpp + include/zinpaint/*.hpp): the reference's own
unit tests, compiled unmodified against it, pass on the B200.

oracle/_ref/ref_unit_tests is built by `make -C oracle dropin` (__graft_entry__.build() runs it
while /root/reference exists) from /root/reference/proj/tests/unit/test_{morton,zcurve,layouts,
image,builder,engine}.cpp + the doctest shim tests/dropin/doctest.h, linked to
paper_1712_06326_b200/libzinpaint_b200.so.  Those 61 test cases exercise the drop-in's device
paths (from_descriptors, knn_search, collect_dictionary, build_index, make_query,
multi_index::build, query_best_patch, brute_force_best, inpaint) and its host utilities.
test_pca.cpp (Eigen arithmetic on the caller side) and test_io.cpp (image file I/O, out of
scope) are not part of the drop-in's surface.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ref_unit_tests")
N_CASES = 61


def test_dropin_headers_compile(tmp_path):
    """Every forwarding header resolves to the drop-in and the API compiles as C++17 and C++20."""
    src = tmp_path / "tu.cpp"
    names = ["types", "morton", "image", "layouts", "pca", "pool", "zcurve", "builder", "engine", "io_index"]
    src.write_text("".join(f'#include "zinpaint/{n}.hpp"\n' for n in names) +
                   "int main() { zinpaint::index_config c; (void)c; return zinpaint::morton_less("
                   "(const unsigned char*)\"ab\", (const unsigned char*)\"ba\", 2); }\n")
    for std in ("c++17", "c++20"):
        r = subprocess.run(["g++", f"-std={std}", "-fsyntax-only", "-Wall", "-Werror", "-I",
                            os.path.join(ROOT, "include"), str(src)], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-3000:]


def test_dropin_symbols_exported():
    """The C++ layer is part of libzinpaint_b200.so (no separate wrapper library)."""
    so = os.path.join(ROOT, "paper_1712_06326_b200", "libzinpaint_b200.so")
    out = subprocess.run(["nm", "-D", "--defined-only", "-C", so], capture_output=True, text=True).stdout
    for sym in ("zinpaint::knn_search(", "zinpaint::zcurve_index::from_descriptors(", "zinpaint::build_index(",
                "zinpaint::multi_index::build(", "zinpaint::query_best_patch(", "zinpaint::brute_force_best(",
                "zinpaint::inpaint(", "zinpaint::patch_index::make_query(", "zinpaint::load_multi_index(",
                "zinpaint::save_multi_index("):
        assert sym in out, sym


@pytest.mark.gpu
def test_reference_unit_tests_pass_through_dropin():
    assert os.path.exists(BIN), "oracle/_ref/ref_unit_tests missing: run __graft_entry__.build() where /root/reference exists"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900, cwd=ROOT)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert m, r.stdout[-2000:] + r.stderr[-4000:]
    total, passed, failed = map(int, m.groups())
    assert r.returncode == 0 and failed == 0, r.stderr[-6000:]
    assert total == passed == N_CASES
