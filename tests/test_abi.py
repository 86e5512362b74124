"""The C-ABI library loads and exports every symbol include/tilemul_b200.h
declares, the Python loader binds exactly those, and status codes follow the
header's contract (no GPU needed: no compute calls)."""
from __future__ import annotations

import ctypes as C
import os
import re

import pytest

from paper_1904_05717_b200 import _native as N
from paper_1904_05717_b200 import tilemul as T

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "tilemul_b200.h")


def declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tm_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported_and_bound():
    lib = N.lib()
    names = declared()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), f"{name} declared in the header but not exported"
    assert sorted(N.declared_symbols()) == names


def test_no_python_fallback_when_library_missing(monkeypatch):
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "LIB_PATH", "/nonexistent/libtilemul_b200.so")
    with pytest.raises(ImportError):
        N.lib()


def test_status_codes():
    lib = N.lib()
    p = C.c_void_p()
    lv = (N.tm_level * 1)(N.tm_level(64, 1, 0, 1, 1))
    bs = (N.tm_blocksize * 2)(N.tm_blocksize(0, b"m", 4), N.tm_blocksize(0, b"n", 4))
    assert lib.tm_plan_create(b"A3A2C0", lv, 1, 8, 8, 8, bs, 2, C.byref(p)) == 1
    assert lib.tm_last_rules().decode().startswith("consecutive_resident_equal")
    assert lib.tm_plan_create(b"C0", lv, 1, 0, 8, 8, bs, 2, C.byref(p)) == 2
    assert lib.tm_execute(None, None, 1, None, 1, None, 1, None, None) == 2
    assert lib.tm_plan_create(b"C0", lv, 1, 8, 8, 8, bs, 2, C.byref(p)) == 0
    lib.tm_plan_destroy(p)
    assert lib.tm_version().decode().startswith("tilemul_b200")


def test_validation_failure_carries_rules():
    with pytest.raises(T.ValidationFailure) as e:
        T.build_plan(T.parse_name("C0"), T.BlocksizeSet({(0, "m"): 100, (0, "n"): 100}),
                     T.CacheHierarchy.from_capacities([64]), T.Shape(8, 8, 8))
    assert e.value.violations[0].rule == "resident_guest_exceed_capacity"
    assert e.value.violations[0].lhs == 10000 and e.value.violations[0].rhs == 64


def test_cpp_shim_compiles_against_the_reference():
    """include/tilemul_b200.hpp compiles after the reference's own headers
    (checked where the reference tree exists, i.e. in the build container)."""
    import shutil
    import subprocess
    import tempfile

    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc) or shutil.which("g++") is None:
        pytest.skip("reference headers or g++ absent")
    inc = os.path.dirname(HEADER)
    src = ('#include "tilemul/exec.hpp"\n#include "tilemul_b200.hpp"\n'
           "void f(const tilemul::LoopNest& n, const tilemul::MatrixBuffer& a, const tilemul::MatrixBuffer& b,\n"
           "       tilemul::MatrixBuffer& c, const tilemul::CacheHierarchy& h) {\n"
           "    tilemul::b200::execute(n, a, b, c, h, {}, {TM_NUMERICS_EXACT});\n}\n")
    with tempfile.NamedTemporaryFile("w", suffix=".cpp", delete=False) as f:
        f.write(src)
    try:
        r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-I", ref_inc, "-I", inc,
                            f.name], capture_output=True, text=True, timeout=120)
    finally:
        os.unlink(f.name)
    assert r.returncode == 0 and "warning" not in r.stderr, r.stderr


def test_plan_from_loops_checks_and_has_no_model():
    """tm_plan_create_loops (the signature-identical drop-in's plan): cells
    larger than the register tile are a usage error; such a plan has no
    hierarchy, so no model; a valid one walks the given loops."""
    steps = [T.NestStep(1, "k", 32), T.NestStep(1, "n", 40), T.NestStep(0, "n", 20), T.NestStep(0, "m", 64)]
    nest = T.LoopNest.from_loops(steps, 64, 20, T.Shape(130, 70, 90), name=None)
    assert nest.cell_count() == 3 * 2 * 2 * 3 and nest.loops == steps
    with pytest.raises(ValueError):
        nest.model()
    with pytest.raises(ValueError):
        T.LoopNest.from_loops(steps, 32, 20, T.Shape(130, 70, 90))  # 64-row cells > m_r = 32
    named = T.LoopNest.from_loops(steps, 64, 20, T.Shape(130, 70, 90), name="B1C0")
    assert T.format_name(named.descriptor) == "B1C0"


def test_build_id_matches_sources():
    from paper_1904_05717_b200 import build as B

    assert N.build_id() == B.source_hash()
    assert N.build_id() in N.lib().tm_version().decode()
