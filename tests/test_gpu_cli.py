"""`python -m paper_1904_05717_b200 run` on the GPU (test_cli.cpp:70-85
restated): the seeded run verifies (rel <= 1e-12) and is deterministic."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args):
    r = subprocess.run([sys.executable, "-m", "paper_1904_05717_b200", "run"] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    return r.returncode, r.stdout, r.stderr


def test_run_verifies_and_is_deterministic():
    rc, out, err = run(["--alg", "B2A1C0", "--shape", "256", "--format", "json"])
    assert rc == 0, err
    a = json.loads(out)
    assert a["verified"] and a["rel_frobenius_error"] <= 1e-12
    rc, out2, _ = run(["--alg", "B2A1C0", "--shape", "256", "--format", "json"])
    b = json.loads(out2)
    for key in ("algorithm", "shape", "verified", "rel_frobenius_error"):
        assert a[key] == b[key]
    rc, out, _ = run(["--alg", "C2A1C0", "--shape", "2048", "--numerics", "exact", "--format", "json"])
    assert rc == 0 and json.loads(out)["verified"] is False  # 2048^3 > --verify-max 2^27 (tilemul_main.cpp:265)
    rc, out, _ = run(["--alg", "C2A1C0", "--shape", "1024", "--numerics", "exact", "--verify-max", str(1 << 31),
                      "--format", "json"])
    assert rc == 0 and json.loads(out)["rel_frobenius_error"] == 0.0


def test_run_invalid_descriptor_exit_1():
    rc, out, err = run(["--alg", "A3A2C0", "--shape", "64"])
    assert rc == 1 and "consecutive_resident_equal" in out + err
