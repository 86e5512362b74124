"""The drop-in check: the reference's own API (parse_name -> derive_blocksizes
-> build_plan -> execute, compiled unmodified from its headers) with only the
execute call swapped for tilemul::b200::execute (include/tilemul_b200.hpp).
oracle/_ref/dropin_check (oracle/Makefile, built where the reference tree
exists and shipped with the snapshot) prints one JSON line per check:
EXACT numerics bit-identical to the reference's execute() on column-major and
prepacked operands for every expressible family member, DMMA within the
bound, and the reference's exception types / ValidationFailure rule ids for
bad inputs."""
from __future__ import annotations

import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "dropin_check")


def test_reference_api_with_b200_execute():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/dropin_check is built only where the reference tree exists")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    bad = [x for x in lines if "check" in x and not x["ok"]]
    assert not bad, bad
    summary = [x for x in lines if x.get("summary")]
    assert summary and summary[0]["failures"] == 0, (r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stderr[-2000:]
    kinds = {x["check"].split(" ")[0] for x in lines if "check" in x}
    assert {"exact", "dmma", "role", "k-parallel", "bad", "signature-identical", "plan/nest", "hand-built",
            "cells"} <= kinds
