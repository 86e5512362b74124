"""The CLI (python -m paper_1904_05717_b200), restating the reference's CLI
tests (tests/test_cli.cpp:24-68, :105-125) on the CPU-side subcommands;
`run` needs a GPU and is covered in tests/test_gpu_cli.py."""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
I7 = os.path.join(ROOT, "configs", "i7_7700k_like.json")


def cli(args):
    r = subprocess.run([sys.executable, "-m", "paper_1904_05717_b200"] + args, cwd=ROOT, capture_output=True,
                       text=True, timeout=120)
    return r.returncode, r.stdout, r.stderr


def setup_module(_):
    # the i7-7700K hierarchy of the reference's configs, in FP64 elements (restated values)
    os.makedirs(os.path.dirname(I7), exist_ok=True)
    json.dump({"levels": [{"index": 0, "capacity_elements": 64}, {"index": 1, "capacity_elements": 8192},
                          {"index": 2, "capacity_elements": 32768}, {"index": 3, "capacity_elements": 786432}]},
              open(I7, "w"))


def test_analyze_published_intensities():
    rc, out, _ = cli(["analyze", "--alg", "B3A2C0", "--shape", "76800", "--hier", I7, "--bs", "3:n=768", "--bs",
                      "3:k=768", "--bs", "2:m=120", "--bs", "2:k=192", "--format", "json"])
    assert rc == 0
    assert 63.0 < json.loads(out)["intensity_flops_per_byte"] < 64.5
    rc, out, _ = cli(["analyze", "--alg", "A2C0", "--shape", "192000", "--hier", I7, "--bs", "2:m=120", "--bs",
                      "2:k=192", "--bs", "3:n=3000", "--format", "json"])
    assert rc == 0
    assert 23.1 < json.loads(out)["intensity_flops_per_byte"] < 23.4


def test_exit_codes_and_determinism():
    rc, out, _ = cli(["analyze", "--alg", "B3A2C0", "--shape", "1024", "--hier", "/nonexistent/h.json"])
    assert rc == 2 and "level" not in out
    rc, out, err = cli(["analyze", "--alg", "A3A2C0", "--shape", "64", "--hier", I7])
    assert rc == 1 and "consecutive_resident_equal" in out + err
    a = cli(["analyze", "--alg", "B3A2C0", "--shape", "4096", "--hier", I7, "--format", "json"])
    b = cli(["analyze", "--alg", "B3A2C0", "--shape", "4096", "--hier", I7, "--format", "json"])
    assert a[0] == 0 and a[1] == b[1]
    c = cli(["analyze", "--alg", "B3A2C0", "--shape", "4096", "--hier", I7, "--format", "csv"])
    assert c[0] == 0 and c[1].startswith("level,operand,reads,writes\n")


def test_plan_on_gpu_hierarchy_file():
    h = os.path.join(ROOT, "configs", "b200_fp64.json")
    rc, out, _ = cli(["plan", "--shape", "65536x256x1024", "--hier", h])
    assert rc == 0
    j = json.loads(out)
    # B resident at L2 moves only compulsory traffic for the panel-panel shape
    assert j["recommended"] == "B2A1C0"
    assert j["reference_select_algorithm"] == "C"
    ranked = [r["algorithm"] for r in j["ranking"] if r["model_bytes_into_L2"] is not None]
    assert ranked[0] == "B2A1C0"


DESK = ["--alg", "B3A2C0", "--shape", "96", "--bs", "3:n=48", "--bs", "3:k=48", "--bs", "2:m=24", "--bs", "2:k=24",
        "--bs", "0:n=6", "--bs", "0:m=2"]


def _desk_hier(tmp_path):
    p = tmp_path / "desk.json"
    json.dump({"levels": [{"index": 0, "capacity_elements": 16},
                          {"index": 1, "capacity_elements": 512, "write_allocate": False},
                          {"index": 2, "capacity_elements": 2048, "write_allocate": False},
                          {"index": 3, "capacity_elements": 49152, "write_allocate": False}]}, open(p, "w"))
    return str(p)


def test_simulate_json_csv_and_trace_dump(tmp_path):  # tilemul_main.cpp:179-229
    h = _desk_hier(tmp_path)
    rc, out, _ = cli(["simulate", "--hier", h, "--format", "json"] + DESK)
    assert rc == 0
    j = json.loads(out)
    assert j["algorithm"] == "B3A2C0" and set(j) == {"algorithm", "simulation", "model", "comparison"}
    assert j["simulation"]["events"] == 663552
    assert [lv["level"] for lv in j["simulation"]["levels"]] == [1, 2, 3]  # registers not simulated by default
    # the inner levels follow the model exactly at this scale
    assert [c["rel_error"] for c in j["comparison"]["levels"]][:2] == [0.0, 0.0]
    rc, out, _ = cli(["simulate", "--hier", h, "--format", "csv", "--include-registers"] + DESK)
    assert rc == 0
    rows = out.strip().splitlines()
    assert rows[0] == "level,hits,misses,writebacks,sim_elements,model_elements,rel_error"
    assert [r.split(",")[0] for r in rows[1:]] == ["0", "1", "2", "3"]
    dump = tmp_path / "trace.txt"
    rc, _, _ = cli(["simulate", "--hier", h, "--trace-dump", str(dump), "--colmajor-trace"] + DESK)
    assert rc == 0
    lines = open(dump).read().splitlines()
    assert len(lines) == 663552 and lines[0] == "C 0 R" and lines[-1].endswith(" W")


def test_simulate_refuses_long_traces(tmp_path):
    rc, _, err = cli(["simulate", "--hier", _desk_hier(tmp_path), "--max-events", "1000"] + DESK)
    assert rc == 2 and "--max-events" in err


def test_roofline_regimes():  # acceptance.cpp:256-281 (criterion 7)
    rc, out, _ = cli(["roofline", "--peak", "40e9", "--bw", "1e9", "--point", "A2C0=23.26", "--point", "B3A2C0=64.0"])
    assert rc == 0
    assert "A2C0,23.26," in out and ",bandwidth-bound" in out
    assert "B3A2C0,64," in out and ",compute-bound" in out
    rc, out, _ = cli(["roofline", "--peak", "40e9", "--bw", "1e9", "--point", "x=40", "--format", "json"])
    j = json.loads(out)
    assert rc == 0 and j["breakpoint_intensity"] == 40.0 and j["points"][0]["regime"] == "compute-bound"
    rc, _, _ = cli(["roofline", "--peak", "1", "--bw", "1", "--point", "noequals"])
    assert rc == 2


def test_pareto_cli():  # tilemul_main.cpp:390-431
    rc, out, _ = cli(["pareto", "--cache", "262144", "--ratios", "4,16", "--shape", "4096", "--format", "json"])
    assert rc == 0
    pts = json.loads(out)["points"]
    assert [p["ratio"] for p in pts] == [4.0, 16.0] and pts[0]["inner_capacity"] == 65536
    assert cli(["pareto", "--cache", "100", "--ratios", "64", "--shape", "64"])[0] == 1  # infeasible
    assert cli(["pareto", "--cache", "100", "--ratios", "", "--shape", "64"])[0] == 2
