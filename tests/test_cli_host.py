"""CLI front end -- the error paths, which never reach
the GPU: parse errors, flag errors and the legality gate exit 2 with a
diagnostic on stderr and nothing on stdout."""
import os

import pytest

from paper_1806_08299_b200 import cli

DATA = os.path.join(os.path.dirname(__file__), "data")


def run(capsys, *argv):
    rc = cli.main(list(argv))
    out, err = capsys.readouterr()
    return rc, out, err


def test_illegal_skew_exits_2(capsys):
    # SPEC.md cli example: transform/verify with skew 0 on a radius-1 stencil
    rc, out, err = run(capsys, "verify", os.path.join(DATA, "lap1.stencil"), "--mode", "time", "--skew", "0",
                       "--time-tile", "4")
    assert rc == 2 and out == "" and "skew" in err


def test_parse_error_exits_2_with_line(capsys, tmp_path):
    p = tmp_path / "bad.stencil"
    p.write_text("stencil x\ndims 2\nextent 4 4\nsteps 1\nterm 0.5 1 0\n")
    rc, out, err = run(capsys, "run", str(p))
    assert rc == 2 and out == "" and "line 5" in err


@pytest.mark.parametrize("argv", [
    ["frobnicate", "lap1.stencil"],
    ["analyze", "lap1.stencil", "--tiles", "4"],    # arity
    ["analyze", "lap1.stencil", "--profile", "1"],
    ["run", "lap1.stencil", "--mode", "diagonal"],
    ["run", "lap1.stencil", "--tiles", "4,x"],
    ["run", "lap1.stencil", "--mode", "space", "--tiles", "4,4,4"],
    ["run", "missing.stencil"],
    ["tune", "lap1.stencil", "--cost", "bytes"],
    ["simulate", "lap1.stencil", "--cache-elems", "10", "--line-elems", "4"],
])
def test_flag_errors_exit_2(capsys, argv):
    argv = [argv[0], os.path.join(DATA, argv[1])] + argv[2:]
    rc, out, err = run(capsys, *argv)
    assert rc == 2 and out == "" and err


def test_transform_emits_c(capsys, tmp_path):
    """`transform` emits the nest as C99; the illegal-skew
    example exits 2."""
    rc, out, err = run(capsys, "transform", os.path.join(DATA, "lap1.stencil"), "--mode", "time", "--time-tile", "4",
                       "--skew", "1", "--tiles", "8,8")
    assert rc == 0 and "void kernel(float* restrict A)" in out and "MAX(" in out and "#pragma omp parallel for" in out
    dst = tmp_path / "lap1.c"
    rc, out, err = run(capsys, "transform", os.path.join(DATA, "lap1.stencil"), "--mode", "space", "--tiles", "8,8",
                       "-o", str(dst))
    assert rc == 0 and out == "" and dst.read_text().startswith("/* generated")
    rc, out, err = run(capsys, "transform", os.path.join(DATA, "lap1.stencil"), "--mode", "time", "--skew", "0")
    assert rc == 2 and out == "" and "skew" in err


def test_analyze_and_simulate_and_traffic_tune(capsys, tmp_path):
    """analyze / simulate / tune --cost traffic: one JSON
    object each; sim-based output byte-identical across invocations."""
    import json
    spec = os.path.join(DATA, "lap1.stencil")
    rc, out, err = run(capsys, "analyze", spec, "--tiles", "8,8", "--time-tile", "2", "--cache-elems", "100",
                       "--profile", "262.01,17.3")
    assert rc == 0
    d = json.loads(out)
    assert d["estimate"]["ai_tight_tt"] <= d["estimate"]["ai_naive_tt"]
    assert abs(d["ridge_point"] - 15.145) < 0.01
    rc, out, err = run(capsys, "simulate", spec, "--mode", "time", "--time-tile", "2", "--tiles", "8,8",
                       "--cache-elems", "256", "--line-elems", "16")
    assert rc == 0
    d = json.loads(out)
    assert d["bytes"] == 4 * 16 * (d["lines_loaded"] + d["lines_written_back"]) and d["flops"] > 0
    rc, out1, err = run(capsys, "tune", spec, "--cost", "traffic", "--cache-elems", "256", "--line-elems", "1")
    rc2, out2, err = run(capsys, "tune", spec, "--cost", "traffic", "--cache-elems", "256", "--line-elems", "1")
    assert rc == rc2 == 0 and out1 == out2
    d = json.loads(out1)
    assert d["best_cost_bytes"] == min(r["cost_bytes"] for r in d["table"])
