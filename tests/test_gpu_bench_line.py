"""bench.py on a B200 with small extents: the JSON line carries every key of
the driver's contract (value, roofline, e2e with host copies, gpu_launches,
clocks, cpu_baseline) and, for a FAST headline, the bit-exact timing beside
it.  Full sizes are the driver's job; this guards the plumbing."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         env=env, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return lines[0]


def _check(d, workload):
    assert d["metric"].startswith("grid-point updates/sec") and d["unit"] == "GPts/s"
    assert d["config"]["workload"].startswith(workload)
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["higher_is_better"] is True
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["peak"] > 1000 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["gpu_launches"] >= d["steps"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"]
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["kind"] == "port"


def test_default_headline_line_small():
    """The default command (config 5 through the z-slab path), shrunk."""
    d = _run("--extents", "48,96,256", "--time-steps", "8", "--steps", "2", "--warmup", "1")
    _check(d, "config5")
    assert d["config"]["mode"] == "fast" and "1e-5" in d["config"]["tolerance"]
    b = d["bit_exact"]
    assert b["value"] > 0 and b["mode"].startswith("reference")


def test_config2_and_config3_lines_small():
    d = _run("--config", "3", "--extents", "40,72,128", "--time-steps", "8", "--steps", "2", "--warmup", "1")
    _check(d, "config3")
    assert d["bit_exact"]["value"] > 0 and d["config"]["kernel"] == "star"
    d = _run("--config", "2", "--extents", "40,64,128", "--time-steps", "8", "--steps", "2", "--warmup", "1",
             "--mode", "reference")
    _check(d, "config2")
    assert "bit_exact" not in d


def test_reference_arm_line_small():
    d = _run("--impl", "reference", "--config", "2", "--extents", "32,64,64", "--time-steps", "4", "--steps", "1",
             "--warmup", "0")
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
