"""bench.py rank launch (CPU): `--gpus N` runs N ranks -- under torchrun
(WORLD_SIZE must equal N) or by re-launching itself under
torch.distributed.run -- and never degrades silently to one rank."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_rank_launch_modes():
    assert bench.rank_launch(1, {}, [])["mode"] == "single"
    sp = bench.rank_launch(4, {}, ["--gpus", "4", "--steps", "3"])
    assert sp["mode"] == "spawn" and sp["world"] == 4
    argv = sp["argv"]
    assert argv[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in argv and "--master-addr=127.0.0.1" in argv
    assert argv[-4:] == ["--gpus", "4", "--steps", "3"]
    assert bench.rank_launch(2, {"WORLD_SIZE": "2", "RANK": "1"}, [])["mode"] == "rank"
    # torchrun with a different rank count than --gpus: an error, not one rank
    assert bench.rank_launch(8, {"WORLD_SIZE": "1"}, [])["mode"] == "error"
    assert bench.rank_launch(0, {}, [])["mode"] == "error"


def test_dry_run_cli():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["mode"] == "spawn" and d["world"] == 2 and "--dry-run" not in d["argv"]


def test_mismatched_world_exits_nonzero():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode != 0
    assert "WORLD_SIZE" in out.stderr


@pytest.mark.timeout(600)
def test_spawned_two_ranks_reference_arm():
    """`--gpus 2` without torchrun: two gloo ranks (CPU), rank 0 prints one
    reference-arm line with n_gpus = 2, the other rank exits 0."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    env["OMP_NUM_THREADS"] = "2"
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--config", "1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2
