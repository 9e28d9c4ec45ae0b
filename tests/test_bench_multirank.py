"""bench.py's multi-rank path (the driver's scaling run) end to end: two ranks
under torchrun on one GPU with CPU (gloo) collectives at a small RMAT scale.
Checks the one-line contract: rank 0 alone prints, whole-job values, weak
scaling, e2e rows verified, and the reference arm runs on rank 0 only."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _torchrun(args, n=2, port=29611):
    env = dict(os.environ, ND_DIST_BACKEND="gloo", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py"] + args
    p = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    return lines


@pytest.mark.gpu
def test_bench_two_ranks_one_line():
    common = ["--gpus", "2", "--scale", "14", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-tp"]
    lines = _torchrun(common)
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["e2e"]["host_rows_match_device"] is True and d["e2e"]["value"] > 0
    assert "dev_scale" in d["config"] and d["gpu_launches"] > 0
    assert d["config"]["walkers_per_step"] == 2 * 2 * (1 << 14)
    ref = _torchrun(["--impl", "reference"] + common, port=29612)
    assert len(ref) == 1
    r = json.loads(ref[0])
    assert r["impl"] == "reference" and r["value"] > 0 and r["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_run_sharded_two_ranks_equals_one_run(tmp_path):
    """multigpu.run_sharded: each rank samples its worker_ranges share, rows
    gathered to rank 0 in rank order == one single-process run (driver.py:175-186)."""
    res = tmp_path / "sharded.json"
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29613", "tests/_sharded_worker.py", str(res)]
    p = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    verdict = json.loads(res.read_text())
    assert verdict == {"node2vec": True, "ppr": True, "khop": True}


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 3])
def test_sharded_job_pieces_equal_one_run(tmp_path, n):
    """multigpu.ShardedJob (the C5 step): DeepWalk shards in pieces, k-hop
    whole, rows gathered piece by piece to rank 0's pinned host memory; in
    sample-id order they equal one single-process run (driver.py:175-186)."""
    res = tmp_path / "job.json"
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29620 + n),
           "tests/_shardedjob_worker.py", str(res)]
    p = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    assert json.loads(res.read_text()) == {"deepwalk": True, "khop": True}
