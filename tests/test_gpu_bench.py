"""The bench's N > 1 branch, exercised on a one-GPU box: `bench.py --gpus 2`
re-launches itself with 2 ranks (torch.distributed.run), both on cuda:0 with a
gloo process group (--test-one-device).  Checks the contract of the line the
driver's multi-GPU runs will print: n_gpus, weak-scaling C2 (every rank's bytes
over the slowest rank's time), strong-scaling C4 (rows sharded over the ranks),
per-rank round-trip self-checks.  A functional test of the code path, never a
measurement (two ranks share one GPU)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_bench_two_ranks_one_device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
                          "--configs", "C2,C4", "--no-e2e", "--no-cpu-baseline", "--test-one-device"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["roundtrip_check"] is True
    c2, c4 = line["configs"]["C2"], line["configs"]["C4"]
    # weak scaling: both ranks' 16 pairs; strong scaling: rows 0..4095 / 4096..8191
    assert c2["value"] > 0 and "dp2" in c2["config"]["parallelism"]
    assert c4["local_extents"] == [4096, 8192] and "dp2" in c4["config"]["parallelism"]
    assert line["gpu_launches"] > 0


def test_bench_c5_one_rank_ring():
    """`bench.py --config C5` without torchrun: a one-rank ring (the peer is
    this GPU); every leg (fused TMA stores, LSU stores, copy engines, NCCL)
    round-trip checked on the receiving rank."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "C5", "--steps", "2",
                          "--warmup", "3"], capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    line = json.loads(lines[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0
    legs = line["legs"]
    assert {"fused", "fused_lsu", "staged_ce", "staged_nccl"} <= set(legs)
    assert all(v["parity_roundtrip"] for v in legs.values() if isinstance(v, dict) and "parity_roundtrip" in v)
