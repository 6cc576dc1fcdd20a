"""bench.py host logic without a GPU: the reference arm (--impl reference: the
CPU oracle in its OpenMP (p) form on a bounded sample) prints the contract's
JSON line; --gpus N re-launches under torch.distributed.run and refuses a
WORLD_SIZE that disagrees with N; the pair orders share no buffer between
consecutive copies; the pinned CPU-baseline child reports host facts."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert cb["host"]["nproc"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in line["config"]


def test_reference_arm_nonzero_rank_exits_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--gpus", "2"], capture_output=True, text=True, timeout=120, cwd=ROOT,
                         env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_relaunch_command():
    cmd = bench.relaunch_cmd(["--gpus", "4", "--steps", "3"], 4, 29500)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1" and cmd[cmd.index("--master-port") + 1] == "29500"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"] and cmd[-5].endswith("bench.py")


def test_world_must_equal_gpus():
    assert bench.check_world(1, {}) == (1, 0, 0)
    assert bench.check_world(4, {"WORLD_SIZE": "4", "RANK": "2", "LOCAL_RANK": "2"}) == (4, 2, 2)
    with pytest.raises(SystemExit):
        bench.check_world(1, {"WORLD_SIZE": "2"})
    with pytest.raises(SystemExit):
        bench.check_world(8, {})


def test_relaunch_runs_n_processes_without_a_gpu():
    """bench.py --gpus 2 (no torchrun) really starts 2 ranks: exercised on the
    reference arm, where rank 0 prints the one line and rank 1 exits 0."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["n_gpus"] == 2


@pytest.mark.parametrize("name", ["C2", "C2_soa_sb", "C3", "C3_soa_sb", "C4", "C4_pairs", "F1_hep", "F1_listing1"])
def test_pair_orders(name):
    pairs = bench.pairs_of(name)
    expected = {"C2": 16, "C2_soa_sb": 9, "C3": 6, "C3_soa_sb": 4, "C4": 1, "C4_pairs": 12, "F1_hep": 4,
                "F1_listing1": 6}[name]
    assert len(pairs) == len(set(pairs)) == expected
    if name == "C2":
        kinds = bench.SUBCFG["C2"]["kinds"]
        assert set(pairs) == {(a, b) for a in kinds for b in kinds}
    if name == "C4_pairs":
        kinds = bench.SUBCFG[name]["kinds"]
        assert set(pairs) == {(a, b) for a in kinds for b in kinds if a != b}
    if name in ("C2_soa_sb", "C3_soa_sb"):
        assert all("soa_sb" in p for p in pairs)
    for j in range(len(pairs) - (0 if name in ("C2", "C3", "C4_pairs") else 1)):
        a, b = pairs[j], pairs[(j + 1) % len(pairs)]
        if ("soa_sb", "soa_sb") in (a, b) or name.startswith("F1"):  # (F1: splits against 2-3 kinds)
            continue
        if len(pairs) > 1:
            assert a[0] != b[0] and a[1] != b[1], (a, b)


def test_cpu_child_reports_host_and_legs():
    env = dict(os.environ, OMP_PROC_BIND="close", OMP_PLACES="cores")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--cpu-child", "--config", "C2"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["kind"] == "oracle" and r["value"] > 0 and r["cores"] >= 1
    assert r["one_thread"]["value"] > 0 and r["memcpy_1_thread_gbs"] > 0 and r["memcpy_all_threads_gbs"] > 0
    h = r["host"]
    assert h["nproc"] >= 1 and h.get("physical_cores", 1) >= 1 and "ram_gb" in h
    assert r["omp"] == {"OMP_PROC_BIND": "close", "OMP_PLACES": "cores"}
