#!/usr/bin/env python
"""Benchmark: layout-copy GB/s (read + write bytes) per mapping pair on B200.

Headline (BASELINE.json configs[1], "C2"): 16,777,216 Particle7 records
(7 x f32), all 16 ordered pairs of {packed AoS, SoA multi-blob,
AoSoA8, AoSoA32}.  One step = the 16 layout-aware copies, each one llama_copy
through the C ABI.  value = sum over pairs of (src footprint + dst footprint) /
step time, summed over ranks (weak scaling: every rank relayouts its own 16M
records; no data-path collective).

The same run also measures, as sub-objects of the line (`configs`):
  C2_soa_sb  the 9 further ordered pairs with SoA single-blob
  C3         67,108,864 HEP100 event records, packed AoS <-> aligned AoS <-> SoA MB
             (the paper's 100-leaf event workload), weak scaling
  C3_soa_sb  the same records, the 4 pairs of {packed, aligned AoS} <-> SoA single-blob
  C4         Listing-1 8192 x 8192, AoSoA32 -> SoA SB, rows sharded over ranks (strong)
  F1_hep / F1_listing1  Split mappings against plain ones
each with per-pair GB/s, the dominant kernel's roofline and an in-run
device-memcpy ceiling; `min_pair_frac` is the weakest pair over all of them.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2|C3|C4|C5|MOVE] [--configs C2,C2_soa_sb,C3,C3_soa_sb,C4,C4_pairs,F1_hep,F1_listing1]

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
with N processes (one per GPU); under torchrun WORLD_SIZE must equal N.

--impl reference times the CPU oracle (oracle/, plain C naive copy, in
its OpenMP (p) form on the host's physical cores) on a bounded sample
of the same workload; it needs no GPU.

--config MOVE: the n-body move (Listing P:643-645) on 256Mi
Particle7 particles per GPU; --config C5: cross-device relayout (AoS on GPU i
-> SoA MB on GPU i+1) with its in-run NVLink ceiling and the staged baselines.
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC = os.path.join(ROOT, "profiles", "traffic.json")
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
NOMINAL_HBM_GBS = 8000.0
METRIC = "layout-copy GB/s (read+write) per mapping pair vs 8 TB/s HBM, 1/2/4/8 B200"
KERNEL = {"permute": "k_permute_ws", "permute_direct": "k_permute_direct", "permute_jit": "llb_jit_permute",
          "blobcopy": "k_bulkcopy",
          "run": "k_run", "naive": "k_naive", "transpose": "k_transpose2d", "transpose_jit": "llb_jit_transpose",
          "transpose_wide": "k_transpose_wide"}
DEFAULT_CONFIGS = "C2,C2_soa_sb,C3,C3_soa_sb,C4,C4_pairs,F1_hep,F1_listing1,F4_p7,F4_hep"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C2", "C3", "C4", "C5", "MOVE"],
                    help="the headline config of the line (value)")
    ap.add_argument("--configs", default=None,
                    help=f"configs measured in this run (default with --config C2: {DEFAULT_CONFIGS}; "
                         "otherwise just --config)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-child", action="store_true", help=argparse.SUPPRESS)  # the pinned CPU-baseline process
    # functional test of the N > 1 branch on a one-GPU box (tests/test_gpu_bench.py): every rank on
    # cuda:0, gloo process group -- exercises the code path, is never a measurement
    ap.add_argument("--test-one-device", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--per-pair", default=None, help="write per-pair timings (json) to this file")
    return ap.parse_args(argv)


def hbm_peak():
    try:
        with open(MEASURED_PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def traffic_for(cfg_name, kernel):
    """DRAM read+write bytes per launch of `kernel` in config `cfg_name` from
    the committed ncu capture (profiles/traffic.json, keyed by config/kernel)."""
    try:
        with open(TRAFFIC) as f:
            e = json.load(f).get(f"{cfg_name}/{kernel}")
        return (e or {}).get("dram_bytes_per_launch"), (e or {}).get("cold_frac")
    except Exception:
        return None, None


# -------------------------------------------------------------- launching
def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_cmd(argv, gpus, port):
    """torch.distributed.run command that runs this script with one process per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + list(argv)


def check_world(gpus, env):
    """(world, rank, local_rank); raises when torchrun's WORLD_SIZE disagrees with --gpus."""
    world = int(env.get("WORLD_SIZE", "1"))
    if world != gpus:
        raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={world}; n_gpus must equal the ranks that run")
    return world, int(env.get("RANK", "0")), int(env.get("LOCAL_RANK", "0"))


def l2_free_order(kinds, identities=True):
    """Ordered pairs of `kinds` such that consecutive pairs (also across the
    step boundary) share neither the source nor the destination buffer, so no
    copy starts on bytes the previous one left in L2."""
    n = len(kinds)
    if identities:
        return [(kinds[k % n], kinds[(k % n + k // n) % n]) for k in range(n * n)]
    # without identities (3 kinds): the cycle a -> a+1, then the reverse cycle
    assert n == 3
    fwd = [(kinds[a], kinds[(a + 1) % n]) for a in range(n)]
    rev = [(kinds[(-a) % n], kinds[(-a - 1) % n]) for a in range(n)]
    return fwd + rev


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in self.rows if len(r) >= 9 for j in range(4)
                          if r[5 + j].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------- CPU baseline
def host_info():
    """nproc, CPU model, physical cores, RAM of this host (P:592, P:599 report them)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                info["model"] = line.split(":", 1)[1].strip()
        cores = subprocess.run(["lscpu", "-p=CORE,SOCKET"], capture_output=True, text=True, timeout=10).stdout
        info["physical_cores"] = len({ln for ln in cores.splitlines() if ln and not ln.startswith("#")})
    except Exception:
        pass
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemTotal:"):
                    info["ram_gb"] = round(int(line.split()[1]) * 1024 / 1e9, 1)
    except Exception:
        pass
    try:  # the cores this process may run on (a container may see fewer than the host)
        info["affinity_cpus"] = len(os.sched_getaffinity(0))
    except Exception:
        pass
    return info


def _physical_threads(info):
    phys = info.get("physical_cores") or info.get("nproc") or 1
    return max(1, min(phys, info.get("affinity_cpus") or phys))


def _avg_runs(fn, runs=5):
    fn()  # one warm-up ("average of 5 consecutive runs")
    ts = []
    for _ in range(runs):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.mean(ts)


def cpu_child(cfg_name):
    """Runs in its own process with OMP_PROC_BIND=close OMP_PLACES=cores set
    before libgomp loads ("as many pinned threads as cores").  Times the
    oracle (i) with 1 thread and (ii) in its OpenMP (p) form on the physical
    cores, and (iii) host memcpy with 1 and all those threads, each the
    average of 5 runs after 1 warm-up, on bounded prefixes of the workload."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    import oracle
    cfg = W.CONFIGS[cfg_name]
    schema = W.SCHEMAS[cfg["schema"]]
    info = host_info()
    P = _physical_threads(info)
    names = sorted({x for p in cfg["pairs"] for x in p})

    def views(n):
        maps = {k: oracle.Mapping(schema, [n], *W.MAPPINGS[k]) for k in names}
        src = {k: oracle.make_view(maps[k], 42) for k in names}
        dst = {k: maps[k].alloc() for k in names}
        nbytes = sum(sum(maps[a].blob_sizes()) + sum(maps[b].blob_sizes()) for a, b in cfg["pairs"])
        return maps, src, dst, nbytes

    def leg(n, threads):
        maps, src, dst, nbytes = views(n)

        def run():
            for a, b in cfg["pairs"]:
                oracle.copy(maps[a], src[a], maps[b], dst[b], nthreads=threads)
        dt = _avg_runs(run)
        return nbytes / dt / 1e9, dt, nbytes

    # (i) one thread: a 2^20-record prefix (well beyond the LLC, "naive")
    n1 = 1 << 20
    g1, dt1, b1 = leg(n1, 1)
    # (ii) OpenMP (p) on the physical cores: prefix sized to ~2 s per run from the
    # 1-thread rate, >= 2^22 records, at most the full per-GPU extent
    full = int(cfg["extents"][0]) if len(cfg["extents"]) == 1 else 1 << 24
    want = int(n1 * 2.0 / max(dt1, 1e-3) * P)
    n_p = max(1 << 22, min(full, want))
    n_p -= n_p % 32
    gp, dtp, bp = leg(n_p, P)
    # (iii) host memcpy of 1 GiB, 1 thread and P threads
    x = np.ones(1 << 30, np.uint8)
    y = np.empty_like(x)
    m1 = 2 * x.nbytes / _avg_runs(lambda: np.copyto(y, x)) / 1e9
    chunks = np.array_split(np.arange(x.nbytes), P)
    bounds = [(int(c[0]), int(c[-1]) + 1) for c in chunks if len(c)]
    pool = ThreadPoolExecutor(P)

    def par():
        list(pool.map(lambda ab: np.copyto(y[ab[0]:ab[1]], x[ab[0]:ab[1]]), bounds))
    mp = 2 * x.nbytes / _avg_runs(par) / 1e9
    pool.shutdown()
    return {"value": gp, "unit": "GB/s", "cores": P, "kind": "oracle",
            "sample": f"{cfg_name}: all {len(cfg['pairs'])} pairs on a prefix of {n_p} records per run "
                      f"({bp / 1e9:.2f} GB moved), oracle OpenMP (p) with {P} threads pinned one per physical "
                      f"core (OMP_PROC_BIND=close OMP_PLACES=cores), average of 5 runs after 1 warm-up",
            "one_thread": {"value": g1, "unit": "GB/s", "sample": f"prefix of {n1} records, {b1 / 1e9:.2f} GB per run"},
            "memcpy_1_thread_gbs": m1, "memcpy_all_threads_gbs": mp,
            "memcpy_note": "host memcpy (numpy copyto) of 1 GiB, read+write bytes, the host ceiling (P:762)",
            "host": info, "omp": {"OMP_PROC_BIND": os.environ.get("OMP_PROC_BIND"),
                                  "OMP_PLACES": os.environ.get("OMP_PLACES")},
            "flags": "gcc -O3 -fopenmp (oracle/__init__.py build; no -march=native: the .so travels between hosts)"}


def cpu_baseline(cfg_name):
    env = dict(os.environ, OMP_PROC_BIND="close", OMP_PLACES="cores")
    out = subprocess.run([sys.executable, os.path.abspath(__file__), "--cpu-child", "--config", cfg_name],
                         capture_output=True, text=True, env=env, timeout=900)
    if out.returncode != 0:
        raise RuntimeError(out.stderr[-400:])
    return json.loads(out.stdout.strip().splitlines()[-1])


def run_reference(args, cfg):
    """The base contract's reference arm: the oracle, as it stands, in its
    OpenMP (p) form on the host's physical cores, on a bounded prefix of the
    same workload per step (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    os.environ.setdefault("OMP_PROC_BIND", "close")  # before liboracle / libgomp load
    os.environ.setdefault("OMP_PLACES", "cores")
    import oracle
    info = host_info()
    P = _physical_threads(info)
    schema = W.SCHEMAS[cfg["schema"]]
    names = sorted({x for p in cfg["pairs"] for x in p})
    n = 1 << 20
    if cfg["name"] == "C4":
        n = 1 << 18
    maps = {k: oracle.Mapping(schema, [n], *W.MAPPINGS[k]) for k in names}
    views = {k: oracle.make_view(maps[k], 42) for k in names}
    dsts = {k: maps[k].alloc() for k in names}
    step_bytes = sum(sum(maps[a].blob_sizes()) + sum(maps[b].blob_sizes()) for a, b in cfg["pairs"])

    def step():
        for a, b in cfg["pairs"]:
            oracle.copy(maps[a], views[a], maps[b], dsts[b], nthreads=P)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / max(1, args.steps)
    value = step_bytes / dt / 1e9
    sample = (f"{cfg['name']} pairs on a prefix of {n} records per step, oracle OpenMP (p) with {P} threads "
              "(one per physical core, pinned)")
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong" if cfg["name"] == "C4" else "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (splitmix64, seed 42)",
            "config": dict(workload_desc(cfg["name"], 1), sample_records=n), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": P, "kind": "oracle", "sample": sample,
                             "host": info},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- ours
def workload_desc(name, world):
    if name == "C2":
        return dict(workload="C2: Particle7 (7x f32) x 16,777,216 records per GPU, 16 ordered pairs of "
                             "{packed AoS, SoA MB, AoSoA8, AoSoA32}",
                    records_per_gpu=16_777_216, pairs=16,
                    l2="inputs larger than L2 (each pair reads 470 MB and writes 470 MB; L2 is 126 MB); "
                       "consecutive copies share no buffer",
                    parallelism=f"dp{world} (independent per-GPU relayout, weak scaling)")
    if name == "C2_soa_sb":
        return dict(workload="C2 + SoA SB: the 9 further ordered pairs of {packed AoS, SoA MB, AoSoA8, AoSoA32, "
                             "SoA SB} that involve SoA single-blob, 16,777,216 Particle7 records per GPU",
                    records_per_gpu=16_777_216, pairs=9, l2="inputs larger than L2",
                    parallelism=f"dp{world} (weak scaling)")
    if name == "F1_hep":
        return dict(workload="F1: HEP100 x 16,777,216 records per GPU, split_hep (the 4-momenta of the 10 objects -> SoA "
                             "MB, the rest aligned AoS; P:479-481) <-> packed AoS / SoA MB, 4 pairs",
                    records_per_gpu=16_777_216, pairs=4, l2="inputs larger than L2", parallelism=f"dp{world} (weak scaling)")
    if name == "C4_pairs":
        return dict(workload="C4 record (Listing-1: 1- to 8-byte leaves, 21-byte packed / 32-byte aligned) x "
                             "67,108,864 per GPU, the 12 ordered pairs of {packed AoS, aligned AoS, SoA MB, AoSoA32}",
                    records_per_gpu=67_108_864, pairs=12, l2="inputs larger than L2; consecutive copies share no buffer",
                    parallelism=f"dp{world} (weak scaling)")
    if name == "F4_p7":
        return dict(workload="F4: Particle7 x 4096 x 4096 per GPU, 6 transposing copies between row-major / column-major "
                             "/ Morton views (P:140-142) of packed AoS and SoA MB",
                    records_per_gpu=16_777_216, pairs=6, l2="inputs larger than L2", parallelism=f"dp{world} (weak scaling)")
    if name == "F4_hep":
        return dict(workload="F4: HEP100 x 2048 x 2048 per GPU, 5 transposing copies (AoS -> SoA, SoA -> AoS, packed -> "
                             "aligned AoS, AoS col -> Morton, SoA SB -> MB; the wide-record kernel and the JIT's "
                             "short tiles)", records_per_gpu=4_194_304, pairs=5, l2="inputs larger than L2",
                    parallelism=f"dp{world} (weak scaling)")
    if name == "F1_listing1":
        return dict(workload="F1: Listing-1 record x 67,108,864 per GPU, split_pos (Pos -> SoA MB, the rest packed AoS; "
                             "S:304) <-> packed / aligned AoS / SoA MB, 6 pairs",
                    records_per_gpu=67_108_864, pairs=6, l2="inputs larger than L2", parallelism=f"dp{world} (weak scaling)")
    if name == "C3_soa_sb":
        return dict(workload="C3 + SoA SB: HEP100 stand-in x 67,108,864 records per GPU, the 4 ordered pairs of "
                             "{packed AoS, aligned AoS} <-> SoA single-blob", records_per_gpu=67_108_864, pairs=4,
                    l2="inputs larger than L2", parallelism=f"dp{world} (weak scaling)")
    if name == "C3":
        return dict(workload="C3: HEP100 stand-in (100 leaves, packed 380 B / aligned 480 B) x 67,108,864 records "
                             "per GPU, 6 ordered pairs of {packed AoS, aligned AoS, SoA MB}",
                    records_per_gpu=67_108_864, pairs=6,
                    l2="inputs larger than L2 (each pair moves 51-58 GB; L2 is 126 MB)",
                    parallelism=f"dp{world} (independent per-GPU relayout, weak scaling)")
    return dict(workload="C4: Listing-1 record (u16, f32 x2, f64, bool x3) 8192 x 8192, AoSoA32 -> SoA SB, "
                         "rows sharded over GPUs", records=8192 * 8192, pairs=1,
                l2="inputs larger than L2 (2.8 GB per copy at 1 GPU)",
                parallelism=f"dp{world} (extent sharding, strong scaling)")


SUBCFG = {
    "C2": dict(schema="particle7", extents=[16_777_216], kinds=["aos", "soa_mb", "aosoa8", "aosoa32"]),
    "C2_soa_sb": dict(schema="particle7", extents=[16_777_216], kinds=["aos", "soa_mb", "aosoa8", "aosoa32", "soa_sb"]),
    "C3": dict(schema="hep100", extents=[67_108_864], kinds=["aos", "aos_aligned", "soa_mb"]),
    "C3_soa_sb": dict(schema="hep100", extents=[67_108_864], kinds=["aos", "aos_aligned", "soa_sb"]),
    "C4": dict(schema="listing1", extents=[8192, 8192], kinds=["aosoa32", "soa_sb"]),
    # Split mappings in the same line
    "F1_hep": dict(schema="hep100", extents=[16_777_216], kinds=["aos", "soa_mb", "split_hep"]),
    "F1_listing1": dict(schema="listing1", extents=[67_108_864], kinds=["aos", "aos_aligned", "soa_mb", "split_pos"]),
    "C4_pairs": dict(schema="listing1", extents=[67_108_864], kinds=["aos", "aos_aligned", "soa_mb", "aosoa32"]),
    # transposing copies between storage orders; a
    # view is "kind/linearisation"
    "F4_p7": dict(schema="particle7", extents=[4096, 4096],
                  kinds=["aos/row", "aos/col", "aos/morton", "soa_mb/row", "soa_mb/col", "soa_mb/morton"]),
    "F4_hep": dict(schema="hep100", extents=[2048, 2048],
                   kinds=["aos/row", "aos_aligned/col", "soa_mb/row", "soa_mb/col", "aos/col", "aos/morton",
                          "soa_sb/row"]),
}


def pairs_of(name):
    sc = SUBCFG[name]
    if name == "C2":
        return l2_free_order(sc["kinds"])
    if name == "C2_soa_sb":
        # the 9 pairs with SoA SB, alternating directions so consecutive copies share no buffer
        o = sc["kinds"][:4]
        return ([("soa_sb", "soa_sb")] + [p for k in o for p in (("soa_sb", k), (k, "soa_sb"))])[::-1]
    if name == "C3":
        return l2_free_order(sc["kinds"], identities=False)
    if name == "C3_soa_sb":  # the 4 pairs with SoA SB, alternating directions
        return [("aos", "soa_sb"), ("soa_sb", "aos_aligned"), ("aos_aligned", "soa_sb"), ("soa_sb", "aos")]
    if name == "F1_hep":
        return [("aos", "split_hep"), ("split_hep", "soa_mb"), ("soa_mb", "split_hep"), ("split_hep", "aos")]
    if name == "C4_pairs":  # the 12 non-identity pairs, consecutive ones sharing no buffer
        return l2_free_order(sc["kinds"])[len(sc["kinds"]):]
    if name == "F4_p7":  # the 6 transposes measured since round 1
        return [("aos/row", "aos/col"), ("aos/row", "soa_mb/col"), ("soa_mb/col", "soa_mb/row"),
                ("aos/row", "aos/morton"), ("soa_mb/morton", "aos/col"), ("soa_mb/row", "aos/col")]
    if name == "F4_hep":  # one HEP100 pair per wide-transpose mode (+ the JIT's short tiles)
        return [("aos/row", "soa_mb/col"), ("soa_mb/col", "aos/row"), ("aos/row", "aos_aligned/col"),
                ("aos/col", "aos/morton"), ("soa_sb/row", "soa_mb/col")]
    if name == "F1_listing1":
        return [("aos", "split_pos"), ("split_pos", "aos_aligned"), ("soa_mb", "split_pos"), ("split_pos", "aos"),
                ("aos_aligned", "split_pos"), ("split_pos", "soa_mb")]
    return [("aosoa32", "soa_sb")]


class Ctx:
    def __init__(self, args, world, rank, local):
        import torch
        import torch.distributed as dist

        import paper_2106_04284_b200 as llama
        self.torch, self.dist, self.llama = torch, dist, llama
        self.args, self.world, self.rank, self.local = args, world, rank, local
        self.stream = torch.cuda.current_stream()
        self.rdev = "cpu" if getattr(args, "test_one_device", False) else "cuda"  # reduction tensors (gloo: host)

    def barrier(self):
        from paper_2106_04284_b200 import dist as D
        D.barrier()

    def max_over_ranks(self, v):
        from paper_2106_04284_b200 import dist as D
        return D.max_over_ranks(v, device=self.rdev)

    def min_over_ranks(self, v):
        return -self.max_over_ranks(-v)

    def event(self):
        return self.torch.cuda.Event(enable_timing=True)


def setup_views(ctx, name):
    llama = ctx.llama
    sc = SUBCFG[name]
    schema = W.SCHEMAS[sc["schema"]]
    ext = list(sc["extents"])
    if name == "C4":
        from paper_2106_04284_b200.shard import shard_extents
        ext, _ = shard_extents(ext, ctx.world, ctx.rank, multiple=32)
    pairs = pairs_of(name)
    kinds = sorted({x for p in pairs for x in p})
    maps = {k: llama.Mapping.from_spec(schema, ext, W.resolve_spec(k.split("/")[0]),
                                       lin=k.split("/")[1] if "/" in k else "row") for k in kinds}
    src = {k: maps[k].alloc("cuda") for k in kinds}
    dst = {k: maps[k].alloc("cuda") for k in kinds}
    for k in kinds:
        llama.generate(maps[k], src[k], 42 + ctx.rank)
    return maps, src, dst, pairs, ext


def roundtrip_check(ctx, maps, src, dst, pairs):
    """Per-rank self-check without the oracle (bench may not run it): for each
    pair, after the copy src[a] -> dst[b], the element-wise NAIVE kernel
    copies dst[b] back into dst[a]'s layout, which must equal src[a]
    byte for byte (round-trip identity; two different kernels)."""
    llama, torch = ctx.llama, ctx.torch
    ok = True
    for a, b in pairs:
        llama.copy(maps[a], src[a], maps[b], dst[b], stream=ctx.stream)
        if a != b:
            llama.copy(maps[b], dst[b], maps[a], dst[a], stream=ctx.stream, path="naive")
        torch.cuda.synchronize()
        ok = ok and all(blobs_equal(torch, x, y) for x, y in zip(dst[a], src[a]))
    return bool(ctx.min_over_ranks(1.0 if ok else 0.0) > 0.5)


def blobs_equal(torch, x, y, chunk=1 << 30):
    """Byte equality of two device blobs in 1 GiB chunks (C3's views leave no
    room for a full-size comparison temporary)."""
    if x.numel() != y.numel():
        return False
    return all(torch.equal(x[i:i + chunk], y[i:i + chunk]) for i in range(0, x.numel(), chunk))


def measure_config(ctx, name, steps, warmup, headline=False):
    """Times `steps` steps of the config's pairs (one llama_copy each) after
    `warmup` steps; per-pair times from a separate event-bracketed pass."""
    llama, torch = ctx.llama, ctx.torch
    maps, src, dst, pairs, ext = setup_views(ctx, name)
    stream = ctx.stream
    pair_bytes = [maps[a].footprint() + maps[b].footprint() for a, b in pairs]
    step_bytes = sum(pair_bytes)
    plans = [llama.plan(maps[a], maps[b]) for a, b in pairs]

    def step():
        for a, b in pairs:
            llama.copy(maps[a], src[a], maps[b], dst[b], stream=stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(ctx.local)  # every config: C3's 60-ms steps draw the most power
    clocks.start()
    time.sleep(0.3)
    ctx.barrier()
    torch.cuda.synchronize()
    l0 = llama.launch_count()
    t0, t1 = ctx.event(), ctx.event()
    t0.record(stream)
    for _ in range(steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    ctx.barrier()
    launches = llama.launch_count() - l0
    clk = clocks.stop()
    ms = ctx.max_over_ranks(t0.elapsed_time(t1) / steps)
    value = sum_over_ranks(ctx, step_bytes) / (ms * 1e-3) / 1e9  # every rank's bytes / the slowest rank's time

    # per pair: a separate pass, CUDA events around each copy
    ev = [[(ctx.event(), ctx.event()) for _ in pairs] for _ in range(steps)]
    for s in range(steps):
        for j, (a, b) in enumerate(pairs):
            ev[s][j][0].record(stream)
            llama.copy(maps[a], src[a], maps[b], dst[b], stream=stream)
            ev[s][j][1].record(stream)
    torch.cuda.synchronize()
    peak, peak_src = hbm_peak()
    per_pair = []
    for j, (a, b) in enumerate(pairs):
        t = statistics.median(ev[s][j][0].elapsed_time(ev[s][j][1]) for s in range(steps))
        path = plans[j]["path"] + ("_direct" if plans[j].get("direct") else "") + ("_jit" if plans[j].get("jit") else "") \
            + ("_wide" if plans[j].get("wide") else "")
        per_pair.append({"src": a, "dst": b, "path": path, "kernel": KERNEL.get(path, path), "bytes": pair_bytes[j],
                         "ms": t, "gbs": pair_bytes[j] / (t * 1e6), "frac": pair_bytes[j] / (t * 1e6) / peak})

    # dominant kernel: the largest share of the step
    share = {}
    for p in per_pair:
        e = share.setdefault(p["kernel"], [0.0, 0, 0])
        e[0] += p["ms"]
        e[1] += p["bytes"]
        e[2] += 1
    dom = max(share, key=lambda k: share[k][0])
    if share[dom][2] == len(pairs):
        # every launch of the step is the dominant kernel: its average launch
        # duration is the timed region divided by the launches (CUDA events on
        # the launching stream, back-to-back launches with PDL overlap)
        dom_ms, dom_bytes, how = ms / len(pairs), step_bytes / len(pairs), "timed region / launches per step"
    else:
        dom_ms, dom_bytes = share[dom][0] / share[dom][2], share[dom][1] / share[dom][2]
        how = "per-launch CUDA events (separate pass)"
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic, cold_frac = traffic_for(name, dom)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": dom, "launches_per_step": share[dom][2],
                "algorithmic_bytes_per_launch": dom_bytes, "peak_source": peak_src,
                "share_of_step": share[dom][0] / sum(v[0] for v in share.values()), "duration_from": how,
                "frac_isolated_launches": dom_bytes / (share[dom][0] / share[dom][2] * 1e-3) / 1e9 / peak,
                "frac_ncu_cold": cold_frac}

    # in-run references: a device memcpy of equal read+write bytes, and
    # the naive element-wise copy (the paper's comparison)
    a0 = max(maps, key=lambda k: maps[k].footprint())
    big_s, big_d = max(src[a0], key=lambda t: t.numel()), max(dst[a0], key=lambda t: t.numel())
    big_d.copy_(big_s)
    e0, e1 = ctx.event(), ctx.event()
    e0.record(stream)
    for _ in range(3):
        big_d.copy_(big_s)
    e1.record(stream)
    torch.cuda.synchronize()
    memcpy_gbs = 2 * big_s.numel() * 3 / (e0.elapsed_time(e1) * 1e-3) / 1e9
    naive_ms = 0.0
    for a, b in pairs:
        e0, e1 = ctx.event(), ctx.event()
        e0.record(stream)
        llama.copy(maps[a], src[a], maps[b], dst[b], stream=stream, path="naive")
        e1.record(stream)
        torch.cuda.synchronize()
        naive_ms += e0.elapsed_time(e1)
    rt = roundtrip_check(ctx, maps, src, dst, pairs)
    out = {"value": value, "unit": "GB/s", "ms_per_step": ms, "steps": steps, "warmup": warmup,
           "config": workload_desc(name, ctx.world), "local_extents": ext,
           "frac_of_measured_copy": value / ctx.world / peak,
           "frac_of_8tbs": value / ctx.world / NOMINAL_HBM_GBS,
           "roofline": roofline, "per_pair": per_pair,
           "min_pair_frac": min(p["frac"] for p in per_pair),
           "memcpy_gbs": memcpy_gbs, "memcpy_bytes": 2 * big_s.numel(),
           "naive_gpu_gbs": step_bytes / (naive_ms * 1e-3) / 1e9,
           "roundtrip_check": rt, "gpu_launches": launches}
    if clk is not None:
        out["clocks"] = clk
    views = (maps, src, dst, pairs) if headline else None
    return out, views


def sum_over_ranks(ctx, v):
    from paper_2106_04284_b200 import dist as D
    return D.sum_over_ranks(v, device=ctx.rdev)


def e2e_leg(ctx, maps, src, dst, pairs, steps):
    """End to end through the public API with HOST buffers: the step's 16
    copies as llama_copy_staged_batch from pinned host sources to pinned host
    destinations (slab H2D, relayout, D2H overlapped), timed on
    the device with the copies inside."""
    llama, torch = ctx.llama, ctx.torch
    names = sorted({x for p in pairs for x in p})
    hsrc = {k: [torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True) for t in src[k]] for k in names}
    hdst = {k: [torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True) for t in dst[k]] for k in names}
    for k in names:
        for h, t in zip(hsrc[k], src[k]):
            h.copy_(t)
    h2d = sum(maps[a].footprint() for a, b in pairs)
    d2h = sum(maps[b].footprint() for a, b in pairs)
    stager = llama.Stager(256 << 20)  # measured: 256 MiB slabs 87.7 vs 83.7 GB/s at 64 MiB
    batch = [(maps[a], hsrc[a], maps[b], hdst[b]) for a, b in pairs]
    llama.copy_staged_batch(stager, batch, stream=ctx.stream)
    torch.cuda.synchronize()
    ctx.barrier()
    e0, e1 = ctx.event(), ctx.event()
    e0.record(ctx.stream)
    for _ in range(steps):
        llama.copy_staged_batch(stager, batch, stream=ctx.stream)
    e1.record(ctx.stream)
    torch.cuda.synchronize()
    ems = ctx.max_over_ranks(e0.elapsed_time(e1) / steps)
    step_bytes = h2d + d2h
    value = step_bytes * ctx.world / (ems * 1e-3) / 1e9
    # in-run ceiling: pinned H2D and D2H at once on two streams, 512 MiB each
    # way (cudaMemcpyAsync through torch), the most any staged pipeline can move
    n = 512 << 20
    hs, hd = hsrc[names[0]][0][:n], hdst[names[0]][0][:n]
    da, db = torch.empty(n, dtype=torch.uint8, device="cuda"), torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def both():
        s1.wait_stream(ctx.stream)
        s2.wait_stream(ctx.stream)
        with torch.cuda.stream(s1):
            da[:hs.numel()].copy_(hs, non_blocking=True)
        with torch.cuda.stream(s2):
            hd.copy_(db[:hd.numel()], non_blocking=True)
        ctx.stream.wait_stream(s1)
        ctx.stream.wait_stream(s2)
    both()
    torch.cuda.synchronize()
    c0, c1 = ctx.event(), ctx.event()
    c0.record(ctx.stream)
    for _ in range(3):
        both()
    c1.record(ctx.stream)
    torch.cuda.synchronize()
    ceil = (hs.numel() + hd.numel()) / (c0.elapsed_time(c1) / 3 * 1e-3) / 1e9
    del da, db
    return {"value": value, "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ems,
            "ceiling_gbs": ceil, "frac_of_ceiling": value / ctx.world / ceil,
            "ceiling_method": "pinned H2D + D2H cudaMemcpyAsync at once on two streams, 512 MiB each way, per GPU",
            "method": "llama_copy_staged_batch: pinned host src -> device relayout -> pinned host dst, "
                      f"256 MiB slabs, one pipeline over the step's {len(pairs)} copies"}


def run_ours(args, world, rank, local):
    import torch
    import torch.distributed as dist
    if args.test_one_device:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.test_one_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = Ctx(args, world, rank, local)
    names = (args.configs or (DEFAULT_CONFIGS if args.config == "C2" else args.config)).split(",")
    head = args.config if args.config in names else names[0]
    warm = max(3, args.warmup)
    results = {}
    e2e = None
    for name in [head] + [n for n in names if n != head]:
        res, views = measure_config(ctx, name, args.steps, warm, headline=(name == head))
        results[name] = res
        if name == head and name == "C2" and not args.no_e2e:
            e2e = e2e_leg(ctx, *views, steps=max(1, args.e2e_steps))
        del views
        torch.cuda.empty_cache()
    h = results[head]
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline("C2" if head in ("C2", "C2_soa_sb") else head)
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": "GB/s", "cores": None, "kind": "oracle", "sample": f"failed: {ex}"}
    if e2e is None:
        e2e = {"value": None, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "skipped": "the end-to-end leg is measured on C2 (C3's 166 GB of views cannot be pinned on the host)"}
    if rank == 0:
        # the layout copies of BASELINE's configs and the split mappings (same
        # storage order on both sides); the transposing copies (F4_*, SURVEY
        # 8(f) f4) are reported as their own minimum
        allp = [dict(p, config=n) for n, r in results.items() if not n.startswith("F4") for p in r["per_pair"]]
        f4p = [dict(p, config=n) for n, r in results.items() if n.startswith("F4") for p in r["per_pair"]]
        worst = min(allp, key=lambda p: p["frac"])
        line = {"metric": METRIC, "value": h["value"], "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": warm, "ms_per_step": h["ms_per_step"], "higher_is_better": True,
                "scaling": "strong" if head == "C4" else "weak", "vs_baseline": None, "dtype": "u8",
                "data": "synthetic (splitmix64 per leaf, seed 42 + rank)", "config": h["config"],
                "roofline": h["roofline"], "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": h["gpu_launches"], "clocks": h.get("clocks"),
                "frac_of_measured_copy": h["frac_of_measured_copy"], "frac_of_8tbs": h["frac_of_8tbs"],
                "naive_gpu_gbs": h["naive_gpu_gbs"], "memcpy_gbs": h["memcpy_gbs"],
                "roundtrip_check": all(r["roundtrip_check"] for r in results.values()),
                "min_pair_frac": {"frac": worst["frac"], "gbs": worst["gbs"], "config": worst["config"],
                                  "pair": f"{worst['src']}->{worst['dst']}", "kernel": worst["kernel"],
                                  "over_pairs": len(allp)},
                "min_pair_frac_transposes": None if not f4p else (lambda w: {
                    "frac": w["frac"], "gbs": w["gbs"], "config": w["config"], "pair": f"{w['src']}->{w['dst']}",
                    "kernel": w["kernel"], "over_pairs": len(f4p)})(min(f4p, key=lambda p: p["frac"])),
                "configs": results}
        print(json.dumps(line), flush=True)
        if args.per_pair:
            with open(args.per_pair, "w") as f:
                json.dump(allp, f, indent=1)
        sys.stderr.write("\n".join(f"{p['config']:>9} {p['src']:>8} -> {p['dst']:<8} {p['path']:<15} "
                                   f"{p['ms']:.3f} ms {p['gbs']:.0f} GB/s ({p['frac']:.3f})" for p in allp) + "\n")
    if world > 1:
        dist.destroy_process_group()
    return 0


# --------------------------------------------------------- C5 cross-device
def run_c5(args, world, rank, local):
    """Cross-device relayout (BASELINE configs[4]): packed AoS on
    GPU i -> SoA MB on GPU (i+1) % W, 2^27 Particle7 per GPU.  Legs, all in
    this run:
      fused      the copy kernel's TMA bulk stores go straight into GPU i+1's
                 memory (torch symmetric memory peer pointers; the exchange is
                 fused into the relayout)
      fused_lsu  the same through the LSU-store kernel variant (knob no_tma)
      staged_ce  baseline (i), the paper's proposal: local relayout,
                 then cudaMemcpyAsync of every blob into the peer (copy engines)
      staged_nccl baseline (ii): local relayout, then NCCL send/recv around the ring
      ceiling    8 (= W) concurrent peer memcpys of the destination bytes around the ring
    Every leg's received destination is checked on its rank by a round trip
    through the NAIVE kernel against the regenerated source of rank i-1."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm

    import paper_2106_04284_b200 as llama
    torch.cuda.set_device(local)
    if "RANK" not in os.environ:  # `python bench.py --config C5` on one GPU: a one-rank ring (the peer is this GPU)
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(free_port()))
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = Ctx(args, world, rank, local)
    n = W.C5["extents"][0]
    schema = W.SCHEMAS[W.C5["schema"]]
    sm = llama.Mapping(schema, [n], *W.MAPPINGS["aos"])
    dm = llama.Mapping(schema, [n], *W.MAPPINGS["soa_mb"])
    src = sm.alloc("cuda")
    llama.generate(sm, src, 42 + rank)
    sizes = dm.blob_sizes()
    offs = [0]
    for b in sizes:
        offs.append(offs[-1] + (b + 255) // 256 * 256)
    buf = symm.empty(offs[-1], dtype=torch.uint8, device=f"cuda:{local}")
    hdl = symm.rendezvous(buf, dist.group.WORLD)
    peer, prev = (rank + 1) % world, (rank - 1) % world
    dst_peer = [int(hdl.buffer_ptrs[peer]) + offs[j] for j in range(len(sizes))]
    peer_views = [hdl.get_buffer(peer, (sizes[j],), torch.uint8, offs[j]) for j in range(len(sizes))]
    mine = [buf[offs[j]:offs[j] + sizes[j]] for j in range(len(sizes))]
    local_dst = dm.alloc("cuda")
    recv = [torch.empty_like(t) for t in local_dst]
    stream = ctx.stream

    def fused():
        llama.copy(sm, src, dm, dst_peer, stream=stream)

    def fused_lsu():
        llama.copy(sm, src, dm, dst_peer, stream=stream, knobs={"no_tma": 1})

    def staged_ce():
        llama.copy(sm, src, dm, local_dst, stream=stream)
        for pv, t in zip(peer_views, local_dst):
            pv.copy_(t, non_blocking=True)

    def staged_nccl():
        llama.copy(sm, src, dm, local_dst, stream=stream)
        ops = []
        for t, r in zip(local_dst, recv):
            ops.append(dist.P2POp(dist.isend, t, peer))
            ops.append(dist.P2POp(dist.irecv, r, prev))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        for r, m in zip(recv, mine):
            m.copy_(r, non_blocking=True)

    def ceiling():
        for pv, t in zip(peer_views, local_dst):
            pv.copy_(t, non_blocking=True)

    def timed(fn):
        for _ in range(max(3, args.warmup)):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = ctx.event(), ctx.event()
        e0.record(stream)
        for _ in range(args.steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        return ctx.max_over_ranks(e0.elapsed_time(e1) / args.steps)

    def check():
        """mine (written by rank prev) back to AoS with the naive kernel ==
        rank prev's source, regenerated here (seed 42 + prev)."""
        torch.cuda.synchronize()
        dist.barrier()
        ref = sm.alloc("cuda")
        llama.generate(sm, ref, 42 + prev)
        back = sm.alloc("cuda")
        llama.copy(dm, mine, sm, back, path="naive")
        torch.cuda.synchronize()
        ok = blobs_equal(torch, back[0], ref[0])
        for t in mine:
            t.fill_(0x5A)
        del ref, back
        return bool(ctx.min_over_ranks(1.0 if ok else 0.0) > 0.5)

    link_bytes = dm.footprint()  # every destination byte crosses NVLink once
    hbm_bytes = sm.footprint() + dm.footprint()
    legs = {}
    l0 = llama.launch_count()
    for name, fn in (("fused", fused), ("fused_lsu", fused_lsu), ("staged_ce", staged_ce),
                     ("staged_nccl", staged_nccl)):
        ms = timed(fn)
        legs[name] = {"ms": ms, "link_gbs_per_gpu": link_bytes / (ms * 1e-3) / 1e9,
                      "hbm_gbs_per_gpu": hbm_bytes / (ms * 1e-3) / 1e9, "parity_roundtrip": check()}
    launches = llama.launch_count() - l0
    llama.copy(sm, src, dm, local_dst, stream=stream)
    cms = timed(ceiling)
    ceil_gbs = link_bytes / (cms * 1e-3) / 1e9
    f = legs["fused"]
    if rank == 0:
        line = {"metric": METRIC, "value": hbm_bytes * world / (f["ms"] * 1e-3) / 1e9, "unit": "GB/s",
                "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": f["ms"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
                "data": "synthetic (splitmix64, seed 42 + rank)",
                "config": {"workload": "C5: Particle7 x 2^27 per GPU, packed AoS on GPU i -> SoA MB on GPU (i+1)%W "
                                       "through peer pointers (NVLink P2P stores fused into the relayout)",
                           "parallelism": f"ring of {world}"},
                "roofline": ({"bound": "nvlink", "achieved": f["link_gbs_per_gpu"], "peak": ceil_gbs, "unit": "GB/s",
                              "frac": f["link_gbs_per_gpu"] / ceil_gbs, "traffic": None, "kernel": "k_permute_ws",
                              "peak_source": f"in-run ceiling: {world} concurrent peer memcpys of {link_bytes} B "
                                             "around the ring"}
                             if world > 1 else
                             {"bound": "hbm", "achieved": f["hbm_gbs_per_gpu"], "unit": "GB/s", "peak": hbm_peak()[0],
                              "frac": f["hbm_gbs_per_gpu"] / hbm_peak()[0], "traffic": None, "kernel": "k_permute_ws",
                              "note": "1 rank: the peer is this GPU (no NVLink)"}),
                "legs": legs, "nvlink_ceiling_gbs_per_gpu": ceil_gbs, "gpu_launches": launches,
                "roundtrip_check": all(v["parity_roundtrip"] for v in legs.values()),
                "cpu_baseline": None,
                "e2e": {"value": None, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                        "skipped": "device-resident cross-device config"}}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
    return 0


# ------------------------------------------------------ n-body move (f3)
MOVE_METRIC = "n-body move GB/s (24 B read + 12 B written per particle), 256Mi Particle7 per GPU"
MOVE_LAYOUTS = ["aos", "soa_mb", "aosoa32", "split_p7"]
MOVE_USEFUL = 36  # bytes per particle: Pos + Vel read (24), Pos written (12)


def move_workload(world):
    return {"workload": "MOVE: n-body move (Listing P:643-645) on 268,435,456 Particle7 particles per GPU in "
                        "{packed AoS, SoA MB, AoSoA32, Split(Pos->SoA MB | Vel,Mass->AoSoA8)}",
            "particles_per_gpu": W.NBODY_MOVE_N, "layouts": MOVE_LAYOUTS, "dt": W.NBODY_TIMESTEP,
            "l2": "inputs larger than L2 (7.5 GB per layout; L2 is 126 MB)",
            "parallelism": f"dp{world} (independent particles per GPU, weak scaling)"}


def move_cpu_sample(target_s=10.0):
    """The oracle's move (1 thread) on a bounded prefix, all four layouts."""
    import numpy as np

    import oracle
    n = 1 << 18
    while True:
        aos = oracle.Mapping(W.PARTICLE7, [n], "aos")
        src = [np.frombuffer(W.particle_values(n, seed=42).tobytes(), np.uint8).copy()]
        views = {}
        for name in MOVE_LAYOUTS:
            m = oracle.mapping_from_spec(W.PARTICLE7, [n], W.resolve_spec(name))
            views[name] = (m, oracle.copy(aos, src, m))
        t0 = time.perf_counter()
        for name in MOVE_LAYOUTS:
            oracle.nbody_move(views[name][0], views[name][1], W.NBODY_TIMESTEP)
        dt = time.perf_counter() - t0
        if dt * 4 >= target_s or n >= W.NBODY_MOVE_N:
            return n, dt, MOVE_USEFUL * n * len(MOVE_LAYOUTS) / dt / 1e9
        n = min(W.NBODY_MOVE_N, max(n * 2, int(n * target_s / max(dt, 1e-3))))


def run_move_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    if args.warmup:
        move_cpu_sample(target_s=1.0)
    n, dt, value = move_cpu_sample(target_s=10.0)
    line = {"metric": MOVE_METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": 1,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic particles (S:685 recipe, seed 42)",
            "config": dict(move_workload(1), sample_particles=n), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"oracle move on {n} particles x {len(MOVE_LAYOUTS)} layouts"},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_move(args, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2106_04284_b200 as llama
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = Ctx(args, world, rank, local)
    n = W.NBODY_MOVE_N
    dt = float(np.float32(W.NBODY_TIMESTEP))
    stream = ctx.stream
    # initial particles (S:685 recipe; rank r holds particles r*n ..) as packed
    # AoS, relayouted into each layout with llama.copy
    aos = llama.Mapping(W.PARTICLE7, [n], "aos")
    a0 = aos.alloc("cuda")
    chunk = 1 << 24
    for i0 in range(0, n, chunk):
        v = W.particle_values(chunk, seed=42, i0=rank * n + i0)
        a0[0][i0 * 28:(i0 + chunk) * 28].copy_(torch.from_numpy(np.frombuffer(v.tobytes(), np.uint8).copy()))
    maps = {k: llama.Mapping.from_spec(W.PARTICLE7, [n], W.resolve_spec(k)) for k in MOVE_LAYOUTS}
    blobs = {}
    for k in MOVE_LAYOUTS:
        blobs[k] = maps[k].alloc("cuda")
        llama.copy(aos, a0, maps[k], blobs[k], stream=stream)
    del a0
    torch.cuda.synchronize()
    paths = {k: llama.nbody_move(maps[k], blobs[k], 0.0, stream=stream) for k in MOVE_LAYOUTS}

    def step():
        for k in MOVE_LAYOUTS:
            llama.nbody_move(maps[k], blobs[k], dt, stream=stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ctx.barrier()
    torch.cuda.synchronize()
    l0 = llama.launch_count()
    t0, t1 = ctx.event(), ctx.event()
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    ctx.barrier()
    launches = llama.launch_count() - l0
    clk = clocks.stop()
    ms = ctx.max_over_ranks(t0.elapsed_time(t1) / args.steps)
    step_bytes = MOVE_USEFUL * n * len(MOVE_LAYOUTS)
    value = step_bytes * world / (ms * 1e-3) / 1e9
    per = {}
    for k in MOVE_LAYOUTS:  # per layout (separate event-bracketed pass)
        e0, e1 = ctx.event(), ctx.event()
        e0.record(stream)
        for _ in range(args.steps):
            llama.nbody_move(maps[k], blobs[k], dt, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        kms = e0.elapsed_time(e1) / args.steps
        dram = (28 + 28) * n if k == "aos" else MOVE_USEFUL * n  # AoS moves whole records
        per[k] = {"path": paths[k], "ms": kms, "useful_gbs": MOVE_USEFUL * n / (kms * 1e-3) / 1e9,
                  "dram_gbs_expected": dram / (kms * 1e-3) / 1e9}
    peak, peak_src = hbm_peak()
    runs_ms = [per[k]["ms"] for k in MOVE_LAYOUTS if per[k]["path"] == "runs"]
    achieved = MOVE_USEFUL * n / (statistics.mean(runs_ms) * 1e-3) / 1e9
    traffic, cold = traffic_for("MOVE", "k_move_runs")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "k_move_runs", "launches_per_step": len(runs_ms),
                "algorithmic_bytes_per_launch": MOVE_USEFUL * n, "peak_source": peak_src,
                "share_of_step": sum(runs_ms) / sum(p["ms"] for p in per.values()),
                "duration_from": "per-layout CUDA events (separate pass)", "frac_ncu_cold": cold}
    e2e = None
    if not args.no_e2e:
        # through the public API with host buffers: slabs of every layout's
        # blobs DMA'd in, moved, DMA'd out (llama_nbody_move_staged); a split
        # view goes in whole, is moved, and comes back
        host = {k: [torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True) for t in blobs[k]]
                for k in MOVE_LAYOUTS}
        for k in MOVE_LAYOUTS:
            for h, t in zip(host[k], blobs[k]):
                h.copy_(t)
        nbytes = sum(maps[k].footprint() for k in MOVE_LAYOUTS)
        stager = llama.Stager(256 << 20)

        def e2e_step():
            for k in MOVE_LAYOUTS:
                if maps[k].kind != "split":
                    llama.nbody_move_staged(stager, maps[k], host[k], dt, stream=stream)
                    continue
                for h, t in zip(host[k], blobs[k]):
                    t.copy_(h, non_blocking=True)
                llama.nbody_move(maps[k], blobs[k], dt, stream=stream)
                for h, t in zip(host[k], blobs[k]):
                    h.copy_(t, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        ctx.barrier()
        e0, e1 = ctx.event(), ctx.event()
        e0.record(stream)
        for _ in range(max(1, args.e2e_steps)):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = ctx.max_over_ranks(e0.elapsed_time(e1) / max(1, args.e2e_steps))
        e2e = {"value": step_bytes * world / (ems * 1e-3) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "ms_per_step": ems,
               "method": "llama_nbody_move_staged: pinned host blobs -> 256 MiB slabs DMA'd in, moved, DMA'd out, "
                         "overlapped (split view: whole-view DMA in, move, DMA out)"}
        del host
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cn, cdt, cval = move_cpu_sample()
            cpu = {"value": cval, "unit": "GB/s", "cores": 1, "kind": "oracle",
                   "sample": f"oracle move on a prefix of {cn} particles x {len(MOVE_LAYOUTS)} layouts, {cdt:.1f} s"}
        except Exception as ex:
            cpu = {"value": None, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": f"failed: {ex}"}
    if rank == 0:
        ratio = per["soa_mb"]["ms"] / per["aos"]["ms"]
        line = {"metric": MOVE_METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic particles (S:685 recipe, seed 42)",
                "config": move_workload(world), "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk, "per_layout": per,
                "soa_over_aos_runtime": ratio,
                "paper_soa_over_aos_runtime": {"gpu": [0.55, 0.60, 0.62], "cpu": 0.646, "cite": "P:734, P:691",
                                               "aos_useful_fraction": 1 - (1 + 4) / (7 + 7)}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.cpu_child:
        print(json.dumps(cpu_child(args.config)), flush=True)
        return 0
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run; rank 0 prints the line
        return subprocess.call(relaunch_cmd(argv, args.gpus, free_port()))
    world, rank, local = check_world(args.gpus, os.environ)
    if args.impl == "reference":
        if args.config == "MOVE":
            return run_move_reference(args)
        return run_reference(args, W.CONFIGS["C2" if args.config == "C5" else args.config])
    if args.config == "MOVE":
        return run_move(args, world, rank, local)
    if args.config == "C5":
        return run_c5(args, world, rank, local)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
