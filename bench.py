#!/usr/bin/env python
"""Benchmark: layout-copy GB/s (read + write bytes) per mapping pair on B200.

Default workload (BASELINE.json configs[1], "C2"): 16,777,216 Particle7
records (7 x f32), all 16 ordered pairs of {packed AoS, SoA
multi-blob, AoSoA8, AoSoA32}.  One step = the 16 layout-aware copies, each one
llama_copy through the C ABI.  value = sum over pairs of (src footprint + dst
footprint) / step time, summed over ranks (weak scaling: every rank relayouts
its own 16M records; no data-path collective).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

--impl reference times the CPU oracle (oracle/, plain C naive copy) on a
bounded sample of the same workload; it needs no GPU.

--config MOVE: the n-body move (Listing P:643-645) on 256Mi
Particle7 particles per GPU in four layouts {packed AoS, SoA MB,
AoSoA32, Split(Pos -> SoA MB | rest -> AoSoA8)}; one step = one move per layout;
value = algorithmic bytes (24 read + 12 written per particle) / step time.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
METRIC = W_METRIC = "layout-copy GB/s (read+write) per mapping pair vs 8 TB/s HBM, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C2", "C3", "C4", "C5", "MOVE"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--per-pair", default=None, help="write per-pair timings (json) to this file")
    ap.add_argument("--pair-events", action="store_true",
                    help="record CUDA events around every copy inside the timed region (costs ~5%%); by default "
                         "per-pair times come from a separate event-bracketed pass")
    return ap.parse_args()


def hbm_peak():
    try:
        with open(MEASURED_PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def workload_desc(cfg, world):
    if cfg["name"] == "C2":
        return dict(workload="C2: Particle7 (7x f32) x 16,777,216 records per GPU, 16 ordered pairs of "
                             "{packed AoS, SoA MB, AoSoA8, AoSoA32}",
                    records_per_gpu=cfg["extents"][0], pairs=len(cfg["pairs"]),
                    l2="inputs larger than L2 (each pair reads 470 MB and writes 470 MB; L2 is 126 MB)",
                    parallelism=f"dp{world} (independent per-GPU relayout, weak scaling)")
    if cfg["name"] == "C3":
        return dict(workload="C3: HEP100 stand-in (100 leaves, packed 380 B / aligned 480 B) x 67,108,864 records "
                             "per GPU, 6 ordered pairs of {packed AoS, aligned AoS, SoA MB}",
                    records_per_gpu=cfg["extents"][0], pairs=len(cfg["pairs"]),
                    l2="inputs larger than L2 (each pair moves 51-64 GB; L2 is 126 MB)",
                    parallelism=f"dp{world} (independent per-GPU relayout, weak scaling)")
    return dict(workload="C4: Listing-1 record (u16, f32 x2, f64, bool x3) 8192 x 8192, AoSoA32 -> SoA SB, "
                         "rows sharded over GPUs", records=8192 * 8192, pairs=1,
                l2="inputs larger than L2", parallelism=f"dp{world} (extent sharding, strong scaling)")


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
def cpu_baseline(cfg, target_s=12.0):
    """The oracle (plain C naive copy, 1 thread) on a bounded prefix of the
    workload: every pair on the same prefix of n' records."""
    import oracle
    schema = W.SCHEMAS[cfg["schema"]]
    names = sorted({x for p in cfg["pairs"] for x in p})
    # calibrate n' so that all pairs together take ~target_s
    n_try = 1 << 16
    views, maps = {}, {}

    def setup(n):
        for name in names:
            maps[name] = oracle.Mapping(schema, [n], *W.MAPPINGS[name])
            views[name] = oracle.make_view(maps[name], 42)

    setup(n_try)
    t0 = time.perf_counter()
    for a, b in cfg["pairs"]:
        oracle.copy(maps[a], views[a], maps[b])
    dt = time.perf_counter() - t0
    n = int(n_try * max(1.0, target_s / max(dt, 1e-6)))
    n = max(1 << 16, min(n, cfg["extents"][0] if cfg["name"] == "C2" else 1 << 24))
    n -= n % 32
    setup(n)
    dsts = {b: maps[b].alloc() for b in names}
    total_bytes = 0
    t0 = time.perf_counter()
    for a, b in cfg["pairs"]:
        oracle.copy(maps[a], views[a], maps[b], dsts[b])
        total_bytes += sum(maps[a].blob_sizes()) + sum(maps[b].blob_sizes())
    dt = time.perf_counter() - t0
    return {"value": total_bytes / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"{cfg['name']} pairs on a prefix of {n} records ({total_bytes / 1e9:.2f} GB moved, "
                      f"{dt:.1f} s, plain C naive copy, 1 thread)"}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    schema = W.SCHEMAS[cfg["schema"]]
    names = sorted({x for p in cfg["pairs"] for x in p})
    # each step: all pairs on a bounded prefix, sized so steps+warmup take minutes at most
    n = 1 << 20
    maps = {k: oracle.Mapping(schema, [n], *W.MAPPINGS[k]) for k in names}
    views = {k: oracle.make_view(maps[k], 42) for k in names}
    dsts = {k: maps[k].alloc() for k in names}
    step_bytes = sum(sum(maps[a].blob_sizes()) + sum(maps[b].blob_sizes()) for a, b in cfg["pairs"])

    def step():
        for a, b in cfg["pairs"]:
            oracle.copy(maps[a], views[a], maps[b], dsts[b])

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / max(1, args.steps)
    value = step_bytes / dt / 1e9
    line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (splitmix64, seed 42)",
            "config": dict(workload_desc(cfg, 1), sample_records=n), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"{cfg['name']} pairs on a prefix of {n} records per step"},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- ours
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2106_04284_b200 as llama

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    schema = W.SCHEMAS[cfg["schema"]]
    if cfg["name"] == "C4":
        from paper_2106_04284_b200.shard import shard_extents
        ext, _ = shard_extents(list(cfg["extents"]), world, rank, multiple=32)
    else:
        ext = list(cfg["extents"])
    names = sorted({x for p in cfg["pairs"] for x in p})
    maps = {k: llama.Mapping(schema, ext, *W.MAPPINGS[k]) for k in names}
    src = {k: maps[k].alloc("cuda") for k in names}
    dst = {k: maps[k].alloc("cuda") for k in names}
    for k in names:
        llama.generate(maps[k], src[k], 42)
    stream = torch.cuda.current_stream()
    pairs = cfg["pairs"]
    pair_bytes = [sum(maps[a].blob_sizes()) + sum(maps[b].blob_sizes()) for a, b in pairs]
    step_bytes = sum(pair_bytes)
    plans = [llama.plan(maps[a], maps[b]) for a, b in pairs]

    def barrier():
        if world > 1:
            dist.barrier()

    def step(events=None):
        for j, (a, b) in enumerate(pairs):
            if events is not None:
                events[j][0].record(stream)
            llama.copy(maps[a], src[a], maps[b], dst[b], stream=stream)
            if events is not None:
                events[j][1].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    # timed region: K steps; per-launch events on the launching stream
    ev = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in pairs]
          for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    launches0 = llama.launch_count()
    t_start.record(stream)
    for s in range(args.steps):
        step(ev[s] if args.pair_events else None)
    t_end.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = llama.launch_count() - launches0
    clk = clocks.stop()
    if not args.pair_events:  # per-pair times from a separate, event-bracketed pass
        for s in range(args.steps):
            step(ev[s])
        torch.cuda.synchronize()
    ms = t_start.elapsed_time(t_end) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = step_bytes * world / (ms * 1e-3) / 1e9

    per_pair = []
    for j, (a, b) in enumerate(pairs):
        times = [ev[s][j][0].elapsed_time(ev[s][j][1]) for s in range(args.steps)]
        per_pair.append({"src": a, "dst": b, "path": plans[j]["path"] + ("_direct" if plans[j].get("direct") else ""),
                         "bytes": pair_bytes[j],
                         "ms": statistics.median(times), "gbs": pair_bytes[j] / (statistics.median(times) * 1e6)})
    # dominant kernel path = largest share of the step
    share = {}
    for p in per_pair:
        share.setdefault(p["path"], [0.0, 0, 0])
        share[p["path"]][0] += p["ms"]
        share[p["path"]][1] += p["bytes"]
        share[p["path"]][2] += 1
    dom = max(share, key=lambda k: share[k][0])
    peak, peak_src = hbm_peak()
    if share[dom][2] == len(pairs):
        # every launch of the step is the dominant kernel: its average launch
        # duration is the timed region (CUDA events on the launching stream)
        # divided by the launches, gaps between launches included
        dom_ms_avg = ms / len(pairs)
        dom_bytes_avg = step_bytes / len(pairs)
        how = "timed region / launches per step"
    else:
        dom_ms_avg = share[dom][0] / share[dom][2]
        dom_bytes_avg = share[dom][1] / share[dom][2]
        how = "per-launch CUDA events (separate pass)"
    achieved = dom_bytes_avg / (dom_ms_avg * 1e-3) / 1e9
    traffic = None
    try:  # dram read+write bytes per launch of this kernel from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(dom, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": {"permute": "k_permute_ws", "permute_direct": "k_permute_direct", "blobcopy": "k_bulkcopy",
                           "run": "k_run", "naive": "k_naive"}.get(dom, dom),
                "launches_per_step": share[dom][2], "algorithmic_bytes_per_launch": dom_bytes_avg,
                "peak_source": peak_src, "share_of_step": share[dom][0] / sum(v[0] for v in share.values()),
                "duration_from": how}

    extra = {}
    if rank == 0:
        # in-run references: naive element-wise GPU copy and a plain device memcpy of equal bytes
        naive_ms = 0.0
        for j, (a, b) in enumerate(pairs):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            llama.copy(maps[a], src[a], maps[b], dst[b], stream=stream, path="naive")
            e0.record(stream)
            llama.copy(maps[a], src[a], maps[b], dst[b], stream=stream, path="naive")
            e1.record(stream)
            torch.cuda.synchronize()
            naive_ms += e0.elapsed_time(e1)
        nb = min(pair_bytes[0] // 2, 2 << 30)
        x = torch.empty(nb, dtype=torch.uint8, device="cuda")
        y = torch.empty_like(x)
        y.copy_(x)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(5):
            y.copy_(x)
        e1.record(stream)
        torch.cuda.synchronize()
        memcpy_gbs = 2 * nb * 5 / (e0.elapsed_time(e1) * 1e-3) / 1e9
        del x, y
        extra = {"naive_gpu_gbs": step_bytes / (naive_ms * 1e-3) / 1e9, "memcpy_gbs": memcpy_gbs,
                 "frac_of_8tbs": value / world / 8000.0, "frac_of_measured_copy": value / world / peak}

    # end to end through the public API with HOST buffers: H2D of each pair's
    # source, the copy, D2H of its destination, every step
    e2e = None
    if cfg["name"] == "C3" and not args.no_e2e:
        e2e = {"value": None, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
               "skipped": "C3's host views (83 GB of sources + 83 GB of destinations, pinned) are not "
                          "allocated; the staged host path is measured on C2"}
    elif not args.no_e2e:
        hsrc = {k: [torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True) for t in src[k]] for k in names}
        hdst = {k: [torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True) for t in dst[k]] for k in names}
        for k in names:
            for h, t in zip(hsrc[k], src[k]):
                h.copy_(t)
        h2d = sum(sum(maps[a].blob_sizes()) for a, b in pairs)
        d2h = sum(sum(maps[b].blob_sizes()) for a, b in pairs)

        stager = llama.Stager(256 << 20)  # measured: 256 MiB slabs 87.7 vs 83.7 GB/s at 64 MiB

        batch = [(maps[a], hsrc[a], maps[b], hdst[b]) for a, b in pairs]

        def e2e_step():
            # the public API's cross-address-space copy (llama_copy_staged_batch,
            # P:578-579): slab DMA in, relayout on the device, DMA out, overlapped
            # across all 16 copies of the step
            llama.copy_staged_batch(stager, batch, stream=stream)

        e2e_step()
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / args.e2e_steps
        if world > 1:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": step_bytes * world / (ems * 1e-3) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": ems,
               "method": "llama_copy_staged_batch: pinned host src -> device relayout -> pinned host dst, "
                         f"256 MiB slabs, one pipeline over the step's {len(pairs)} copies"}
        del hsrc, hdst

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg)
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": "GB/s", "cores": 1, "kind": "oracle", "sample": f"failed: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
                "scaling": "weak" if cfg["name"] in ("C2", "C3") else "strong", "vs_baseline": None, "dtype": "u8",
                "data": "synthetic (splitmix64 per leaf, seed 42)", "config": workload_desc(cfg, world),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk, **extra}
        print(json.dumps(line), flush=True)
        if args.per_pair:
            with open(args.per_pair, "w") as f:
                json.dump(per_pair, f, indent=1)
        else:
            sys.stderr.write("\n".join(f"{p['src']:>8} -> {p['dst']:<8} {p['path']:<9} {p['ms']:.3f} ms "
                                       f"{p['gbs']:.0f} GB/s" for p in per_pair) + "\n")
    if world > 1:
        dist.destroy_process_group()
    return 0


# --------------------------------------------------------- C5 cross-device
def run_c5(args, cfg):
    """Cross-device relayout (BASELINE configs[4]): packed AoS on
    GPU i -> SoA MB on GPU (i+1) % W.  Each rank's destination blobs live in
    one torch symmetric-memory buffer; rank i's copy kernel writes (TMA bulk
    stores) straight into rank i+1's buffer through its peer pointers -- the
    exchange step is fused into the copy, NCCL only for barriers and the
    max-over-ranks time.  Needs >= 2 GPUs with peer access (torchrun)."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm

    import paper_2106_04284_b200 as llama
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = cfg["extents"][0]
    schema = W.SCHEMAS[cfg["schema"]]
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
    peer = (rank + 1) % world
    dst_peer = [int(hdl.buffer_ptrs[peer]) + offs[j] for j in range(len(sizes))]
    stream = torch.cuda.current_stream()
    for _ in range(max(3, args.warmup)):
        llama.copy(sm, src, dm, dst_peer, stream=stream)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        llama.copy(sm, src, dm, dst_peer, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    nbytes = sm.footprint() + dm.footprint()
    link_bytes = dm.footprint()  # every destination byte crosses NVLink
    # the rank's own destination (written by rank - 1) against the oracle, sampled
    import numpy as np

    import oracle
    prev = (rank - 1) % world
    so = oracle.Mapping(schema, [n], *W.MAPPINGS["aos"])
    do = oracle.Mapping(schema, [n], *W.MAPPINGS["soa_mb"])
    ok = True
    for a in (0, n // 2, n - 4096):
        b = a + 4096
        swin = [np.zeros((b - a) * 28, np.uint8)]
        oracle.generate(so, swin, 42 + prev, a, b, base=[a * 28])
        exp = [np.zeros((b - a) * 4, np.uint8) for _ in range(7)]
        oracle.copy_range(so, swin, [a * 28], do, exp, [a * 4] * 7, a, b)
        for j in range(7):
            got = buf[offs[j] + a * 4: offs[j] + b * 4].cpu().numpy()
            ok = ok and np.array_equal(got, exp[j])
    okt = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    if rank == 0:
        gbs = nbytes * world / (ms * 1e-3) / 1e9
        link = link_bytes / (ms * 1e-3) / 1e9
        print(json.dumps({"metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
                          "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic (splitmix64)",
                          "config": {"workload": "C5: Particle7 x 2^27 per GPU, packed AoS on GPU i -> SoA MB on "
                                                 "GPU (i+1)%W through peer pointers (NVLink P2P stores)",
                                     "parallelism": f"ring of {world}"},
                          "roofline": ({"bound": "nvlink", "achieved": link, "peak": 770.0, "unit": "GB/s",
                                        "frac": link / 770.0, "traffic": None,
                                        "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction"}
                                       if world > 1 else
                                       {"bound": "hbm", "achieved": nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s",
                                        "peak": hbm_peak()[0], "frac": nbytes / (ms * 1e-3) / 1e9 / hbm_peak()[0],
                                        "traffic": None, "note": "1 rank: the peer is this GPU (no NVLink)"}),
                          "parity_sampled": bool(okt.item())}), flush=True)
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


def run_move(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2106_04284_b200 as llama
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = W.NBODY_MOVE_N
    dt = float(np.float32(W.NBODY_TIMESTEP))
    stream = torch.cuda.current_stream()
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

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        for k in MOVE_LAYOUTS:
            llama.nbody_move(maps[k], blobs[k], dt, stream=stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    l0 = llama.launch_count()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    launches = llama.launch_count() - l0
    clk = clocks.stop()
    ms = t0.elapsed_time(t1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    step_bytes = MOVE_USEFUL * n * len(MOVE_LAYOUTS)
    value = step_bytes * world / (ms * 1e-3) / 1e9
    # per layout (separate event-bracketed pass)
    per = {}
    for k in MOVE_LAYOUTS:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
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
    dom = "runs"
    runs_ms = [per[k]["ms"] for k in MOVE_LAYOUTS if per[k]["path"] == "runs"]
    achieved = MOVE_USEFUL * n / (statistics.mean(runs_ms) * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get("move_runs", {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "k_move_runs", "launches_per_step": len(runs_ms),
                "algorithmic_bytes_per_launch": MOVE_USEFUL * n, "peak_source": peak_src,
                "share_of_step": sum(runs_ms) / sum(p["ms"] for p in per.values()),
                "duration_from": "per-layout CUDA events (separate pass)"}
    e2e = None
    if not args.no_e2e:
        # through the public API with host buffers: H2D of the step's particles
        # (every layout's blobs), the moves, D2H of the results
        host = {k: [torch.empty(t.numel(), dtype=torch.uint8, pin_memory=True) for t in blobs[k]]
                for k in MOVE_LAYOUTS}
        for k in MOVE_LAYOUTS:
            for h, t in zip(host[k], blobs[k]):
                h.copy_(t)
        nbytes = sum(maps[k].footprint() for k in MOVE_LAYOUTS)
        stager = llama.Stager(256 << 20)  # measured: 256 MiB slabs 87.7 vs 83.7 GB/s at 64 MiB

        def e2e_step():
            # the public API on host blobs: slabs DMA'd in, moved, DMA'd out,
            # overlapped (llama_nbody_move_staged); a split view (no slab
            # views) goes in whole, is moved, and comes back
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
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(max(1, args.e2e_steps)):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / max(1, args.e2e_steps)
        if world > 1:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
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


def main():
    args = parse()
    if args.config == "MOVE":
        return run_move_reference(args) if args.impl == "reference" else run_move(args)
    cfg = W.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.config == "C5":
        return run_c5(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
