"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host path:
extent sharding and the max-over-ranks timing reduction that
bench.py uses.  Each rank relayouts its own slab with the oracle; the slabs
together must equal the global copy (AoS/AoSoA byte-identical concatenation,
SoA per-shard sub-arrays; reading #18)."""
import os
import socket

import numpy as np
import pytest

import workloads as W
from paper_2106_04284_b200.shard import shard_extents


def test_shard_extents_partition():
    for ext in ([8192, 8192], [100], [37, 3], [1, 64], [0, 4]):
        for world in (1, 2, 3, 4, 8):
            for mult in (1, 8, 32):
                rows = []
                first = 0
                for r in range(world):
                    loc, f = shard_extents(ext, world, r, multiple=mult)
                    assert loc[1:] == ext[1:]
                    assert f == first
                    inner = int(np.prod(ext[1:])) if len(ext) > 1 else 1
                    first += loc[0] * inner
                    rows.append(loc[0])
                assert sum(rows) == ext[0]
    loc, f = shard_extents([8192, 8192], 8, 3, multiple=32)
    assert loc == [1024, 8192] and f == 3 * 1024 * 8192


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import oracle
    from paper_2106_04284_b200.dist import max_over_ranks
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ext = [64, 48]
        loc, first = shard_extents(ext, world, rank, multiple=32)
        out = {}
        for a, b in [("aosoa32", "soa_sb"), ("aos", "aosoa8"), ("soa_mb", "aos_aligned")]:
            sm = oracle.Mapping(W.LISTING1, loc, *W.MAPPINGS[a])
            dm = oracle.Mapping(W.LISTING1, loc, *W.MAPPINGS[b])
            src = sm.alloc()
            # the rank's local view holds global records [first, first + n_local): its blobs are the
            # global source's bytes for that slab (the generator is keyed by the global record index)
            gsm = oracle.Mapping(W.LISTING1, ext, *W.MAPPINGS[a])
            gsrc = gsm.alloc()
            oracle.generate(gsm, gsrc, 42)
            n_loc = int(np.prod(loc))
            # local source = global source restricted to the slab (AoS / AoSoA / SoA MB slab bytes)
            for k in range(sm.blob_count):
                if a == "soa_mb":
                    s_k = sm.sizes[k]
                    src[k][:] = gsrc[k][first * s_k:(first + n_loc) * s_k]
                else:
                    span = sm.blob_sizes()[0]
                    off = gsm.addr(first, 0)[1] if n_loc else 0
                    src[k][:] = gsrc[k][off:off + span]
            out[(a, b)] = [x.tobytes() for x in oracle.copy(sm, src, dm)]
        objs = [None] * world
        dist.all_gather_object(objs, (first, loc, out))
        t = max_over_ranks(1.0 + rank)
        if rank == 0:
            q.put((objs, t))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_relayout_gloo():
    import torch.multiprocessing as mp

    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    objs, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0  # max over ranks of (1 + rank)
    ext = [64, 48]
    for (a, b) in [("aosoa32", "soa_sb"), ("aos", "aosoa8"), ("soa_mb", "aos_aligned")]:
        gs = oracle.Mapping(W.LISTING1, ext, *W.MAPPINGS[a])
        gd = oracle.Mapping(W.LISTING1, ext, *W.MAPPINGS[b])
        full = oracle.copy(gs, oracle.make_view(gs, 42), gd)
        if b == "soa_sb":
            sizes = gd.sizes
            n = 64 * 48
            starts = np.cumsum([0] + [n * s for s in sizes])
            for first, loc, out in objs:
                nl = int(np.prod(loc))
                lstarts = np.cumsum([0] + [nl * s for s in sizes])
                for k, s in enumerate(sizes):
                    got = out[(a, b)][0][lstarts[k]:lstarts[k + 1]]
                    assert got == full[0][starts[k] + first * s:starts[k] + (first + nl) * s].tobytes()
        else:
            cat = b"".join(o[2][(a, b)][0] for o in objs)
            assert cat == full[0].tobytes()
