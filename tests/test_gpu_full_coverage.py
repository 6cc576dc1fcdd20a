"""Full-coverage GPU parity at BASELINE.json's full sizes, in the launch
configuration bench.py times (AUTO plans): every destination byte (padding
included) and every generated source byte is compared with the CPU oracle
(SURVEY §8(c) "chunked parity": slabs of records, each slab's byte ranges
copied to the host and checked against the oracle's windowed generator and
copy, slabs spread over host threads; the oracle is plain C called through
ctypes, which releases the GIL).

  C3   67,108,864 HEP100 records, all 6 ordered pairs of {packed AoS, aligned
       AoS, SoA MB} (the paper's 100-leaf event workload)
  C4   sharded as bench.py shards it (rows over world in {1, 2, 4, 8}); each
       rank's local copy equals the global oracle copy restricted to its slab
       (SoA SB: per-shard sub-arrays, reading #18)
  C5   2^27 Particle7 records, packed AoS -> SoA MB (the cross-device copy's
       kernel; with one GPU the peer is this GPU)
  f4   the 4096 x 4096 transposing copies DESIGN.md §8 reports
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def llama():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_04284_b200 as m
    return m


def _threads(per_thread_bytes):
    """Host threads for the slab walk: cores, bounded by host memory."""
    try:
        avail = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        avail = 16 << 30
    by_mem = max(1, int(avail * 0.5 // max(per_thread_bytes, 1)))
    return max(1, min(len(os.sched_getaffinity(0)), 48, by_mem))


def _par_generate(oracle, m, blobs, seed, n, threads, pad=None):
    """oracle.generate over [0, n) in record windows on several host threads
    (disjoint bytes of the same blobs)."""
    if pad is not None:
        for b in blobs:
            b.fill(pad)
    step = max(1, -(-n // (threads * 4)))
    with ThreadPoolExecutor(threads) as ex:
        list(ex.map(lambda a: oracle.generate(m, blobs, seed, a, min(n, a + step)), range(0, n, step)))


def _per_record(m, n):
    """Bytes per record of each blob for AoS / SoA MB layouts (blob size / N)."""
    return [s // n for s in m.blob_sizes()]


# -------------------------------------------------------------------- C3
@pytest.mark.parametrize("a", ["aos", "aos_aligned", "soa_mb"])
def test_c3_full_coverage(llama, oracle_mod, a):
    """C3 at 67,108,864 records: source layout `a` into both other layouts,
    every source and destination byte of the 2 pairs compared."""
    cfg = W.C3
    schema, ext = W.SCHEMAS[cfg["schema"]], list(cfg["extents"])
    n = ext[0]
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if free < 100e9:
        pytest.skip("needs ~97 GB of device memory")
    outs = [b for (x, b) in cfg["pairs"] if x == a]
    sm = llama.Mapping(schema, ext, *W.MAPPINGS[a])
    so = oracle_mod.Mapping(schema, ext, *W.MAPPINGS[a])
    sb = sm.alloc()
    llama.generate(sm, sb, 42, pad_byte=0xCD)  # poisoned source padding (reading #13)
    dms = {b: llama.Mapping(schema, ext, *W.MAPPINGS[b]) for b in outs}
    dos = {b: oracle_mod.Mapping(schema, ext, *W.MAPPINGS[b]) for b in outs}
    dbs = {}
    for b in outs:
        dbs[b] = dms[b].alloc()
        for t in dbs[b]:
            t.fill_(0x5A)  # an unwritten byte cannot pass
        llama.copy(sm, sb, dms[b], dbs[b])
    torch.cuda.synchronize()
    sper = _per_record(so, n)
    dper = {b: _per_record(dos[b], n) for b in outs}
    slab = 1 << 18
    threads = _threads(slab * (2 * sum(sper) + 2 * sum(sum(p) for p in dper.values())))

    def check(r0):
        r1 = min(n, r0 + slab)
        slo = [r0 * p for p in sper]
        ref = [np.full((r1 - r0) * p, 0xCD, np.uint8) for p in sper]
        oracle_mod.generate(so, ref, 42, r0, r1, base=slo)
        for j, p in enumerate(sper):  # the GPU source is the oracle's (P13)
            if not np.array_equal(sb[j][r0 * p:r1 * p].cpu().numpy(), ref[j]):
                return ("src", a, r0, j)
        for b in outs:
            dlo = [r0 * p for p in dper[b]]
            exp = [np.zeros((r1 - r0) * p, np.uint8) for p in dper[b]]
            oracle_mod.copy_range(so, ref, slo, dos[b], exp, dlo, r0, r1)
            for j, p in enumerate(dper[b]):
                if not np.array_equal(dbs[b][j][r0 * p:r1 * p].cpu().numpy(), exp[j]):
                    return ("dst", a, b, r0, j)
        return None

    with ThreadPoolExecutor(threads) as ex:
        bad = [r for r in ex.map(check, range(0, n, slab)) if r is not None]
    assert not bad, bad[:5]
    # every byte of every blob lies in some slab: the windows tile the blobs
    assert all(s == n * p for s, p in zip(so.blob_sizes(), sper))
    for b in outs:
        assert all(s == n * p for s, p in zip(dos[b].blob_sizes(), dper[b]))
    del sb, dbs
    torch.cuda.empty_cache()


# -------------------------------------------------------------------- C4
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_c4_sharded_full_coverage(llama, oracle_mod, world):
    """C4 (Listing-1, 8192 x 8192, AoSoA32 -> SoA SB) sharded over `world`
    ranks exactly as bench.py shards it (shard_extents, 32-record multiples),
    the ranks' copies run one after another on this GPU: each rank's local
    source is the global source's bytes of its slab (AoSoA: a contiguous block
    range), and each rank's local SoA SB equals the global oracle copy's
    sub-arrays restricted to its slab (reading #18); the slabs cover every
    record once."""
    from paper_2106_04284_b200.shard import shard_extents
    cfg = W.C4
    schema, ext = W.SCHEMAS[cfg["schema"]], list(cfg["extents"])
    n = ext[0] * ext[1]
    gs = llama.Mapping(schema, ext, *W.MAPPINGS["aosoa32"])
    gsb = gs.alloc()
    llama.generate(gs, gsb, 42)
    go = oracle_mod.Mapping(schema, ext, *W.MAPPINGS["aosoa32"])
    gdo = oracle_mod.Mapping(schema, ext, *W.MAPPINGS["soa_sb"])
    threads = _threads(256 << 20)
    src = go.alloc()
    _par_generate(oracle_mod, go, src, 42, n, threads)
    assert np.array_equal(gsb[0].cpu().numpy(), src[0])
    exp = oracle_mod.copy(go, src, gdo, nthreads=threads)[0]
    sizes = [2, 4, 4, 8, 1, 1, 1]  # Listing-1 leaves
    starts = np.cumsum([0] + [n * s for s in sizes])
    block = 32 * sum(sizes)  # AoSoA32 block bytes
    covered = 0
    for rank in range(world):
        loc, first = shard_extents(ext, world, rank, multiple=32)
        nl = loc[0] * loc[1]
        assert first == covered and first % 32 == 0
        covered += nl
        sm = llama.Mapping(schema, loc, *W.MAPPINGS["aosoa32"])
        dm = llama.Mapping(schema, loc, *W.MAPPINGS["soa_sb"])
        off = first // 32 * block
        lsrc = [gsb[0][off:off + sm.blob_sizes()[0]]]  # the slab's blocks of the global blob
        db = dm.alloc()
        db[0].fill_(0x5A)
        llama.copy(sm, lsrc, dm, db)
        torch.cuda.synchronize()
        got = db[0].cpu().numpy()
        want = np.concatenate([exp[starts[k] + first * s:starts[k] + (first + nl) * s] for k, s in enumerate(sizes)])
        assert np.array_equal(got, want), (world, rank)
    assert covered == n


# -------------------------------------------------------------------- C5
def test_c5_size_full_coverage(llama, oracle_mod):
    """The cross-device copy's kernel at C5's per-GPU size (2^27 Particle7,
    packed AoS -> SoA MB), every destination byte."""
    n = W.C5["extents"][0]
    schema = W.PARTICLE7
    sm = llama.Mapping(schema, [n], "aos")
    dm = llama.Mapping(schema, [n], "soa_mb")
    sb = sm.alloc()
    llama.generate(sm, sb, 43)
    db = dm.alloc()
    for t in db:
        t.fill_(0x5A)
    llama.copy(sm, sb, dm, db)
    torch.cuda.synchronize()
    so = oracle_mod.Mapping(schema, [n], "aos")
    do = oracle_mod.Mapping(schema, [n], "soa_mb")
    threads = _threads(256 << 20)
    src = so.alloc()
    _par_generate(oracle_mod, so, src, 43, n, threads)
    assert np.array_equal(sb[0].cpu().numpy(), src[0])
    exp = oracle_mod.copy(so, src, do, nthreads=threads)
    for j, t in enumerate(db):
        assert np.array_equal(t.cpu().numpy(), exp[j]), j


# -------------------------------------------------------------------- f4
F4 = [(("soa_mb", 1, False), "col", ("soa_mb", 1, False), "row"),
      (("aos", 1, False), "row", ("soa_mb", 1, False), "col"),
      (("soa_mb", 1, False), "morton", ("aos", 1, False), "col"),
      (("aos", 1, False), "row", ("aos", 1, False), "col"),
      (("aos", 1, False), "row", ("aos", 1, False), "morton"),
      (("soa_mb", 1, False), "row", ("aos", 1, False), "col")]


@pytest.mark.parametrize("case", range(len(F4)))
def test_f4_transposes_full_size(llama, oracle_mod, case):
    """The measured transposing copies (DESIGN.md §8 f4 table) at 4096 x 4096
    Particle7: whole blobs against the oracle's copy through its own
    linearisations."""
    sspec, slin, dspec, dlin = F4[case]
    ext = [4096, 4096]
    n = ext[0] * ext[1]
    sm = llama.Mapping.from_spec(W.PARTICLE7, ext, sspec, lin=slin)
    dm = llama.Mapping.from_spec(W.PARTICLE7, ext, dspec, lin=dlin)
    assert llama.plan(sm, dm)["path"] == "transpose"
    sb = sm.alloc()
    llama.generate(sm, sb, 11)
    db = dm.alloc()
    for t in db:
        t.fill_(0x5A)
    llama.copy(sm, sb, dm, db)
    torch.cuda.synchronize()
    so = oracle_mod.mapping_from_spec(W.PARTICLE7, ext, sspec, lin=slin)
    do = oracle_mod.mapping_from_spec(W.PARTICLE7, ext, dspec, lin=dlin)
    threads = _threads(64 << 20)
    src = so.alloc()
    _par_generate(oracle_mod, so, src, 11, n, threads)
    for j, t in enumerate(sb):
        assert np.array_equal(t.cpu().numpy(), src[j]), ("src", j)
    exp = oracle_mod.copy(so, src, do, nthreads=threads)
    for j, t in enumerate(db):
        assert np.array_equal(t.cpu().numpy(), exp[j]), ("dst", j)


F4_HEP = [("aos", "row", "soa_mb", "col"), ("soa_mb", "col", "aos", "row"), ("aos", "row", "aos_aligned", "col"),
          ("aos", "col", "aos", "morton"), ("soa_sb", "row", "soa_mb", "col")]


@pytest.mark.parametrize("case", range(len(F4_HEP)))
def test_f4_hep100_transposes_bench_size(llama, oracle_mod, case):
    """The bench's F4_hep pairs (bench.pairs_of("F4_hep")) at its 2048 x 2048
    HEP100 size and launch configuration (default plans: the wide kernel and
    the JIT's short tiles): whole blobs against the oracle, source padding
    poisoned."""
    import bench
    assert [(a + "/" + sl, b + "/" + dl) for a, sl, b, dl in F4_HEP] == bench.pairs_of("F4_hep")
    a, slin, b, dlin = F4_HEP[case]
    sspec, dspec = W.resolve_spec(a), W.resolve_spec(b)
    ext = list(bench.SUBCFG["F4_hep"]["extents"])
    n = ext[0] * ext[1]
    sm = llama.Mapping.from_spec(W.HEP100, ext, sspec, lin=slin)
    dm = llama.Mapping.from_spec(W.HEP100, ext, dspec, lin=dlin)
    assert llama.plan(sm, dm)["path"] == "transpose"
    sb = sm.alloc()
    llama.generate(sm, sb, 13, pad_byte=0xCD)
    db = dm.alloc()
    for t in db:
        t.fill_(0x5A)
    llama.copy(sm, sb, dm, db)
    torch.cuda.synchronize()
    so = oracle_mod.mapping_from_spec(W.HEP100, ext, sspec, lin=slin)
    do = oracle_mod.mapping_from_spec(W.HEP100, ext, dspec, lin=dlin)
    threads = _threads(64 << 20)
    src = so.alloc()
    _par_generate(oracle_mod, so, src, 13, n, threads, pad=0xCD)
    for j, t in enumerate(sb):
        assert np.array_equal(t.cpu().numpy(), src[j]), ("src", j)
    exp = oracle_mod.copy(so, src, do, nthreads=threads)
    for j, t in enumerate(db):
        assert np.array_equal(t.cpu().numpy(), exp[j]), ("dst", j)
