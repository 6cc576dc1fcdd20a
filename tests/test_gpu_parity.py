"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, byte
for byte (the copy is integer/byte work: bit-exact is the bar).

Each case generates the source on the GPU (llama_generate) and on the CPU
(oracle.generate), checks the two sources are identical, copies on
the GPU into destination blobs pre-filled with garbage (so an unwritten byte
cannot pass), and compares every byte of every destination blob with the
oracle's copy.  Source padding is poisoned with 0xCD (reading #13)."""
import os
import random

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


KINDS = {
    "aos": ("aos", 1, False), "aos_aligned": ("aos", 1, True), "soa_sb": ("soa_sb", 1, False),
    "soa_sb_aligned": ("soa_sb", 1, True), "soa_mb": ("soa_mb", 1, False), "aosoa4": ("aosoa", 4, False),
    "aosoa8": ("aosoa", 8, False), "aosoa32": ("aosoa", 32, False), "aosoa3": ("aosoa", 3, False),
    "aosoa8_aligned": ("aosoa", 8, True), "aosoa64": ("aosoa", 64, False),
}


def _host(t):
    return t.cpu().numpy()


def run_case(llama, oracle, schema, ext, sk, dk, seed=42, paths=("auto",), pad=0xCD, check_src=True, knobs=None):
    sm = llama.Mapping(schema, ext, *sk)
    dm = llama.Mapping(schema, ext, *dk)
    so = oracle.Mapping(schema, ext, *sk)
    do = oracle.Mapping(schema, ext, *dk)
    sb = sm.alloc("cuda")
    llama.generate(sm, sb, seed, pad_byte=pad)
    src_host = oracle.make_view(so, seed, pad_fill=pad)
    if check_src:
        for j, t in enumerate(sb):
            assert np.array_equal(_host(t), src_host[j]), f"generated source differs in blob {j}"
    exp = oracle.copy(so, src_host, do)
    for path in paths:
        if path != "auto":
            try:
                llama.plan(sm, dm, path=path, knobs=knobs)
            except llama.LlamaError:
                continue  # path not applicable to this pair
        db = dm.alloc("cuda")
        for t in db:
            t.fill_(0x5A)
        llama.copy(sm, sb, dm, db, path=path, knobs=knobs)
        torch.cuda.synchronize()
        for j, t in enumerate(db):
            got = _host(t)
            if not np.array_equal(got, exp[j]):
                bad = np.nonzero(got != exp[j])[0]
                raise AssertionError(f"{sk}->{dk} ext={ext} path={path} plan={llama.plan(sm, dm, path=path, knobs=knobs)}: "
                                     f"blob {j}: {bad.size} bytes differ, first at {bad[:8]}")


ALL_PATHS = ("auto", "naive", "permute", "run", "blobcopy")


@pytest.mark.parametrize("n", [1, 7, 31, 32, 33, 100, 4095, 4097, 65537])
@pytest.mark.parametrize("schema_name", ["particle7", "listing1"])
def test_all_pairs_small(llama, oracle_mod, schema_name, n):
    schema = W.SCHEMAS[schema_name]
    for a in KINDS:
        for b in KINDS:
            run_case(llama, oracle_mod, schema, [n], KINDS[a], KINDS[b], seed=42 + n, paths=ALL_PATHS)


@pytest.mark.parametrize("n", [1, 33, 1000, 4097])
def test_all_pairs_hep100(llama, oracle_mod, n):
    kinds = ["aos", "aos_aligned", "soa_mb", "soa_sb", "aosoa8", "aosoa32", "aosoa3"]
    for a in kinds:
        for b in kinds:
            run_case(llama, oracle_mod, W.HEP100, [n], KINDS[a], KINDS[b], seed=1, paths=ALL_PATHS)


@pytest.mark.parametrize("ext", [[4, 3], [64, 33], [7, 5, 9], [128, 256]])
def test_multidim_extents(llama, oracle_mod, ext):
    for schema in (W.LISTING1, W.VEC, W.OUTER):
        for a, b in [("aos", "soa_mb"), ("aosoa32", "soa_sb"), ("soa_sb", "aos_aligned"), ("aosoa8", "aosoa4")]:
            run_case(llama, oracle_mod, schema, ext, KINDS[a], KINDS[b], seed=2, paths=ALL_PATHS)


def _random_schema(rng):
    types = ["i8", "u8", "bool", "i16", "u16", "i32", "u32", "f32", "i64", "u64", "f64"]
    fields = []
    for j in range(rng.randint(1, 24)):
        t = rng.choice(types)
        if rng.random() < 0.15:
            t += f"[{rng.randint(1, 4)}]"
        fields.append(f"f{j}:{t}")
    if rng.random() < 0.3:
        fields.append("n{" + ",".join(f"g{j}:{rng.choice(types)}" for j in range(rng.randint(1, 4))) + "}")
    return "R{" + ",".join(fields) + "}"


@pytest.mark.parametrize("seed", range(12))
def test_random_schema_fuzz(llama, oracle_mod, seed):
    rng = random.Random(seed)
    schema = _random_schema(rng)
    n = rng.choice([1, 5, 17, 64, 333, 1024, 5000])
    names = list(KINDS)
    for _ in range(12):
        a, b = rng.choice(names), rng.choice(names)
        run_case(llama, oracle_mod, schema, [n], KINDS[a], KINDS[b], seed=seed, paths=ALL_PATHS)


def test_tile_sizes_and_empty(llama, oracle_mod):
    for t in (32, 64, 96, 256, 1024):
        for a, b in [("aos", "soa_mb"), ("aos_aligned", "aos"), ("soa_sb", "aosoa32")]:
            sm = llama.Mapping(W.LISTING1, [3000], *KINDS[a])
            dm = llama.Mapping(W.LISTING1, [3000], *KINDS[b])
            try:
                llama.plan(sm, dm, path="permute", tile_records=t)
            except llama.LlamaError:
                continue
            so = oracle_mod.Mapping(W.LISTING1, [3000], *KINDS[a])
            do = oracle_mod.Mapping(W.LISTING1, [3000], *KINDS[b])
            sb = sm.alloc()
            llama.generate(sm, sb, 3, pad_byte=0xCD)
            db = dm.alloc()
            for x in db:
                x.fill_(0x5A)
            llama.copy(sm, sb, dm, db, path="permute", tile_records=t)
            exp = oracle_mod.copy(so, oracle_mod.make_view(so, 3, 0xCD), do)
            for j, x in enumerate(db):
                assert np.array_equal(_host(x), exp[j]), (t, a, b)
    e = llama.Mapping(W.LISTING1, [0], "aos")
    llama.copy(e, e.alloc(), llama.Mapping(W.LISTING1, [0], "soa_mb"),
               llama.Mapping(W.LISTING1, [0], "soa_mb").alloc())


def test_streams_and_launch_count(llama, oracle_mod):
    sm = llama.Mapping(W.PARTICLE7, [100000], "aos")
    dm = llama.Mapping(W.PARTICLE7, [100000], "soa_mb")
    sb, db = sm.alloc(), dm.alloc()
    s = torch.cuda.Stream()
    before = llama.launch_count()
    with torch.cuda.stream(s):
        llama.generate(sm, sb, 42)
        llama.copy(sm, sb, dm, db)
    s.synchronize()
    assert llama.launch_count() - before >= 2
    exp = oracle_mod.copy(oracle_mod.Mapping(W.PARTICLE7, [100000], "aos"),
                          oracle_mod.make_view(oracle_mod.Mapping(W.PARTICLE7, [100000], "aos"), 42),
                          oracle_mod.Mapping(W.PARTICLE7, [100000], "soa_mb"))
    for j, x in enumerate(db):
        assert np.array_equal(_host(x), exp[j])


# ------------------------------------------------------- full BASELINE sizes
def test_c1_parity(llama, oracle_mod):
    cfg = W.C1
    for a, b in cfg["pairs"]:
        run_case(llama, oracle_mod, W.SCHEMAS[cfg["schema"]], list(cfg["extents"]), W.MAPPINGS[a],
                 W.MAPPINGS[b], seed=42, paths=("auto", "naive"))


def test_c2_full_size_all_pairs(llama, oracle_mod):
    """C2 at its full size (16M particles), all 16 ordered pairs, in the
    launch configuration bench.py times (AUTO plan), every byte compared."""
    cfg = W.C2
    schema, ext = W.SCHEMAS[cfg["schema"]], list(cfg["extents"])
    views = {}
    for name in ("aos", "soa_mb", "aosoa8", "aosoa32"):
        om = oracle_mod.Mapping(schema, ext, *W.MAPPINGS[name])
        views[name] = oracle_mod.make_view(om, 42)
    for a, b in cfg["pairs"]:
        sm = llama.Mapping(schema, ext, *W.MAPPINGS[a])
        dm = llama.Mapping(schema, ext, *W.MAPPINGS[b])
        sb = sm.alloc()
        llama.generate(sm, sb, 42)
        db = dm.alloc()
        for x in db:
            x.fill_(0x5A)
        llama.copy(sm, sb, dm, db)
        torch.cuda.synchronize()
        for j, x in enumerate(db):
            assert np.array_equal(_host(x), views[b][j]), (a, b, j)
        del sb, db


def test_c4_full_size(llama, oracle_mod):
    """C4: Listing-1 record, 8192 x 8192, AoSoA32 -> SoA SB, whole blob compared."""
    cfg = W.C4
    for a, b in cfg["pairs"]:
        run_case(llama, oracle_mod, W.SCHEMAS[cfg["schema"]], list(cfg["extents"]), W.MAPPINGS[a],
                 W.MAPPINGS[b], seed=42, paths=("auto",))


# ------------------------------------------------ staged host <-> device copy
@pytest.mark.parametrize("cap", [4096, 1 << 16, 0])
def test_staged_copy_host_buffers(llama, oracle_mod, cap):
    """llama_copy_staged with pinned host source and destination:
    slabs DMA'd in, relayouted on the device, DMA'd out; every destination byte
    compared with the oracle, including small staging buffers (many slabs, a
    partial last slab) and aligned SoA single-blob gaps."""
    st = llama.Stager(cap)
    cases = [(W.PARTICLE7, 5000, "aos", "soa_mb"), (W.PARTICLE7, 4097, "aosoa8", "aosoa32"),
             (W.LISTING1, 3001, "aosoa32", "soa_sb"), (W.LISTING1, 777, "soa_sb", "aos_aligned"),
             (W.LISTING1, 999, "aos", "soa_sb_aligned"), (W.HEP100, 333, "aos", "aos_aligned"),
             (W.HEP100, 200, "soa_mb", "aosoa3")]
    for schema, n, a, b in cases:
        sm, dm = llama.Mapping(schema, [n], *KINDS[a]), llama.Mapping(schema, [n], *KINDS[b])
        so, do = oracle_mod.Mapping(schema, [n], *KINDS[a]), oracle_mod.Mapping(schema, [n], *KINDS[b])
        src_host = oracle_mod.make_view(so, 7, pad_fill=0xCD)
        hs = [torch.from_numpy(x).pin_memory() for x in src_host]
        hd = [torch.full((x,), 0x5A, dtype=torch.uint8).pin_memory() for x in dm.blob_sizes()]
        llama.copy_staged(st, sm, hs, dm, hd)
        torch.cuda.synchronize()
        exp = oracle_mod.copy(so, src_host, do)
        for j, x in enumerate(hd):
            assert np.array_equal(x.numpy(), exp[j]), (schema[:10], n, a, b, j, cap)
        # device -> host and host -> device mixes
        ds = sm.alloc()
        for t, h in zip(ds, hs):
            t.copy_(h)
        hd2 = [torch.full((x,), 0x33, dtype=torch.uint8).pin_memory() for x in dm.blob_sizes()]
        llama.copy_staged(st, sm, ds, dm, hd2)
        torch.cuda.synchronize()
        for j, x in enumerate(hd2):
            assert np.array_equal(x.numpy(), exp[j])


@pytest.mark.parametrize("cap", [4096, 1 << 16, 0])
def test_staged_copy_batch(llama, oracle_mod, cap):
    """llama_copy_staged_batch: the same cases as one pipeline (the buffers
    rotate from one copy into the next), every destination byte checked."""
    st = llama.Stager(cap)
    cases = [(W.PARTICLE7, 5000, "aos", "soa_mb"), (W.LISTING1, 3001, "aosoa32", "soa_sb"),
             (W.LISTING1, 999, "aos", "soa_sb_aligned"), (W.HEP100, 333, "aos", "aos_aligned"),
             (W.PARTICLE7, 0, "aos", "soa_mb"), (W.PARTICLE7, 4097, "aosoa8", "aosoa32")]
    batch, expect = [], []
    for schema, n, a, b in cases:
        sm, dm = llama.Mapping(schema, [n], *KINDS[a]), llama.Mapping(schema, [n], *KINDS[b])
        so, do = oracle_mod.Mapping(schema, [n], *KINDS[a]), oracle_mod.Mapping(schema, [n], *KINDS[b])
        src_host = oracle_mod.make_view(so, 9, pad_fill=0xCD)
        hs = [torch.from_numpy(x).pin_memory() for x in src_host]
        hd = [torch.full((max(x, 1),), 0x5A, dtype=torch.uint8).pin_memory() for x in dm.blob_sizes()]
        batch.append((sm, hs, dm, hd))
        expect.append(oracle_mod.copy(so, src_host, do))
    llama.copy_staged_batch(st, batch)
    torch.cuda.synchronize()
    for (sm, hs, dm, hd), exp, case in zip(batch, expect, cases):
        for j, x in enumerate(hd):
            assert np.array_equal(x.numpy()[:dm.blob_sizes()[j]], exp[j][:dm.blob_sizes()[j]]), (case, j, cap)


# ------------------------------------------------------------ One / Split (f1)
def run_spec_case(llama, oracle, schema, ext, s_spec, d_spec, seed=7, pad=0xCD, knobs=None, paths=None):
    """run_case for workloads spec trees (MAPPINGS tuples or split trees)."""
    sm = llama.Mapping.from_spec(schema, ext, s_spec)
    dm = llama.Mapping.from_spec(schema, ext, d_spec)
    so = oracle.mapping_from_spec(schema, ext, s_spec)
    do = oracle.mapping_from_spec(schema, ext, d_spec)
    sb = sm.alloc("cuda")
    llama.generate(sm, sb, seed, pad_byte=pad)
    src_host = oracle.make_view(so, seed, pad_fill=pad)
    for j, t in enumerate(sb):
        assert np.array_equal(_host(t), src_host[j]), f"generated source differs in blob {j}"
    exp = oracle.copy(so, src_host, do)
    for path in (paths or ALL_PATHS):
        if path != "auto":
            try:
                llama.plan(sm, dm, path=path, knobs=knobs)
            except llama.LlamaError:
                continue
        db = dm.alloc("cuda")
        for t in db:
            t.fill_(0x5A)
        llama.copy(sm, sb, dm, db, path=path, knobs=knobs)
        torch.cuda.synchronize()
        for j, t in enumerate(db):
            got = _host(t)
            assert np.array_equal(got, exp[j]), (f"{sm!r}->{dm!r} ext={ext} path={path}: blob {j}: "
                                                 f"{int((got != exp[j]).sum())} bytes differ")


_SPLIT_SETS = {
    "particle7": ["aos", "soa_mb", "aosoa8", "split_p7"],
    "listing1": ["aos", "aos_aligned", "soa_sb", "split_pos"],
    "hep100": ["aos", "soa_mb", "split_hep"],
}


@pytest.mark.parametrize("n", [1, 33, 4097, 100_003])
@pytest.mark.parametrize("schema_name", sorted(_SPLIT_SETS))
def test_split_pairs(llama, oracle_mod, schema_name, n):
    names = _SPLIT_SETS[schema_name]
    if schema_name == "hep100" and n > 5000:
        n = 5000
    schema = W.SCHEMAS[schema_name]
    for a in names:
        for b in names:
            if "split" in a or "split" in b:
                run_spec_case(llama, oracle_mod, schema, [n], W.resolve_spec(a), W.resolve_spec(b))


@pytest.mark.parametrize("n", [1, 9, 1000])
def test_one_and_mapping_c_sources(llama, oracle_mod, n):
    """One / MappingC (Listing P:499-509) as sources broadcast their One
    record; as destinations only a single record is allowed (reading #24)."""
    for src in ("one", "mapping_c"):
        for dst in ("aos", "soa_mb", "split_pos"):
            run_spec_case(llama, oracle_mod, W.LISTING1, [n], W.resolve_spec(src), W.resolve_spec(dst))
    if n == 1:
        for dst in ("one", "mapping_c"):
            run_spec_case(llama, oracle_mod, W.LISTING1, [1], W.resolve_spec("aos"), W.resolve_spec(dst))
    else:
        sm = llama.Mapping(W.LISTING1, [n])
        with pytest.raises(llama.LlamaError, match="UNSUPPORTED"):
            llama.copy(sm, sm.alloc("cuda"), llama.Mapping(W.LISTING1, [n], "one"),
                       llama.Mapping(W.LISTING1, [n], "one").alloc("cuda"))


# ------------------------------------------------ direct AoS <-> SoA variant
@pytest.mark.parametrize("schema_name", ["listing1", "particle7", "hep100"])
@pytest.mark.parametrize("n", [1, 31, 64, 65, 1000, 4097])
@pytest.mark.parametrize("use_async", ["1", "0", "nostage", "nochunk"])
def test_direct_variant_forced(llama, oracle_mod, schema_name, n, use_async):
    """The direct permute (AoS side through TMA, SoA side element-wise) for
    every AoS <-> SoA pair, forced for few-leaf records too (knob direct=2):
    odd record strides exercise the byte-wise shared-memory accesses; SoA ->
    AoS with the cp.async classes (with and without the staged misaligned
    classes and the 16-byte chunk-staged 1- / 2-byte classes) and with
    registers only."""
    knobs = {"jit": 0, "direct": 2, "direct_async": 0 if use_async == "0" else 1,
             "direct_staging": 0 if use_async == "nostage" else 1,
             "direct_chunks": 0 if use_async == "nochunk" else 1}
    schema = W.SCHEMAS[schema_name]
    names = ["aos", "aos_aligned", "soa_mb", "soa_sb", "soa_sb_aligned"]
    for a in names:
        for b in names:
            if ("aos" in a) == ("aos" in b):
                continue
            sm = llama.Mapping(schema, [n], *KINDS[a])
            dm = llama.Mapping(schema, [n], *KINDS[b])
            assert llama.plan(sm, dm, knobs=knobs)["direct"], (a, b)
            run_case(llama, oracle_mod, schema, [n], KINDS[a], KINDS[b], knobs=knobs)


def test_direct_chosen_for_hep_without_jit(llama):
    m = {k: llama.Mapping(W.HEP100, [4096], *KINDS[k]) for k in ("aos", "aos_aligned", "soa_mb")}
    kn = {"jit": 0}
    assert llama.plan(m["aos_aligned"], m["soa_mb"], knobs=kn)["direct"]
    assert llama.plan(m["soa_mb"], m["aos_aligned"], knobs=kn)["direct"]
    assert llama.plan(m["aos"], m["soa_mb"], knobs=kn)["direct"]  # packed: funnel-shifted gathers
    assert llama.plan(m["soa_mb"], m["aos"], knobs=kn)["direct"]  # packed destination: staged misaligned classes
    assert not llama.plan(m["aos"], m["aos_aligned"], knobs=kn)["direct"]


def test_c5_symmetric_memory_path_one_rank(llama):
    """bench.py --config C5 (cross-device relayout through peer pointers from
    torch symmetric memory) under torchrun with one rank: the peer is this
    GPU.  Every leg (fused TMA stores, LSU stores, copy-engine and NCCL
    baselines) passes its round-trip check; the kernel's result at this size
    is compared with the oracle in test_gpu_full_coverage.py."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "bench.py"),
                        "--gpus", "1", "--config", "C5", "--steps", "2", "--warmup", "3"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["roundtrip_check"] is True
    assert set(line["legs"]) == {"fused", "fused_lsu", "staged_ce", "staged_nccl"}
    assert all(v["parity_roundtrip"] for v in line["legs"].values())
    assert line["value"] > 0 and line["nvlink_ceiling_gbs_per_gpu"] > 0


def _random_spec(rng, n_leaves, depth=0):
    """A random mapping spec over n_leaves leaves: a plain kind or a split."""
    kinds = [("aos", 1, False), ("aos", 1, True), ("soa_mb", 1, False), ("soa_sb", 1, False),
             ("soa_sb", 1, True), ("aosoa", rng.choice([2, 4, 8, 32]), False), ("aosoa", 8, True)]
    if n_leaves >= 2 and depth < 2 and rng.random() < 0.5:
        k = rng.randint(1, n_leaves - 1)
        leaves_a = sorted(rng.sample(range(n_leaves), k))
        return (leaves_a, _random_spec(rng, k, depth + 1), _random_spec(rng, n_leaves - k, depth + 1))
    return rng.choice(kinds)


@pytest.mark.parametrize("seed", range(40))
def test_random_split_lin_fuzz(llama, oracle_mod, seed):
    """Random schemas x random (nested) splits x random storage orders, every
    applicable path, against the oracle byte for byte."""
    rng = random.Random(1000 + seed)
    schema = _random_schema(rng)
    k = len(oracle_mod.leaf_sizes(schema))
    ext = rng.choice([[37], [64, 33], [32, 32], [5, 7, 3], [64, 64]])
    lins = ["row", "col"] + (["morton"] if len(set(ext)) == 1 and ext[0] & (ext[0] - 1) == 0 else [])
    for _ in range(6):
        sspec, dspec = _random_spec(rng, k), _random_spec(rng, k)
        slin = dlin = rng.choice(lins)
        if len(ext) == 2 and rng.random() < 0.5:
            dlin = rng.choice(lins)
        sm = llama.Mapping.from_spec(schema, ext, sspec, lin=slin)
        dm = llama.Mapping.from_spec(schema, ext, dspec, lin=dlin)
        so = oracle_mod.mapping_from_spec(schema, ext, sspec, lin=slin)
        do = oracle_mod.mapping_from_spec(schema, ext, dspec, lin=dlin)
        sb = sm.alloc("cuda")
        llama.generate(sm, sb, seed, pad_byte=0xCD)
        src = oracle_mod.make_view(so, seed, pad_fill=0xCD)
        for j, t in enumerate(sb):
            assert np.array_equal(_host(t), src[j]), ("generated", sspec, slin)
        exp = oracle_mod.copy(so, src, do)
        for path in ("auto", "naive", "permute", "run", "blobcopy", "transpose"):
            try:
                llama.plan(sm, dm, path=path)
            except llama.LlamaError:
                continue
            db = dm.alloc("cuda")
            for t in db:
                t.fill_(0x5A)
            llama.copy(sm, sb, dm, db, path=path)
            torch.cuda.synchronize()
            for j, t in enumerate(db):
                assert np.array_equal(_host(t), exp[j]), (schema, ext, sspec, slin, dspec, dlin, path, j)


def test_empty_views_every_feature(llama, oracle_mod):
    """Zero records through splits, One, storage orders, tracing, the move and
    the staged copy: nothing launched that could touch memory, no errors."""
    for spec in (W.resolve_spec("split_p7"), ("soa_mb", 1, False), ("aosoa", 8, False)):
        for ext in ([0], [0, 32], [32, 0]):
            sm = llama.Mapping.from_spec(W.PARTICLE7, ext, spec)
            dm = llama.Mapping.from_spec(W.PARTICLE7, ext, ("aos", 1, False))
            llama.copy(sm, sm.alloc("cuda"), dm, dm.alloc("cuda"))
            assert llama.nbody_move(sm, sm.alloc("cuda"), 0.1) in ("runs", "aos", "generic")
            if len(ext) == 2:
                llama.copy(sm.with_linearizer("col"), sm.alloc("cuda"), dm, dm.alloc("cuda"))
            t = sm.traced(fields=True, bytes=True)
            llama.copy(t, t.alloc("cuda"), dm, dm.alloc("cuda"))
            torch.cuda.synchronize()
            assert t.field_hits() == [0] * 7
    st = llama.Stager(1 << 16)
    a, b = llama.Mapping(W.PARTICLE7, [0]), llama.Mapping(W.PARTICLE7, [0], "soa_mb")
    llama.copy_staged(st, a, [torch.empty(16, dtype=torch.uint8).pin_memory()], b,
                      [torch.empty(16, dtype=torch.uint8).pin_memory() for _ in range(7)])
    llama.nbody_move_staged(st, b, [torch.empty(16, dtype=torch.uint8).pin_memory() for _ in range(7)], 0.1)
    torch.cuda.synchronize()
