"""GPU parity of the wide-record transposing copy (k_transpose_wide.cu; SURVEY
§8(f) f4: rank-2 views of different storage orders, reading #26)
against the oracle: every byte of every destination blob, destinations
pre-filled with 0x5A, source padding poisoned with 0xCD."""
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


def _check(llama, oracle, schema, ext, a, slin, b, dlin, knobs=None, expect_wide=True, seed=5):
    sspec, dspec = W.resolve_spec(a), W.resolve_spec(b)
    sm = llama.Mapping.from_spec(schema, ext, sspec, lin=slin)
    dm = llama.Mapping.from_spec(schema, ext, dspec, lin=dlin)
    if expect_wide:  # the wide kernel, or the JIT transpose's 4- / 8-row tiles (AoS images of different layouts)
        pl = llama.plan(sm, dm, knobs=knobs)
        assert pl["wide"] or (pl["jit"] and pl["path"] == "transpose"), (a, slin, b, dlin)
    so = oracle.mapping_from_spec(schema, ext, sspec, lin=slin)
    do = oracle.mapping_from_spec(schema, ext, dspec, lin=dlin)
    sb = sm.alloc("cuda")
    llama.generate(sm, sb, seed, pad_byte=0xCD)
    src = oracle.make_view(so, seed, pad_fill=0xCD)
    exp = oracle.copy(so, src, do, nthreads=8)
    db = dm.alloc("cuda")
    for t in db:
        t.fill_(0x5A)
    llama.copy(sm, sb, dm, db, knobs=knobs)
    torch.cuda.synchronize()
    for j, t in enumerate(db):
        got = t.cpu().numpy()
        if not np.array_equal(got, exp[j]):
            bad = np.nonzero(got != exp[j])[0]
            raise AssertionError(f"{a}/{slin} -> {b}/{dlin} {ext}: blob {j}: {bad.size} bytes differ, first at {bad[0]}")


HEP_KINDS = ["aos", "aos_aligned", "soa_mb", "soa_sb", "aosoa8", "soa_sb_aligned", "split_hep"]
LINS = [("row", "col"), ("col", "row"), ("row", "morton"), ("morton", "col"), ("col", "morton")]


@pytest.mark.parametrize("lins", LINS)
@pytest.mark.parametrize("ext", [[64, 64], [32, 32]])
def test_hep100_every_kind_pair(llama, oracle_mod, lins, ext):
    """HEP100 (380 / 480-byte records) over every ordered kind pair; Morton
    extents equal powers of two."""
    for a in HEP_KINDS:
        for b in HEP_KINDS:
            if b == "split_hep" or a == "split_hep":
                _check(llama, oracle_mod, W.HEP100, ext, a, lins[0], b, lins[1], expect_wide=False)
            else:
                _check(llama, oracle_mod, W.HEP100, ext, a, lins[0], b, lins[1])


@pytest.mark.parametrize("ext", [[37, 70], [1, 300], [300, 1], [33, 129], [1, 1], [5, 3]])
@pytest.mark.parametrize("lins", [("row", "col"), ("col", "row")])
def test_hep100_ragged(llama, oracle_mod, ext, lins):
    """Partial tiles on every edge (row / column extents not multiples of the tile)."""
    for a, b in [("aos", "soa_mb"), ("soa_mb", "aos_aligned"), ("aos", "aos_aligned"), ("aos", "aos"),
                 ("aos_aligned", "aos"), ("soa_sb", "soa_mb"), ("aosoa8", "aos"), ("aos", "aosoa8"),
                 ("soa_mb", "soa_sb_aligned")]:
        _check(llama, oracle_mod, W.HEP100, ext, a, lins[0], b, lins[1])


@pytest.mark.parametrize("ext", [[8, 8], [4, 4], [2, 2], [16, 16]])
def test_hep100_small_morton(llama, oracle_mod, ext):
    """Morton views smaller than the tile: the tile is clipped and stays square
    or 1 x 2 (E -> E needs 32 x 32 and falls back to the naive kernel)."""
    for a, b in [("aos", "soa_mb"), ("soa_mb", "aos"), ("aos", "aos_aligned"), ("soa_mb", "soa_sb")]:
        for lins in [("row", "morton"), ("morton", "col")]:
            _check(llama, oracle_mod, W.HEP100, ext, a, lins[0], b, lins[1],
                   expect_wide=not (a.startswith("soa") and b.startswith("soa")))


def test_hep100_aosoa_odd_lanes(llama, oracle_mod):
    """AoSoA with a lane count that is not a power of two (division in the
    block split, reading #8) on either side."""
    sm = ("aosoa", 3, False)
    for sl, dl in [("row", "col"), ("col", "morton")]:
        for a, b in [(sm, "aos"), ("aos_aligned", sm), (sm, "soa_mb"), ("soa_sb", sm)]:
            _check(llama, oracle_mod, W.HEP100, [32, 32], a, sl, b, dl)


@pytest.mark.parametrize("schema", [W.PARTICLE7, W.LISTING1])
def test_small_records_forced(llama, oracle_mod, schema):
    """Knob wide=2: records the JIT transpose handles, forced onto the wide
    kernel (Listing-1 packed, 21 B, is an element-wise side; aligned 32 B an
    image side)."""
    kn = {"wide": 2}
    for a in ["aos", "aos_aligned", "soa_mb", "aosoa8"]:
        for b in ["aos", "aos_aligned", "soa_sb"]:
            for sl, dl in [("row", "col"), ("morton", "row")]:
                _check(llama, oracle_mod, schema, [64, 64], a, sl, b, dl, knobs=kn)


def test_hep100_full_size(llama, oracle_mod):
    """1024 x 1024 HEP100 (the pair-matrix size), whole blobs."""
    for a, sl, b, dl in [("aos", "row", "soa_mb", "col"), ("soa_mb", "col", "aos_aligned", "row"),
                         ("aos", "row", "aos_aligned", "morton"), ("soa_sb", "morton", "soa_mb", "row")]:
        _check(llama, oracle_mod, W.HEP100, [1024, 1024], a, sl, b, dl)


@pytest.mark.parametrize("ext", [[64, 64], [8, 96], [1024, 1024]])
def test_hep100_jit_short_tiles(llama, oracle_mod, ext):
    """Packed <-> aligned AoS transposes of 380 / 480-byte records, and AoS into
    row-major SoA (incl. the aligned single blob's zeroed gaps), through the
    JIT transpose with 8- / 4-row tiles (per-record programs)."""
    for a, sl, b, dl in [("aos", "row", "aos_aligned", "col"), ("aos_aligned", "col", "aos", "row"),
                         ("aos", "col", "aos_aligned", "row"), ("aos_aligned", "row", "aos", "col"),
                         ("aos", "col", "soa_mb", "row"), ("aos_aligned", "col", "soa_sb", "row"),
                         ("aos", "col", "soa_sb_aligned", "row"), ("aos_aligned", "col", "soa_mb", "row")]:
        sm = llama.Mapping.from_spec(W.HEP100, ext, W.resolve_spec(a), lin=sl)
        dm = llama.Mapping.from_spec(W.HEP100, ext, W.resolve_spec(b), lin=dl)
        pl = llama.plan(sm, dm)
        assert pl["jit"] and pl["tile_records"] in (128, 256), pl
        _check(llama, oracle_mod, W.HEP100, ext, a, sl, b, dl)


def test_hep100_staged_knob(llama, oracle_mod):
    """Knob wide_stage=1 (measured slower, off by default): element-wise -> AoS
    through a cp.async staging area."""
    kn = {"wide_stage": 1}
    for a, sl, b, dl in [("soa_mb", "col", "aos", "row"), ("soa_sb", "morton", "aos_aligned", "row"),
                         ("aosoa8", "row", "aos", "col")]:
        for ext in ([64, 64], [36, 68]):
            if "morton" in (sl, dl) and ext[0] != ext[1]:
                continue
            _check(llama, oracle_mod, W.HEP100, ext, a, sl, b, dl, knobs=kn)


def _wide_schema(rng):
    """A random record of 40-110 leaves (1- to 8-byte, arrays, nesting): too
    wide for the JIT transpose's 16 x 32 tiles."""
    types = ["i8", "u8", "bool", "i16", "u16", "i32", "u32", "f32", "i64", "u64", "f64"]
    fields = []
    while len(fields) < rng.randint(40, 100):
        t = rng.choice(types)
        if rng.random() < 0.1:
            t += f"[{rng.randint(2, 4)}]"
        fields.append(f"f{len(fields)}:{t}")
    fields.append("n{" + ",".join(f"g{j}:{rng.choice(types)}" for j in range(rng.randint(1, 6))) + "}")
    return "R{" + ",".join(fields) + "}"


@pytest.mark.parametrize("seed", range(16))
def test_wide_transpose_fuzz(llama, oracle_mod, seed):
    """Random wide schemas x kinds (packed / aligned AoS, SoA SB / MB, aligned
    SB, AoSoA with 3 / 4 / 8 / 16 lanes) x storage orders x ragged extents,
    random wide-kernel knobs; the default plan (wide kernel, JIT short tiles
    or naive) against the oracle byte for byte."""
    import random
    rng = random.Random(9000 + seed)
    schema = _wide_schema(rng)
    kinds = [("aos", 1, False), ("aos", 1, True), ("soa_mb", 1, False), ("soa_sb", 1, False), ("soa_sb", 1, True),
             ("aosoa", 3, False), ("aosoa", 4, True), ("aosoa", 8, False), ("aosoa", 16, False)]
    for _ in range(4):
        ext = rng.choice([[32, 32], [64, 64], [16, 16], [40, 72], [33, 65], [128, 8], [8, 128], [64, 36]])
        lins = ["row", "col"] + (["morton"] if ext[0] == ext[1] else [])
        slin = rng.choice(lins)
        dlin = rng.choice([x for x in lins if x != slin])
        knobs = {}
        for name, choices in (("wide_group", [0, 1]), ("wide_torder", [0, 1, 2]), ("wide_stage", [0, 1]),
                              ("wide_chunk4", [0, 1]), ("wide", [1, 2]), ("wide_tma", [0, 1]), ("wide_async", [0, 1])):
            if rng.random() < 0.4:
                knobs[name] = rng.choice(choices)
        _check(llama, oracle_mod, schema, ext, rng.choice(kinds), slin, rng.choice(kinds), dlin, knobs=knobs or None,
               expect_wide=False, seed=seed)


@pytest.mark.parametrize("knobs", [{"wide_tma": 0}, {"wide_async": 1}, {"wide_chunk4": 1}, {"wide_torder": 1}])
def test_hep100_knob_variants(llama, oracle_mod, knobs):
    """Every wide-kernel variant a knob selects, on ragged and full tiles, each
    mode: byte-exact like the defaults."""
    for ext in ([64, 64], [37, 68]):
        for a, sl, b, dl in [("aos", "row", "soa_mb", "col"), ("soa_mb", "col", "aos_aligned", "row"),
                             ("soa_sb", "row", "aos", "col"), ("aos", "col", "aos", "row"),
                             ("aos_aligned", "row", "aos_aligned", "col"), ("soa_mb", "row", "soa_sb", "col")]:
            _check(llama, oracle_mod, W.HEP100, ext, a, sl, b, dl, knobs=knobs)


@pytest.mark.parametrize("ext", [[64, 64], [37, 64], [64, 40], [16, 16]])
def test_hep100_aosoa_images(llama, oracle_mod, ext):
    """AoSoA-L sides staged as images when the tile's runs hold whole blocks
    (L = 4 / 8 / 16, aligned AoSoA with padding inside the blocks), on full and
    ragged tiles; knob wide_aosoa_img=0 keeps them element-wise."""
    kinds = [("aosoa", 8, False), ("aosoa", 4, True), ("aosoa", 16, False)]
    others = ["aos", "aos_aligned", "soa_mb"]
    lins = [("row", "col"), ("col", "row")] + ([("row", "morton"), ("morton", "col")] if ext[0] == ext[1] else [])
    for sl, dl in lins:  # (small Morton views between element-wise sides take the naive kernel)
        for k in kinds:
            for o in others:
                _check(llama, oracle_mod, W.HEP100, ext, k, sl, o, dl, expect_wide=False)
                _check(llama, oracle_mod, W.HEP100, ext, o, sl, k, dl, expect_wide=False)
                _check(llama, oracle_mod, W.HEP100, ext, o, sl, k, dl, knobs={"wide_aosoa_img": 2}, expect_wide=False)
            _check(llama, oracle_mod, W.HEP100, ext, k, sl, kinds[0], dl, expect_wide=False)
    _check(llama, oracle_mod, W.HEP100, ext, kinds[0], "row", "aos", "col", knobs={"wide_aosoa_img": 0},
           expect_wide=False)


@pytest.mark.parametrize("seed", range(16))
def test_wide_forced_small_fuzz(llama, oracle_mod, seed):
    """Random small / medium schemas (1-24 fields, odd record sizes) forced onto
    the wide kernel (knob wide=2) x kinds incl. AoSoA-L image sides x storage
    orders x extents: byte-exact against the oracle (the odd per-record
    strides exercise the image chunk / alignment rules)."""
    import random

    from test_gpu_parity import _random_schema
    rng = random.Random(7000 + seed)
    schema = _random_schema(rng)
    kinds = [("aos", 1, False), ("aos", 1, True), ("soa_mb", 1, False), ("soa_sb", 1, False),
             ("aosoa", 4, False), ("aosoa", 8, True), ("aosoa", 16, False), ("aosoa", 32, False)]
    for _ in range(4):
        ext = rng.choice([[32, 32], [64, 64], [48, 32], [32, 48], [36, 64], [64, 40]])
        lins = ["row", "col"] + (["morton"] if ext[0] == ext[1] else [])
        slin = rng.choice(lins)
        dlin = rng.choice([x for x in lins if x != slin])
        _check(llama, oracle_mod, schema, ext, rng.choice(kinds), slin, rng.choice(kinds), dlin, knobs={"wide": 2},
               expect_wide=False, seed=seed)
