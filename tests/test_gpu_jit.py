"""GPU parity of the plan-time specialised permute (k_jit_permute: a move
program generated per mapping pair and compiled with NVRTC), byte
for byte against the oracle: every ordered pair of the HEP100 kinds (the
paper's 100-leaf event records), ragged extents (full tiles, a partial
last tile, fewer records than a tile, AoSoA tail lanes), small records forced
onto it (knob jit=2), splits, every tile size and stage count."""
import numpy as np
import pytest

import workloads as W
from test_gpu_parity import KINDS, run_case, run_spec_case

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def llama():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_04284_b200 as m
    return m


HEP_KINDS = ["aos", "aos_aligned", "soa_mb", "soa_sb", "aosoa8", "aosoa32", "aosoa8_aligned"]


@pytest.mark.parametrize("n", [1, 31, 64, 65, 1000, 4097, 100_003])
def test_hep100_pairs_jit(llama, oracle_mod, n):
    for a in HEP_KINDS:
        for b in HEP_KINDS:
            if a == b:
                continue
            sm = llama.Mapping(W.HEP100, [n], *KINDS[a])
            dm = llama.Mapping(W.HEP100, [n], *KINDS[b])
            pl = llama.plan(sm, dm, path="permute", knobs={"jit": 2})
            if "soa_sb" not in (a, b):  # SB sub-arrays of N * s_k bytes start 16-byte aligned only for some N
                assert pl["jit"], (a, b, pl)
            run_case(llama, oracle_mod, W.HEP100, [n], KINDS[a], KINDS[b], seed=3 + n, paths=("permute",),
                     knobs={"jit": 2})


@pytest.mark.parametrize("schema_name", ["particle7", "listing1"])
@pytest.mark.parametrize("n", [1, 33, 4097, 70_001])
def test_small_records_forced_jit(llama, oracle_mod, schema_name, n):
    """Small records through the JIT kernel (knob jit=2): every eligible pair
    of the 11 kinds; ineligible pairs fall back to the other kernels."""
    schema = W.SCHEMAS[schema_name]
    for a in KINDS:
        for b in KINDS:
            run_case(llama, oracle_mod, schema, [n], KINDS[a], KINDS[b], seed=5 + n, paths=("permute",),
                     knobs={"jit": 2})


@pytest.mark.parametrize("knobs", [{"jit_tile": 32}, {"jit_tile": 64}, {"jit_tile": 128}, {"jit_stages": 3},
                                   {"jit_stages": 4, "jit_dst_bufs": 3}, {"jit_tile": 256}, {"jit_stages": 2, "jit_dst_bufs": 2},
                                   {"jit_soa_tma": 1}, {"jit_soa_tma": 1, "jit_tile": 32}, {"jit_soa_tma": 2},
                                   {"jit_soa_tma": 2, "jit_tile": 128}])
def test_jit_geometry_knobs(llama, oracle_mod, knobs):
    for a, b in [("aos", "soa_mb"), ("soa_mb", "aos_aligned"), ("aos", "aos_aligned"), ("soa_sb", "aosoa8"),
                 ("aos_aligned", "soa_sb")]:
        run_case(llama, oracle_mod, W.HEP100, [20_011], KINDS[a], KINDS[b], seed=9, paths=("permute",),
                 knobs=dict(knobs, jit=2))


@pytest.mark.parametrize("n", [100, 4097, 50_000])
def test_splits_jit(llama, oracle_mod, n):
    """Split mappings through the JIT kernel: the parts' images side
    by side, AoS-like parts by TMA, SoA leaves by cp.async chunks / direct stores."""
    cases = [("hep100", "aos", "split_hep"), ("hep100", "split_hep", "soa_mb"), ("hep100", "split_hep", "aos"),
             ("particle7", "aos", "split_p7"), ("particle7", "split_p7", "soa_mb"), ("listing1", "split_pos", "aos_aligned")]
    for schema_name, a, b in cases:
        schema = W.SCHEMAS[schema_name]
        run_spec_case(llama, oracle_mod, schema, [n], W.resolve_spec(a), W.resolve_spec(b), seed=n,
                      knobs={"jit": 2}, paths=("permute",))


@pytest.mark.parametrize("pad", [0, 1, 2])
@pytest.mark.parametrize("n", [64, 4097, 70_001])
def test_jit_padded_images(llama, oracle_mod, pad, n):
    """AoS part images with a 16-byte pad per record group (knob jit_pad;
    group strides multiple of 128 bytes by default: Listing-1 aligned 32-byte
    records in groups of 4), moved as 2-word-table 16-byte chunks on both
    sides, next to SoA leaves and packed parts."""
    cases = [("listing1", "aos_aligned", "split_pos"), ("listing1", "split_pos", "aos_aligned"),
             ("listing1", "aos", "aos_aligned"), ("listing1", "aos_aligned", "soa_mb"),
             ("listing1", "soa_mb", "aos_aligned"), ("hep100", "aos_aligned", "soa_mb"),
             ("hep100", "split_hep", "aos_aligned"), ("particle7", "aos_aligned", "soa_mb")]
    for schema_name, a, b in cases:
        run_spec_case(llama, oracle_mod, W.SCHEMAS[schema_name], [n], W.resolve_spec(a), W.resolve_spec(b), seed=n + pad,
                      knobs={"jit": 2, "jit_pad": pad}, paths=("permute",))


T2D_KINDS = [("aos", 1, False), ("aos", 1, True), ("soa_mb", 1, False), ("soa_sb", 1, True)]
T2D_AOSOA = [("aosoa", 8, False), ("aosoa", 4, True), ("aosoa", 32, False)]
T2D_LINS = [("row", "col"), ("col", "row"), ("row", "morton"), ("morton", "col"), ("col", "morton"), ("morton", "row")]


@pytest.mark.parametrize("knobs", [{}, {"jit_block": 0}, {"jit_bmap": 0}, {"jit_bmap": 1}, {"jit_bmap": 2},
                                   {"jit_bmap": 3}, {"jit_bmap": 4}, {"jit_tile": 512}, {"jit_tile": 1024},
                                   {"jit_dst_lsu": 1}, {"jit_dst_lsu": 1, "jit_block": 1}, {"jit_torder": 1},
                                   {"jit_torder": 2}, {"jit_tile": 2048}, {"jit_tile": 2048, "jit_stages": 2},
                                   {"jit_swizzle": 1}, {"jit_swizzle": 1, "jit_bmap": 2},
                                   {"jit_swizzle": 1, "jit_block": 1, "jit_tile": 1024}])
def test_jit_transpose_knobs(llama, oracle_mod, knobs):
    """The JIT transposing copy (rank 2, different linearisations):
    4 x 4 record blocks under every thread -> block order, per-record
    programs, both tile heights; Particle7 (4-byte leaves) and Listing-1
    (1- to 8-byte leaves, aligned records); every destination byte against
    the oracle."""
    from test_gpu_lin_trace import _pair
    for schema, ext in ((W.PARTICLE7, [64, 96]), (W.LISTING1, [32, 64])):
        for sk in T2D_KINDS:
            for dk in T2D_KINDS:
                for lins in T2D_LINS:
                    _pair(llama, oracle_mod, schema, ext if "morton" not in lins else [64, 64], sk, lins[0], dk,
                          lins[1], seed=21, paths=("auto",), knobs=dict(knobs, jit=2))


@pytest.mark.parametrize("knobs", [{}, {"jit_bmap": 1}, {"jit_swizzle": 1}, {"jit_pad": 0}])
def test_jit_transpose_aosoa(llama, oracle_mod, knobs):
    """AoSoA sides of transposing copies (block programs: a run of 4 records
    is a piece of one block), against every other kind, both schemas."""
    from test_gpu_lin_trace import _pair
    for schema, ext in ((W.PARTICLE7, [64, 96]), (W.LISTING1, [32, 64])):
        for sk in T2D_KINDS + T2D_AOSOA:
            for dk in T2D_KINDS + T2D_AOSOA:
                if sk not in T2D_AOSOA and dk not in T2D_AOSOA:
                    continue
                for lins in T2D_LINS:
                    _pair(llama, oracle_mod, schema, ext if "morton" not in lins else [64, 64], sk, lins[0], dk,
                          lins[1], seed=23, paths=("auto",), knobs=dict(knobs, jit=2))


def test_jit_chosen_for_wide_records(llama):
    m = {k: llama.Mapping(W.HEP100, [1 << 16], *KINDS[k]) for k in ("aos", "aos_aligned", "soa_mb")}
    for a in m:
        for b in m:
            if a != b:
                assert llama.plan(m[a], m[b])["jit"], (a, b)


@pytest.mark.parametrize("seed", range(24))
def test_jit_random_fuzz(llama, oracle_mod, seed):
    """Random schemas (all scalar types, static arrays, nesting) x random
    mapping kinds and splits x ragged extents, forced onto the JIT kernel
    (knob jit=2; pairs it cannot take fall back, the oracle checks every
    byte either way), and a random JIT geometry."""
    import random

    from test_gpu_parity import _random_schema, _random_spec
    rng = random.Random(1000 + seed)
    schema = _random_schema(rng)
    k = llama.Mapping(schema, [1], "aos").leaf_count
    n = rng.choice([1, 31, 64, 65, 500, 4097, 20_000])
    knobs = {"jit": 2}
    if rng.random() < 0.5:
        knobs["jit_tile"] = rng.choice([32, 64, 128, 256])
    if rng.random() < 0.3:
        knobs["jit_soa_tma"] = rng.choice([0, 2])
    if rng.random() < 0.3:
        knobs["jit_pad"] = rng.choice([0, 2])
    for _ in range(6):
        sspec, dspec = _random_spec(rng, k), _random_spec(rng, k)
        run_spec_case(llama, oracle_mod, schema, [n], sspec, dspec, seed=seed, knobs=knobs, paths=("permute",))


@pytest.mark.parametrize("seed", range(24))
def test_jit_transpose_fuzz(llama, oracle_mod, seed):
    """Random schemas (1- to 8-byte leaves, arrays, nesting) x AoS / SoA kinds
    x different storage orders of rank-2 views whose extents fit the 2-d
    tiles, forced onto the JIT transposing copy with a random geometry (block
    or per-record programs, thread -> block order, tile height, copy-out,
    swizzle); every destination byte against the oracle (pairs the JIT path
    cannot take fall back to the other kernels and are checked the same way)."""
    import random

    from test_gpu_lin_trace import _pair
    from test_gpu_parity import _random_schema
    rng = random.Random(5000 + seed)
    schema = _random_schema(rng)
    kinds = [("aos", 1, False), ("aos", 1, True), ("soa_mb", 1, False), ("soa_sb", 1, False), ("soa_sb", 1, True),
             ("aosoa", 4, False), ("aosoa", 8, True), ("aosoa", 16, False), ("aosoa", 32, False)]
    for _ in range(6):  # (about a third of the draws are JIT-eligible: 4-byte-multiple AoS records, SoA)
        ext = rng.choice([[64, 64], [128, 64], [64, 96], [32, 32], [48, 32]])
        lins = ["row", "col"] + (["morton"] if ext[0] == ext[1] else [])
        slin = rng.choice(lins)
        dlin = rng.choice([x for x in lins if x != slin])
        knobs = {"jit": 2}
        for name, choices in (("jit_block", [0, 1]), ("jit_bmap", [0, 1, 2, 3, 4]), ("jit_tile", [512, 1024, 2048]),
                              ("jit_dst_lsu", [0, 1]), ("jit_swizzle", [0, 1]), ("jit_lanes", [0, 1, 2, 3])):
            if rng.random() < 0.4:
                knobs[name] = rng.choice(choices)
        _pair(llama, oracle_mod, schema, ext, rng.choice(kinds), slin, rng.choice(kinds), dlin, seed=seed,
              paths=("auto",), knobs=knobs)
