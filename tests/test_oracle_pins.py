"""Pins for the CPU oracle (oracle/): worked examples, closed forms, the host C
compiler's and numpy's struct layouts, special cases stated in the paper,
invariants and exhaustive checks.  None of these re-types the oracle's formulas:
each compares it with something fixed independently (paper/SPEC text, ctypes'
C-ABI layout, numpy structured dtypes / reshapes, set-theoretic invariants).
"""
import ctypes
import itertools
import random

import numpy as np
import pytest

import workloads as W
from conftest import read_golden


def M(oracle_mod, schema_name, extents, mapping):
    kind, lanes, aligned = W.MAPPINGS[mapping]
    schema = W.SCHEMAS.get(schema_name, schema_name)
    return oracle_mod.Mapping(schema, extents, kind, lanes, aligned)


def leaf_index(schema, tag):
    from oracle.schema import flatten
    return [p for p, _ in flatten(schema)].index(tag)


# ---------------------------------------------------------------- P1 flattening
def test_flatten_listing1(oracle_mod):
    # "7 leaves in order Id, Pos.X, Pos.Y, Mass, Flags.0, Flags.1, Flags.2"
    leaves = oracle_mod.flatten(W.LISTING1)
    assert [p for p, _ in leaves] == ["Id", "Pos.X", "Pos.Y", "Mass", "Flags.0", "Flags.1", "Flags.2"]
    assert [t for _, t in leaves] == ["u16", "f32", "f32", "f64", "bool", "bool", "bool"]


def test_flatten_arrays_and_errors(oracle_mod):
    # f32[2][2] -> Node of 2 Nodes of 2 f32 leaves
    leaves = oracle_mod.flatten("R{a:f32[2][2]}")
    assert [p for p, _ in leaves] == ["a.0.0", "a.0.1", "a.1.0", "a.1.1"]
    # Vec -> [X, Y]
    assert [p for p, _ in oracle_mod.flatten(W.VEC)] == ["X", "Y"]
    assert len(oracle_mod.flatten(W.HEP100)) == 100
    with pytest.raises(oracle_mod.SchemaError):
        oracle_mod.flatten("R{a:f32[0]}")  # S:46 zero-extent array
    with pytest.raises(oracle_mod.SchemaError):
        oracle_mod.flatten("R{a:f16}")
    with pytest.raises(oracle_mod.SchemaError):
        oracle_mod.flatten("R{a:f32,a:f32}")  # S:34 sibling tags unique


# ---------------------------------------------------------- P3 record offsets
@pytest.mark.parametrize("row", read_golden("record_offsets.txt"), ids=lambda r: f"{r[0]}-{r[1]}")
def test_record_offsets_golden(oracle_mod, row):
    schema, mode, offs, size, _cite = row
    m = M(oracle_mod, schema, [1], "aos")
    got, got_size = m.packed_offsets() if mode == "packed" else m.aligned_offsets()
    assert got == [int(x) for x in offs.split(",")]
    assert got_size == int(size)


_CT = {1: ctypes.c_uint8, 2: ctypes.c_uint16, 4: ctypes.c_uint32, 8: ctypes.c_uint64}


def _random_schema(rng, n):
    types = list(oracle_mod_types())
    return "R{" + ",".join(f"f{j}:{rng.choice(types)}" for j in range(n)) + "}"


def oracle_mod_types():
    return ["i8", "u8", "bool", "i16", "u16", "i32", "u32", "f32", "i64", "u64", "f64"]


def _schemas_for_layout():
    rng = random.Random(7)
    out = [W.LISTING1, W.PARTICLE7, W.HEP100, W.VEC]
    out += [_random_schema(rng, rng.randint(1, 12)) for _ in range(40)]
    return out


@pytest.mark.parametrize("schema", _schemas_for_layout())
def test_record_offsets_vs_c_compiler_and_numpy(oracle_mod, schema):
    """The host C compiler's struct layout (via ctypes, flat struct) and numpy
    structured dtypes fix packed/aligned offsets independently."""
    sizes = oracle_mod.leaf_sizes(schema)
    m = oracle_mod.Mapping(schema, [1], "aos")
    fields = [(f"f{k}", _CT[s]) for k, s in enumerate(sizes)]

    class Packed(ctypes.Structure):
        _pack_ = 1
        _fields_ = fields

    class Natural(ctypes.Structure):
        _fields_ = fields

    po, ps = m.packed_offsets()
    ao, asz = m.aligned_offsets()
    assert po == [getattr(Packed, f).offset for f, _ in fields] and ps == ctypes.sizeof(Packed)
    assert ao == [getattr(Natural, f).offset for f, _ in fields] and asz == ctypes.sizeof(Natural)
    spec = {"names": [f for f, _ in fields], "formats": [f"u{s}" for s in sizes]}
    dp, da = np.dtype(spec, align=False), np.dtype(spec, align=True)
    assert po == [dp.fields[f][1] for f, _ in fields] and ps == dp.itemsize
    assert ao == [da.fields[f][1] for f, _ in fields] and asz == da.itemsize


def test_nesting_reading_discriminator(oracle_mod):
    """DESIGN.md reading #3: alignment follows the flattened per-leaf rule
    (S:69-77), not C nested-struct rules.  Outer{A{d:f64,b:bool},c:bool}:
    flattened 16 B, nested C struct 24 B."""
    m = oracle_mod.Mapping(W.OUTER, [1], "aos", aligned=True)
    assert m.aligned_offsets() == ([0, 8, 9], 16)

    class A(ctypes.Structure):
        _fields_ = [("d", ctypes.c_double), ("b", ctypes.c_uint8)]

    class Outer(ctypes.Structure):
        _fields_ = [("a", A), ("c", ctypes.c_uint8)]

    assert ctypes.sizeof(Outer) == 24


def test_hep100_layout(oracle_mod):
    m = oracle_mod.Mapping(W.HEP100, [1], "aos")
    po, ps = m.packed_offsets()
    ao, asz = m.aligned_offsets()
    assert ps == 380 and asz == 480
    assert ao[:10] == [0, 4, 8, 16, 24, 28, 32, 34, 35, 40]
    sizes = oracle_mod.leaf_sizes(W.HEP100)
    assert sorted(set(sizes)) == [1, 2, 4, 8]
    assert [sizes.count(s) for s in (8, 4, 2, 1)] == [20, 40, 20, 20]  # 20 f64, 30 f32 + 10 i32, 20 i16, 20 bool
    misaligned = sum(1 for o, s in zip(po, sizes) if o % s)
    assert misaligned == 36


# -------------------------------------------------------- P4-P6 worked examples
@pytest.mark.parametrize("row", read_golden("worked_examples.txt"), ids=lambda r: "-".join(r[:5]))
def test_worked_examples(oracle_mod, row):
    schema, ext, mapping, i, tag, blob, off, _cite = row
    m = M(oracle_mod, schema, [int(ext)], mapping)
    k = leaf_index(W.SCHEMAS[schema], tag)
    assert m.addr(int(i), k) == (int(blob), int(off))


# --------------------------------------------------------------- P2 blob sizes
@pytest.mark.parametrize("row", read_golden("blob_sizes.txt"), ids=lambda r: "-".join(r[:3]))
def test_blob_sizes_golden(oracle_mod, row):
    schema, ext, mapping, sizes, _cite = row
    m = M(oracle_mod, schema, [int(e) for e in ext.split("x")], mapping)
    assert m.blob_sizes() == [int(s) for s in sizes.split(",")]


def test_blob_count(oracle_mod):
    assert M(oracle_mod, "listing1", [4], "soa_mb").blob_count == 7
    assert M(oracle_mod, "listing1", [4], "aos").blob_count == 1


@pytest.mark.parametrize("row", read_golden("linearize.txt"))
def test_linearize_golden(oracle_mod, row):
    ext, idx, flat, _ = row
    m = oracle_mod.Mapping(W.VEC, [int(e) for e in ext.split(",")], "aos")
    assert m.linearize([int(x) for x in idx.split(",")]) == int(flat)


def test_linearize_matches_enumeration_order(oracle_mod):
    """ArrayDimsIndexRange enumerates {0,0},{0,1},{0,2},{1,0},...;
    itertools.product produces the same lexicographic order independently."""
    for ext in ([3, 3], [4, 3], [2, 2, 2], [5], [2, 3, 4]):
        m = oracle_mod.Mapping(W.VEC, ext, "aos")
        flats = [m.linearize(list(ix)) for ix in itertools.product(*[range(e) for e in ext])]
        assert flats == list(range(int(np.prod(ext))))  # bijection, in order
    m = oracle_mod.Mapping(W.VEC, [3, 3], "aos")
    assert m.linearize([3, 0]) == -1


# ----------------------------------------------------------- P7 special cases
def _all_addrs(m):
    return [m.addr(i, k) for i in range(m.record_count) for k in range(m.n_leaves)]


@pytest.mark.parametrize("schema", [W.LISTING1, W.PARTICLE7, W.OUTER, W.HEP100])
@pytest.mark.parametrize("n", [1, 5, 31, 32, 33])
def test_aosoa_L1_is_aos_and_LN_is_soa_sb(oracle_mod, schema, n):
    """S:286 "L=1 degenerates to packedAoS"; "SoA can be seen as an
    AoSoA with an inner array length equal to the product of the array
    dimensions"."""
    for aligned in (False, True):
        aos = oracle_mod.Mapping(schema, [n], "aos", 1, aligned)
        a1 = oracle_mod.Mapping(schema, [n], "aosoa", 1, aligned)
        assert _all_addrs(aos) == _all_addrs(a1) and aos.blob_sizes() == a1.blob_sizes()
    sb = oracle_mod.Mapping(schema, [n], "soa_sb")
    an = oracle_mod.Mapping(schema, [n], "aosoa", n)
    assert _all_addrs(sb) == _all_addrs(an) and sb.blob_sizes() == an.blob_sizes()


# ----------------------------------------------------------- P10 invariants
def _all_mappings(n):
    out = [("aos", 1, False), ("aos", 1, True), ("soa_sb", 1, False), ("soa_sb", 1, True), ("soa_mb", 1, False)]
    out += [("aosoa", L, a) for L in (1, 2, 3, 4, 8, 32) for a in (False, True)]
    if n > 0:
        out.append(("aosoa", n, False))
    return out


@pytest.mark.parametrize("schema", [W.LISTING1, W.PARTICLE7, W.OUTER, W.VEC, W.HEP100])
@pytest.mark.parametrize("ext", [[4, 3], [5], [1], [33], [2, 2, 2]])
def test_disjoint_contained_tiling(oracle_mod, schema, ext):
    """non-overlap, containment; packed AoS / SoA tile exactly;
    aligned AoS and AoSoA leave padding gaps only."""
    n = int(np.prod(ext))
    sizes = oracle_mod.leaf_sizes(schema)
    for kind, L, aligned in _all_mappings(n):
        m = oracle_mod.Mapping(schema, ext, kind, L, aligned)
        bs = m.blob_sizes()
        used = [np.zeros(s, dtype=np.int32) for s in bs]
        for i in range(n):
            for k in range(len(sizes)):
                b, o = m.addr(i, k)
                assert o + sizes[k] <= bs[b]
                used[b][o:o + sizes[k]] += 1
        assert all(int(u.max(initial=0)) <= 1 for u in used), (kind, L, aligned)
        covered = sum(int(u.sum()) for u in used)
        assert covered == n * sum(sizes)
        if (kind == "aos" and not aligned) or (kind == "soa_mb") or (kind == "soa_sb" and not aligned) \
                or (kind == "aosoa" and not aligned and n % L == 0):
            assert covered == sum(bs), (kind, L, aligned)


def test_splitmix64_reference_vectors(oracle_mod):
    """splitmix64 (Vigna's reference splitmix64.c, seed 1234567): the first two
    outputs of the sequence.  oracle_splitmix64(x) is the output for state x."""
    g = 0x9E3779B97F4A7C15
    assert oracle_mod.splitmix64(1234567) == 6457827717110365317
    assert oracle_mod.splitmix64(1234567 + g) == 3203168211198807973


def test_generate_recipe(oracle_mod):
    """Input recipe: byte b of leaf k of record i = byte b of splitmix64(seed ^ (i*K+k))."""
    m = oracle_mod.Mapping(W.PARTICLE7, [64], "aos")
    blobs = oracle_mod.make_view(m, 42)
    mat = blobs[0].view(np.uint32).reshape(64, 7)
    for i in (0, 5, 63):
        for k in range(7):
            assert int(mat[i, k]) == oracle_mod.splitmix64(42 ^ (i * 7 + k)) & 0xFFFFFFFF


# ------------------------------------------------------- P8 numpy (Particle7)
@pytest.mark.parametrize("n", [32, 256, 4096])
def test_particle7_copies_equal_numpy_reshapes(oracle_mod, n):
    """For 7x f32 every mapping is a numpy view of an (N,7) matrix M:
    SoA SB = M.T, SoA MB = columns, AoSoA-L = M.reshape(N/L,L,7).transpose(0,2,1)."""
    src = oracle_mod.Mapping(W.PARTICLE7, [n], "aos")
    sblobs = oracle_mod.make_view(src, 42)
    Mx = sblobs[0].view(np.uint32).reshape(n, 7)
    sb = oracle_mod.copy(src, sblobs, oracle_mod.Mapping(W.PARTICLE7, [n], "soa_sb"))
    assert np.array_equal(sb[0].view(np.uint32), np.ascontiguousarray(Mx.T).ravel())
    mb = oracle_mod.copy(src, sblobs, oracle_mod.Mapping(W.PARTICLE7, [n], "soa_mb"))
    for k in range(7):
        assert np.array_equal(mb[k].view(np.uint32), Mx[:, k])
    for L in (4, 8, 32):
        a = oracle_mod.copy(src, sblobs, oracle_mod.Mapping(W.PARTICLE7, [n], "aosoa", L))
        exp = np.ascontiguousarray(Mx.reshape(n // L, L, 7).transpose(0, 2, 1)).ravel()
        assert np.array_equal(a[0].view(np.uint32), exp)
    al = oracle_mod.copy(src, sblobs, oracle_mod.Mapping(W.PARTICLE7, [n], "aos", 1, True))
    assert np.array_equal(al[0], sblobs[0])


# --------------------------------------------- P9 numpy structured (hetero)
def _dtypes(schema):
    sizes = [int(s) for s in __import__("oracle").leaf_sizes(schema)]
    spec = {"names": [f"f{k}" for k in range(len(sizes))], "formats": [f"u{s}" for s in sizes]}
    return sizes, np.dtype(spec, align=False), np.dtype(spec, align=True)


@pytest.mark.parametrize("schema", [W.LISTING1, W.HEP100, W.OUTER])
@pytest.mark.parametrize("n", [1, 7, 64])
def test_hetero_copies_equal_numpy_structured(oracle_mod, schema, n):
    """numpy structured arrays fix the heterogeneous layouts: assigning fields
    into a zeroed align=True array gives aligned AoS incl. zero padding; per
    field contiguous arrays give SoA MB/SB; a block dtype with (L,) subarray
    fields gives AoSoA-L."""
    sizes, dp, da = _dtypes(schema)
    src = oracle_mod.Mapping(schema, [n], "aos")
    sblobs = oracle_mod.make_view(src, 1)
    P = np.frombuffer(sblobs[0].tobytes(), dtype=dp)
    A = np.zeros(n, dtype=da)
    for f in dp.names:
        A[f] = P[f]
    got = oracle_mod.copy(src, sblobs, oracle_mod.Mapping(schema, [n], "aos", 1, True))
    assert got[0].tobytes() == A.tobytes()
    mb = oracle_mod.copy(src, sblobs, oracle_mod.Mapping(schema, [n], "soa_mb"))
    assert [b.tobytes() for b in mb] == [np.ascontiguousarray(P[f]).tobytes() for f in dp.names]
    sb = oracle_mod.copy(src, sblobs, oracle_mod.Mapping(schema, [n], "soa_sb"))
    assert sb[0].tobytes() == b"".join(np.ascontiguousarray(P[f]).tobytes() for f in dp.names)
    for L in (1, 4, 8):
        blk = np.dtype({"names": dp.names, "formats": [(f"u{s}", (L,)) for s in sizes]}, align=False)
        nb = -(-n // L)
        B = np.zeros(nb, dtype=blk)
        for f in dp.names:
            col = np.zeros(nb * L, dtype=P[f].dtype)
            col[:n] = P[f]
            B[f] = col.reshape(nb, L)
        a = oracle_mod.copy(src, sblobs, oracle_mod.Mapping(schema, [n], "aosoa", L))
        assert a[0].tobytes() == B.tobytes()


# --------------------------------------------------- P10 copy-level invariants
@pytest.mark.parametrize("schema", [W.LISTING1, W.HEP100])
def test_round_trip_identity(oracle_mod, schema):
    """AoS -> SoA MB -> AoSoA8 -> aligned AoS -> packed AoS is the identity."""
    n = 100
    chain = [("aos", 1, False), ("soa_mb", 1, False), ("aosoa", 8, False), ("aos", 1, True), ("aos", 1, False)]
    maps = [oracle_mod.Mapping(schema, [n], *c) for c in chain]
    first = oracle_mod.make_view(maps[0], 2)
    cur = first
    for a, b in zip(maps, maps[1:]):
        cur = oracle_mod.copy(a, cur, b)
    assert cur[0].tobytes() == first[0].tobytes()


def test_composition_and_generation_agree(oracle_mod):
    """copy(B->C) o copy(A->B) == copy(A->C) == generate-through-C (per-(i,k)
    logical read-back equality)."""
    n = 77
    kinds = [("aos", 1, False), ("aos", 1, True), ("soa_sb", 1, False), ("soa_mb", 1, False),
             ("aosoa", 4, False), ("aosoa", 3, False), ("aosoa", 32, True)]
    for schema in (W.LISTING1, W.HEP100):
        maps = [oracle_mod.Mapping(schema, [n], *c) for c in kinds]
        views = [oracle_mod.make_view(m, 42) for m in maps]
        for a in range(len(maps)):
            for c in range(len(maps)):
                direct = oracle_mod.copy(maps[a], views[a], maps[c])
                assert [x.tobytes() for x in direct] == [x.tobytes() for x in views[c]]
        b = 3
        via = oracle_mod.copy(maps[b], oracle_mod.copy(maps[0], views[0], maps[b]), maps[5])
        assert [x.tobytes() for x in via] == [x.tobytes() for x in views[5]]


def test_src_padding_never_leaks(oracle_mod):
    """Reading #13: poisoned src padding (0xCD) does not influence the output;
    reading #12: dst padding is written as 0."""
    n = 50
    for schema in (W.LISTING1, W.HEP100):
        src = oracle_mod.Mapping(schema, [n], "aosoa", 8, True)
        clean = oracle_mod.make_view(src, 9, pad_fill=0)
        dirty = oracle_mod.make_view(src, 9, pad_fill=0xCD)
        assert clean[0].tobytes() != dirty[0].tobytes()
        for kind in [("aos", 1, True), ("aosoa", 8, True), ("aosoa", 32, False), ("soa_sb", 1, True)]:
            dst = oracle_mod.Mapping(schema, [n], *kind)
            a = oracle_mod.copy(src, clean, dst, dst.alloc(0x77))
            b = oracle_mod.copy(src, dirty, dst, dst.alloc(0x11))
            assert [x.tobytes() for x in a] == [x.tobytes() for x in b]
        ident = oracle_mod.copy(src, dirty, src)
        assert ident[0].tobytes() == clean[0].tobytes()


def test_partition_and_threads_independent(oracle_mod):
    """any worker count / partition yields identical contents."""
    n = 1000
    src = oracle_mod.Mapping(W.LISTING1, [n], "aos")
    dst = oracle_mod.Mapping(W.LISTING1, [n], "aosoa", 8, True)
    sb = oracle_mod.make_view(src, 42)
    ref = oracle_mod.copy(src, sb, dst, nthreads=1)
    for t in (2, 4, 8):
        assert oracle_mod.copy(src, sb, dst, nthreads=t)[0].tobytes() == ref[0].tobytes()
    out = dst.alloc()
    cuts = sorted(random.Random(3).sample(range(1, n), 9))
    bounds = [0] + cuts + [n]
    order = list(range(len(bounds) - 1))
    random.Random(4).shuffle(order)
    for j in order:
        oracle_mod.copy_range(src, sb, None, dst, out, None, bounds[j], bounds[j + 1])
    assert out[0].tobytes() == ref[0].tobytes()


def test_windowed_copy_range_matches(oracle_mod):
    """copy_range over blob windows (used for chunked parity at full sizes)."""
    n = 256
    for (sk, dk) in [(("aos", 1, True), ("soa_sb", 1, False)), (("aosoa", 32, False), ("soa_mb", 1, False))]:
        src = oracle_mod.Mapping(W.LISTING1, [n], *sk)
        dst = oracle_mod.Mapping(W.LISTING1, [n], *dk)
        sb = oracle_mod.make_view(src, 5)
        full = oracle_mod.copy(src, sb, dst)
        a, b = 64, 160
        # window = the byte span each blob uses for records [a,b)
        def span(m, nb):
            lo = [None] * nb
            hi = [0] * nb
            for i in range(a, b):
                for k in range(m.n_leaves):
                    bb, o = m.addr(i, k)
                    lo[bb] = o if lo[bb] is None else min(lo[bb], o)
                    hi[bb] = max(hi[bb], o + m.sizes[k])
            return lo, hi
        slo, shi = span(src, src.blob_count)
        dlo, dhi = span(dst, dst.blob_count)
        swin = [np.ascontiguousarray(sb[j][slo[j]:shi[j]]) for j in range(src.blob_count)]
        dwin = [np.zeros(dhi[j] - dlo[j], np.uint8) for j in range(dst.blob_count)]
        oracle_mod.copy_range(src, swin, slo, dst, dwin, dlo, a, b)
        # compare the bytes owned by records [a,b) (SoA SB windows span other records too)
        owned = [np.zeros(dhi[j] - dlo[j], bool) for j in range(dst.blob_count)]
        for i in range(a, b):
            for k in range(dst.n_leaves):
                bb, o = dst.addr(i, k)
                owned[bb][o - dlo[bb]:o - dlo[bb] + dst.sizes[k]] = True
        for j in range(dst.blob_count):
            assert np.array_equal(dwin[j][owned[j]], full[j][dlo[j]:dhi[j]][owned[j]])
            assert not dwin[j][~owned[j]].any()


def test_errors_and_empty(oracle_mod):
    a = oracle_mod.Mapping(W.LISTING1, [4], "aos")
    with pytest.raises(ValueError):
        oracle_mod.copy(a, a.alloc(), oracle_mod.Mapping(W.LISTING1, [5], "aos"))  # S:486 shape mismatch
    with pytest.raises(ValueError):
        oracle_mod.copy(a, a.alloc(), oracle_mod.Mapping(W.VEC, [4], "aos"))  # record mismatch
    e = oracle_mod.Mapping(W.LISTING1, [0], "aosoa", 8)
    assert e.blob_sizes() == [0] and e.record_count == 0
    out = oracle_mod.copy(e, e.alloc(), oracle_mod.Mapping(W.LISTING1, [0], "soa_mb"))
    assert all(x.size == 0 for x in out)


def test_run_structure_chunk_economy(oracle_mod):
    """S:521 / P:759: maximal common contiguous single-leaf runs number
    K*N/min(Ls,Ld) when min divides max (AoSoA8->AoSoA4: 112, AoSoA8->AoSoA32:
    56, SoA MB->SB: 7, AoS->SoA: 448 for Particle7 with N=64)."""
    n = 64

    def runs(a, b):
        # runs of one leaf ("min(N,M) fields as chunks"), in source order
        items = []
        for k in range(7):
            for i in range(n):
                items.append((k, a.addr(i, k), b.addr(i, k)))
        items.sort()
        count, prev = 0, None
        for k, (bs, os), (bd, od) in items:
            if not (prev and prev == (k, bs, os, bd, od)):
                count += 1
            prev = (k, bs, os + 4, bd, od + 4)
        return count

    mk = lambda *c: oracle_mod.Mapping(W.PARTICLE7, [n], *c)
    assert runs(mk("aosoa", 8), mk("aosoa", 4)) == 112
    assert runs(mk("aosoa", 8), mk("aosoa", 32)) == 56
    assert runs(mk("soa_mb"), mk("soa_sb")) == 7
    assert runs(mk("aos"), mk("soa_mb")) == 448
