"""Pins of the oracle's linearisations and of the
Trace / Heatmap counters."""
import itertools

import numpy as np
import pytest

import workloads as W
from conftest import read_golden


@pytest.mark.parametrize("row", read_golden("linearize_lin.txt"), ids=lambda r: "-".join(r[:3]))
def test_linearize_golden(oracle_mod, row):
    lin, ext, idx, flat, _cite = row
    m = oracle_mod.Mapping(W.VEC, [int(e) for e in ext.split()], "aos", lin=lin)
    assert m.linearize([int(x) for x in idx.split()]) == int(flat)


@pytest.mark.parametrize("lin,ext", [("row", [4, 3]), ("col", [4, 3]), ("col", [2, 3, 5]), ("morton", [8, 8]),
                                     ("morton", [4, 4, 4]), ("morton", [16])])
def test_linearize_is_a_bijection(oracle_mod, lin, ext):
    m = oracle_mod.Mapping(W.VEC, ext, "aos", lin=lin)
    flats = sorted(m.linearize(list(ix)) for ix in itertools.product(*[range(e) for e in ext]))
    assert flats == list(range(int(np.prod(ext))))


def test_morton_structure(oracle_mod):
    """Every aligned 2^j-cube occupies consecutive codes (the Z-order
    recursion); the last index alone sets only the even bits (reading #26)."""
    n = 16
    m = oracle_mod.Mapping(W.VEC, [n, n], "aos", lin="morton")
    for j in (1, 2, 3):
        s = 1 << j
        for y0 in range(0, n, s):
            for x0 in range(0, n, s):
                codes = sorted(m.linearize([y, x]) for y in range(y0, y0 + s) for x in range(x0, x0 + s))
                assert codes == list(range(codes[0], codes[0] + s * s))
    for x in range(n):
        assert m.linearize([0, x]) & 0xAAAA == 0
        assert m.linearize([x, 0]) & 0x5555 == 0
    with pytest.raises(ValueError):
        oracle_mod.Mapping(W.VEC, [4, 8], "aos", lin="morton")  # S:176 equal powers of two
    with pytest.raises(ValueError):
        oracle_mod.Mapping(W.VEC, [6, 6], "aos", lin="morton")


@pytest.mark.parametrize("h,w", [(3, 5), (16, 33)])
def test_col_major_aos_is_numpy_transpose(oracle_mod, h, w):
    """A column-major AoS of an (h, w) Particle7 array is the (w, h) transpose
    of the row-major one (numpy), and the round trip is the identity."""
    row = oracle_mod.Mapping(W.PARTICLE7, [h, w], "aos")
    col = oracle_mod.Mapping(W.PARTICLE7, [h, w], "aos", lin="col")
    src = oracle_mod.make_view(row, 5)
    out = oracle_mod.copy(row, src, col)
    a = src[0].reshape(h, w, 28)
    assert out[0].tobytes() == np.ascontiguousarray(a.transpose(1, 0, 2)).tobytes()
    back = oracle_mod.copy(col, out, row)
    assert (back[0] == src[0]).all()
    # SoA MB column-major: each leaf column is the transposed matrix
    colsoa = oracle_mod.Mapping(W.PARTICLE7, [h, w], "soa_mb", lin="col")
    cs = oracle_mod.copy(row, src, colsoa)
    for k in range(7):
        leaf = a[:, :, 4 * k:4 * k + 4]
        assert cs[k].tobytes() == np.ascontiguousarray(leaf.transpose(1, 0, 2)).tobytes()


def test_morton_copy_round_trip_and_generator(oracle_mod):
    """Data is attached to the array index, not the storage position: a view
    generated in Morton order equals a row-major view copied into Morton."""
    ext = [8, 8]
    row = oracle_mod.Mapping(W.LISTING1, ext, "soa_sb")
    mor = oracle_mod.Mapping(W.LISTING1, ext, "aosoa", lanes=4, lin="morton")
    a = oracle_mod.make_view(row, 9)
    b = oracle_mod.copy(row, a, mor)
    c = oracle_mod.make_view(mor, 9)
    assert all((x == y).all() for x, y in zip(b, c))
    assert all((x == y).all() for x, y in zip(oracle_mod.copy(mor, b, row), a))


@pytest.mark.parametrize("src,dst", [("aos", "aos_aligned"), ("soa_mb", "aosoa8"), ("split_pos", "soa_sb")])
def test_trace_and_heatmap_copy(oracle_mod, src, dst):
    """Copy: every leaf resolved once per record on each side (S:310 counting
    per resolution); heat = 1 on every payload byte, 0 on padding; heat sums
    equal sum(hits x size)."""
    n = 37
    schema = W.LISTING1
    sm = oracle_mod.mapping_from_spec(schema, [n], W.resolve_spec(src))
    dm = oracle_mod.mapping_from_spec(schema, [n], W.resolve_spec(dst))
    sb = oracle_mod.make_view(sm, 2)
    out, sh, dh, sheat, dheat = oracle_mod.copy_counted(sm, sb, dm)
    assert (sh == n).all() and (dh == n).all()
    assert all((x == y).all() for x, y in zip(out, oracle_mod.copy(sm, sb, dm)))
    sizes = np.array(sm.sizes, np.uint64)
    for m, hits, heat in ((sm, sh, sheat), (dm, dh, dheat)):
        assert sum(int(h.sum()) for h in heat) == int((hits * sizes).sum())
        payload = np.zeros(sum(len(h) for h in heat), bool)
        starts = np.cumsum([0] + [len(h) for h in heat])
        for i in range(n):
            for k in range(m.n_leaves):
                b, o = m.addr(i, k)
                payload[starts[b] + o: starts[b] + o + m.sizes[k]] = True
        flat = np.concatenate(heat)
        assert (flat[payload] == 1).all() and (flat[~payload] == 0).all()


@pytest.mark.parametrize("name", ["aos", "soa_mb", "aosoa8"])
def test_trace_and_heatmap_move(oracle_mod, name):
    """after one move each Pos.* and Vel.* counter is N, Mass 0;
    S:319: AoS N = 64: Mass bytes 0, Pos / Vel bytes 1."""
    n = 64
    m = oracle_mod.mapping_from_spec(W.PARTICLE7, [n], W.resolve_spec(name))
    blobs = oracle_mod.copy(oracle_mod.Mapping(W.PARTICLE7, [n], "aos"),
                            [np.frombuffer(W.particle_values(n).tobytes(), np.uint8).copy()], m)
    ref = oracle_mod.nbody_move(m, [b.copy() for b in blobs], 1e-4)
    hits, heat = oracle_mod.nbody_move_counted(m, blobs, 1e-4)
    assert all((x == y).all() for x, y in zip(blobs, ref))
    assert list(hits) == [n] * 6 + [0]
    for i in range(n):
        for k in range(7):
            b, o = m.addr(i, k)
            assert (heat[b][o:o + 4] == (0 if k == 6 else 1)).all()
    assert sum(int(h.sum()) for h in heat) == 6 * n * 4
