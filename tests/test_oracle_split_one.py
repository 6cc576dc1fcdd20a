"""Pins of the oracle's One and Split mappings against
hand-derived worked examples (tests/golden/split_one.txt), numpy's structured
layouts, special cases that reduce to already-pinned mappings, and brute-force
disjointness."""
import itertools

import numpy as np
import pytest

import workloads as W
from conftest import read_golden

ROWS = read_golden("split_one.txt")


def _m(oracle, name, extents, schema=None):
    if name in W.SPLITS:
        schema = W.SCHEMAS[W.SPLITS[name][0]]
    return oracle.mapping_from_spec(schema, extents, W.resolve_spec(name))


@pytest.mark.parametrize("row", [r for r in ROWS if r[0] == "addr"], ids=lambda r: "-".join(r[1:6]))
def test_worked_addresses(oracle_mod, row):
    _, name, ext, i, k, blob, off, _cite = row
    m = _m(oracle_mod, name, [int(e) for e in ext.split()], W.LISTING1)
    assert m.addr(int(i), int(k)) == (int(blob), int(off))


@pytest.mark.parametrize("row", [r for r in ROWS if r[0] == "blobs"], ids=lambda r: "-".join(r[1:4]))
def test_worked_blob_sizes(oracle_mod, row):
    _, name, schema, ext, sizes, _cite = row
    m = _m(oracle_mod, name, [int(e) for e in ext.split()], W.SCHEMAS[schema])
    assert m.blob_sizes() == [int(v) for v in sizes.split()]
    assert m.blob_count == len(sizes.split())


@pytest.mark.parametrize("schema", [W.LISTING1, W.PARTICLE7, W.HEP100, W.OUTER])
def test_one_is_record_zero_of_aligned_aos(oracle_mod, schema):
    """One: every index maps where aligned AoS maps index 0, and the
    blob is one aligned record (aligned AoS is pinned to the C compiler)."""
    one = oracle_mod.Mapping(schema, [3, 5], "one")
    ref = oracle_mod.Mapping(schema, [1], "aos", aligned=True)
    assert one.blob_sizes() == ref.blob_sizes()
    for i in range(15):
        for k in range(one.n_leaves):
            assert one.addr(i, k) == ref.addr(0, k)
    with pytest.raises(IndexError):  # S:291 "bounds error on index (still validated)"
        one.addr(15, 0)


def test_one_copy_keeps_last_record(oracle_mod):
    """Copying N records into One writes every record to the same place; the
    sequential copy leaves the last one.  With N = 1 One equals aligned AoS."""
    src_m = oracle_mod.Mapping(W.LISTING1, [6], "aos")
    src = oracle_mod.make_view(src_m, 3)
    one = oracle_mod.copy(src_m, src, oracle_mod.Mapping(W.LISTING1, [6], "one"))
    last = oracle_mod.Mapping(W.LISTING1, [1], "aos")
    last_blobs = [src[0][5 * 21:6 * 21].copy()]  # packed record 5 (S = 21)
    ref = oracle_mod.copy(last, last_blobs, oracle_mod.Mapping(W.LISTING1, [1], "aos", aligned=True))
    assert (one[0] == ref[0]).all()


@pytest.mark.parametrize("n", [1, 7, 64])
def test_split_pos_equals_numpy_columns_and_struct(oracle_mod, n):
    """S:304 split: Pos -> SoA MB columns, the rest -> packed AoS, checked
    against numpy's packed structured array of the full record."""
    full = np.dtype([("Id", "<u2"), ("X", "<f4"), ("Y", "<f4"), ("Mass", "<f8"),
                     ("F0", "u1"), ("F1", "u1"), ("F2", "u1")], align=False)
    rest = np.dtype([("Id", "<u2"), ("Mass", "<f8"), ("F0", "u1"), ("F1", "u1"), ("F2", "u1")], align=False)
    rng = np.random.default_rng(n)
    arr = np.frombuffer(rng.integers(0, 256, n * full.itemsize, dtype=np.uint8).tobytes(), dtype=full)
    src_m = oracle_mod.Mapping(W.LISTING1, [n], "aos")
    split = _m(oracle_mod, "split_pos", [n])
    out = oracle_mod.copy(src_m, [np.frombuffer(arr.tobytes(), np.uint8).copy()], split)
    assert out[0].tobytes() == arr["X"].tobytes()
    assert out[1].tobytes() == arr["Y"].tobytes()
    r = np.zeros(n, rest)
    for f in rest.names:
        r[f] = arr[f]
    assert out[2].tobytes() == r.tobytes()


@pytest.mark.parametrize("schema", [W.LISTING1, W.PARTICLE7, W.HEP100])
@pytest.mark.parametrize("cut", [1, 2, 5])
def test_split_of_soa_mb_prefix_is_soa_mb(oracle_mod, schema, cut):
    """Splitting off leaves [0, cut) into SoA MB and the rest into SoA MB gives
    exactly SoA MB of the whole record (pins the blob renumbering of S:299)."""
    sizes = oracle_mod.leaf_sizes(schema)
    ext = [13]
    a = oracle_mod.Mapping(sizes[:cut], ext, "soa_mb")
    b = oracle_mod.Mapping(sizes[cut:], ext, "soa_mb")
    s = oracle_mod.Mapping.split(sizes, list(range(cut)), a, b)
    ref = oracle_mod.Mapping(schema, ext, "soa_mb")
    assert s.blob_sizes() == ref.blob_sizes()
    for i in range(13):
        for k in range(len(sizes)):
            assert s.addr(i, k) == ref.addr(i, k)


@pytest.mark.parametrize("name", ["split_pos", "mapping_c", "split_p7", "split_hep"])
@pytest.mark.parametrize("ext", [[4, 3], [5], [1], [33]])
def test_split_disjoint_contained(oracle_mod, name, ext):
    """zero overlapping byte ranges, all inside the blobs -- except
    the One part, whose records all share one place."""
    m = _m(oracle_mod, name, ext)
    sizes = m.blob_sizes()
    n = m.record_count
    owner = {}
    one_leaves = set()
    if name == "mapping_c":
        one_leaves = {3}  # Mass
    for i in range(n):
        for k in range(m.n_leaves):
            b, o = m.addr(i, k)
            assert o + m.sizes[k] <= sizes[b]
            for byte in range(o, o + m.sizes[k]):
                key = (b, byte)
                if k in one_leaves:
                    assert owner.setdefault(key, ("one", k)) == ("one", k)
                else:
                    assert key not in owner, (name, i, k, key)
                    owner[key] = (i, k)
    if name == "split_pos" or (name == "split_p7" and n % 8 == 0):  # packed parts: blobs tiled exactly
        assert len(owner) == sum(sizes)


@pytest.mark.parametrize("name", ["split_pos", "mapping_c", "split_p7", "split_hep"])
def test_split_round_trip(oracle_mod, name):
    schema = W.SCHEMAS[W.SPLITS[name][0]]
    n = 1 if name == "mapping_c" else 37  # a One part holds one record
    aos = oracle_mod.Mapping(schema, [n], "aos")
    src = oracle_mod.make_view(aos, 11)
    s = _m(oracle_mod, name, [n])
    back = oracle_mod.copy(s, oracle_mod.copy(aos, src, s), aos)
    assert all((x == y).all() for x, y in zip(src, back))


def test_mapping_c_source_broadcasts_mass(oracle_mod):
    """MappingC as a source: every record reads the one Mass value."""
    n = 9
    m = _m(oracle_mod, "mapping_c", [n])
    blobs = oracle_mod.make_view(m, 5)
    dst_m = oracle_mod.Mapping(W.LISTING1, [n], "soa_mb")
    out = oracle_mod.copy(m, blobs, dst_m)
    assert all(out[3][8 * i:8 * i + 8].tobytes() == blobs[2].tobytes() for i in range(n))


def test_split_validation(oracle_mod):
    sizes = oracle_mod.leaf_sizes(W.LISTING1)
    a = oracle_mod.Mapping(sizes[:2], [4], "soa_mb")
    b = oracle_mod.Mapping(sizes[2:], [4], "aos")
    oracle_mod.Mapping.split(sizes, [0, 1], a, b)
    with pytest.raises(ValueError):  # S:303 an empty part is rejected
        oracle_mod.Mapping.split(sizes, list(range(7)), oracle_mod.Mapping(sizes, [4], "aos"), b)
    with pytest.raises(ValueError):  # leaf sizes do not match the parts
        oracle_mod.Mapping.split(sizes, [0, 3], a, b)
    with pytest.raises(ValueError):  # extents differ
        oracle_mod.Mapping.split(sizes, [0, 1], a, oracle_mod.Mapping(sizes[2:], [5], "aos"))
    with pytest.raises(ValueError):  # not increasing
        oracle_mod.Mapping.split(sizes, [1, 0], oracle_mod.Mapping([4, 2], [4], "soa_mb"), b)
