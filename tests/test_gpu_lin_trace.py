"""GPU parity of linearised views and of the Trace /
Heatmap counters against the oracle."""
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


def _pair(llama, oracle, schema, ext, sspec, slin, dspec, dlin, seed=3, paths=("auto",), knobs=None):
    sm = llama.Mapping.from_spec(schema, ext, sspec, lin=slin)
    dm = llama.Mapping.from_spec(schema, ext, dspec, lin=dlin)
    so = oracle.mapping_from_spec(schema, ext, sspec, lin=slin)
    do = oracle.mapping_from_spec(schema, ext, dspec, lin=dlin)
    sb = sm.alloc("cuda")
    llama.generate(sm, sb, seed, pad_byte=0xCD)
    src = oracle.make_view(so, seed, pad_fill=0xCD)
    for j, t in enumerate(sb):  # the generator attaches values to the array index
        assert np.array_equal(t.cpu().numpy(), src[j]), f"generated blob {j}"
    exp = oracle.copy(so, src, do)
    for path in paths:
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
            assert np.array_equal(t.cpu().numpy(), exp[j]), (sspec, slin, dspec, dlin, path, j)


KINDS = [("aos", 1, False), ("soa_mb", 1, False), ("aosoa", 8, False), ("aos", 1, True)]


@pytest.mark.parametrize("ext", [[64, 33], [5, 7, 3], [1, 1], [100, 37], [31, 1000], [64, 96], [96, 64]])
@pytest.mark.parametrize("lins", [("row", "col"), ("col", "row"), ("col", "col")])
def test_row_col_copies(llama, oracle_mod, ext, lins):
    for sk in KINDS:
        for dk in KINDS:
            _pair(llama, oracle_mod, W.LISTING1, ext, sk, lins[0], dk, lins[1],
                  paths=("auto", "naive", "permute", "run", "blobcopy", "transpose"))


@pytest.mark.parametrize("ext", [[32, 32], [8, 8, 8], [256]])
def test_morton_copies(llama, oracle_mod, ext):
    for sk, dk in [(KINDS[0], KINDS[1]), (KINDS[2], KINDS[0]), (KINDS[1], KINDS[3])]:
        for lins in [("row", "morton"), ("morton", "col"), ("morton", "morton")]:
            _pair(llama, oracle_mod, W.PARTICLE7, ext, sk, lins[0], dk, lins[1],
                  paths=("auto", "naive", "permute", "transpose"))


def test_split_linearised(llama, oracle_mod):
    ext = [16, 16]
    _pair(llama, oracle_mod, W.PARTICLE7, ext, W.resolve_spec("split_p7"), "morton", ("aos", 1, False), "row")
    _pair(llama, oracle_mod, W.PARTICLE7, ext, ("soa_sb", 1, False), "col", W.resolve_spec("split_p7"), "col",
          paths=("auto", "naive", "permute"))


@pytest.mark.parametrize("src,dst", [("aos", "aos_aligned"), ("soa_mb", "aosoa8"), ("split_pos", "soa_sb")])
def test_traced_copy(llama, oracle_mod, src, dst):
    n = 1037
    schema = W.LISTING1
    sm = llama.Mapping.from_spec(schema, [n], W.resolve_spec(src)).traced(fields=True, bytes=True)
    dm = llama.Mapping.from_spec(schema, [n], W.resolve_spec(dst)).traced(fields=True, bytes=True)
    so = oracle_mod.mapping_from_spec(schema, [n], W.resolve_spec(src))
    do = oracle_mod.mapping_from_spec(schema, [n], W.resolve_spec(dst))
    sb = sm.alloc("cuda")
    llama.generate(sm, sb, 4)
    exp, sh, dh, sheat, dheat = oracle_mod.copy_counted(so, oracle_mod.make_view(so, 4), do)
    db = dm.alloc("cuda")
    assert llama.plan(sm, dm)["path"] == "naive"
    with pytest.raises(llama.LlamaError, match="UNSUPPORTED"):
        llama.copy(sm, sb, dm, db, path="permute")
    llama.copy(sm, sb, dm, db)
    torch.cuda.synchronize()
    for j, t in enumerate(db):
        assert np.array_equal(t.cpu().numpy(), exp[j])
    assert sm.field_hits() == [int(x) for x in sh]
    assert dm.field_hits() == [int(x) for x in dh]
    for b in range(sm.blob_count):
        assert np.array_equal(sm.byte_hits(b), sheat[b][:sm.blob_sizes()[b]])
    for b in range(dm.blob_count):
        assert np.array_equal(dm.byte_hits(b), dheat[b][:dm.blob_sizes()[b]])
    llama.copy(sm, sb, dm, db)  # counters accumulate ...
    torch.cuda.synchronize()
    assert dm.field_hits() == [2 * int(x) for x in dh]
    dm.reset_trace()  # ... until reset
    torch.cuda.synchronize()
    assert dm.field_hits() == [0] * len(dh)


@pytest.mark.parametrize("name", ["aos", "soa_mb", "aosoa8", "split_p7"])
def test_traced_move(llama, oracle_mod, name):
    """each Pos.* and Vel.* counter == N, Mass == 0; S:319 heat."""
    n = 4099
    vals = W.particle_values(n, seed=6)
    om = oracle_mod.mapping_from_spec(W.PARTICLE7, [n], W.resolve_spec(name))
    ob = oracle_mod.copy(oracle_mod.Mapping(W.PARTICLE7, [n], "aos"),
                         [np.frombuffer(vals.tobytes(), np.uint8).copy()], om)
    dm = llama.Mapping.from_spec(W.PARTICLE7, [n], W.resolve_spec(name)).traced(fields=True, bytes=True)
    db = dm.alloc("cuda")
    for t, h in zip(db, ob):
        t.copy_(torch.from_numpy(h))
    hits, heat = oracle_mod.nbody_move_counted(om, ob, 1e-4)
    assert llama.nbody_move(dm, db, 1e-4) == "generic"
    torch.cuda.synchronize()
    for j, t in enumerate(db):
        assert np.array_equal(t.cpu().numpy(), ob[j])
    assert dm.field_hits() == [int(x) for x in hits] == [n] * 6 + [0]
    for b in range(dm.blob_count):
        assert np.array_equal(dm.byte_hits(b), heat[b][:dm.blob_sizes()[b]])


@pytest.mark.parametrize("lins", [("row", "col"), ("col", "morton"), ("morton", "row")])
def test_raw_aos_tiles(llama, oracle_mod, lins):
    """Full 32x32 tiles with plain AoS on both sides take the raw 16-byte
    vector path (Particle7, packed and aligned Listing1 with padding)."""
    for schema, ext in ((W.PARTICLE7, [64, 64]), (W.LISTING1, [64, 64])):
        for sk, dk in (((("aos", 1, False)), ("aos", 1, True)), (("aos", 1, True), ("aos", 1, False)),
                       (("aos", 1, False), ("aos", 1, False))):
            _pair(llama, oracle_mod, schema, ext, sk, lins[0], dk, lins[1], paths=("auto", "naive"))


@pytest.mark.parametrize("knobs", [{"transpose_linear": 0}, {"transpose_raw1": 0},
                                   {"transpose_fixed": 0}, {"transpose_table": 0},
                                   {"transpose_raw_typed": 0},
                                   {"transpose_raw": 0}, {}])
def test_transpose_variants(llama, oracle_mod, knobs):
    """Every k_transpose2d instantiation: linear sides (one multiply-add per
    element) or the block / lane split, a raw AoS side next to an element-wise
    side, raw on both sides or none, the two-leaf pass for one 4-byte leaf
    size; full and ragged tiles, 4- and mixed-size leaves, AoSoA sides (not
    linear)."""
    for schema, ext in ((W.PARTICLE7, [64, 96]), (W.LISTING1, [70, 45]), (W.PARTICLE7, [64, 64])):
        for sk, dk in ((("soa_mb", 1, False), ("aos", 1, False)), (("aos", 1, True), ("soa_sb", 1, True)),
                       (("aos", 1, False), ("aos", 1, True)), (("aosoa", 8, False), ("aos", 1, False)),
                       (("one", 1, True), ("soa_mb", 1, False))):
            for lins in (("morton", "col") if ext[0] == ext[1] else ("row", "col"), ("col", "row")):
                _pair(llama, oracle_mod, schema, ext, sk, lins[0], dk, lins[1], paths=("auto", "transpose"),
                      knobs=knobs)
