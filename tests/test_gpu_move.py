"""GPU parity of the n-body move (llama_nbody_move_ex; Listing P:643-645)
against the oracle, bit for bit (reading #25), for every layout family and
forced path, with ragged tails; plus a sampled check at the paper's 256Mi
size."""
import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

DT = float(np.float32(W.NBODY_TIMESTEP))
LAYOUTS = ["aos", "aos_aligned", "soa_mb", "soa_sb", "aosoa4", "aosoa8", "aosoa32", "aosoa3", "split_p7"]
EXTRA = {"aosoa4": ("aosoa", 4, False), "aosoa3": ("aosoa", 3, False)}


@pytest.fixture(scope="module")
def llama():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_04284_b200 as m
    return m


def _spec(name):
    return EXTRA.get(name) or W.resolve_spec(name)


def _device_view(llama, oracle, name, n, vals, schema=W.PARTICLE7):
    """(device mapping, device blobs, oracle mapping, oracle blobs) holding `vals`."""
    so = oracle.Mapping(schema, [n], "aos")
    src = [np.frombuffer(vals.tobytes(), np.uint8).copy()]
    om = oracle.mapping_from_spec(schema, [n], _spec(name))
    ob = oracle.copy(so, src, om)
    dm = llama.Mapping.from_spec(schema, [n], _spec(name))
    db = dm.alloc("cuda")
    for t, h in zip(db, ob):
        t.copy_(torch.from_numpy(h))
    return dm, db, om, ob


@pytest.mark.parametrize("name", LAYOUTS)
@pytest.mark.parametrize("n", [1, 3, 4, 129, 4099, 100_003])
def test_move_parity(llama, oracle_mod, name, n):
    vals = W.particle_values(n, seed=42)
    om = oracle_mod.mapping_from_spec(W.PARTICLE7, [n], _spec(name))
    exp = oracle_mod.nbody_move(om, oracle_mod.copy(oracle_mod.Mapping(W.PARTICLE7, [n], "aos"),
                                                    [np.frombuffer(vals.tobytes(), np.uint8).copy()], om), DT)
    ran = set()
    for path in ("auto", "generic", "runs", "aos"):
        dm, db, _, _ = _device_view(llama, oracle_mod, name, n, vals)
        try:
            ran.add(llama.nbody_move(dm, db, DT, path=path))
        except llama.LlamaError as e:
            assert "UNSUPPORTED" in str(e) and path in ("runs", "aos")
            continue
        torch.cuda.synchronize()
        for j, t in enumerate(db):
            got = t.cpu().numpy()
            assert np.array_equal(got, exp[j]), f"{name} n={n} path={path} blob {j}"
    # the planner picks the layout's fast path
    auto = llama.nbody_move(*_device_view(llama, oracle_mod, name, n, vals)[:2], DT)
    want = {"aos": "aos", "aos_aligned": "aos", "aosoa3": "generic"}.get(name, "runs")
    if name == "soa_sb" and n % 4:  # sub-array starts n*4*k are not 16-byte aligned
        want = "generic"
    assert auto == want, (name, auto, ran)


def test_move_unaligned_generic(llama, oracle_mod):
    """Packed HEP100: f32 leaves at odd offsets -> the byte-wise generic path."""
    n = 1001
    leaves_p, leaves_v = (0, 1, 2), (10, 11, 12)  # G0.{pt,eta,phi}, G1.{pt,eta,phi}
    om = oracle_mod.Mapping(W.HEP100, [n], "aos")
    blobs = oracle_mod.make_view(om, 3)
    # finite floats in the six leaves (the byte generator may produce NaNs)
    vals = W.particle_values(n, seed=4)
    for c in range(3):
        for k, col in ((leaves_p[c], c), (leaves_v[c], 3 + c)):
            for i in range(n):
                b, o = om.addr(i, k)
                blobs[b][o:o + 4] = np.frombuffer(vals[i, col].tobytes(), np.uint8)
    exp = oracle_mod.nbody_move(om, [b.copy() for b in blobs], DT, pos=leaves_p, vel=leaves_v)
    dm = llama.Mapping(W.HEP100, [n], "aos")
    db = dm.alloc("cuda")
    for t, h in zip(db, blobs):
        t.copy_(torch.from_numpy(h))
    assert llama.nbody_move(dm, db, DT, pos=leaves_p, vel=leaves_v) == "generic"
    torch.cuda.synchronize()
    assert np.array_equal(db[0].cpu().numpy(), exp[0])


def test_move_errors(llama):
    m = llama.Mapping(W.LISTING1, [8])
    b = m.alloc("cuda")
    with pytest.raises(llama.LlamaError, match="INVALID_ARGUMENT"):
        llama.nbody_move(m, b, DT, pos=(1, 2, 3), vel=(1, 2, 0))  # Mass is 8 bytes
    p7 = llama.Mapping(W.PARTICLE7, [8])
    pb = p7.alloc("cuda")
    with pytest.raises(llama.LlamaError, match="INVALID_ARGUMENT"):
        llama.nbody_move(p7, pb, DT, pos=(0, 1, 2), vel=(2, 4, 5))
    one = llama.Mapping(W.PARTICLE7, [8], "one")
    with pytest.raises(llama.LlamaError, match="UNSUPPORTED"):
        llama.nbody_move(one, one.alloc("cuda"), DT)
    soa = llama.Mapping(W.PARTICLE7, [8], "soa_mb")
    with pytest.raises(llama.LlamaError, match="UNSUPPORTED"):
        llama.nbody_move(soa, soa.alloc("cuda"), DT, path="aos")


@pytest.fixture(scope="module")
def full_aos(llama):
    """The 256Mi particles as a packed AoS device blob."""
    n = W.NBODY_MOVE_N
    aos = llama.Mapping(W.PARTICLE7, [n], "aos")
    ab = aos.alloc("cuda")
    chunk = 1 << 24
    for i0 in range(0, n, chunk):
        v = W.particle_values(chunk, seed=42, i0=i0)
        ab[0][i0 * 28:(i0 + chunk) * 28].copy_(torch.from_numpy(np.frombuffer(v.tobytes(), np.uint8).copy()))
    yield aos, ab
    del ab
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["aos", "soa_mb", "aosoa32"])
def test_move_full_size_sampled(llama, oracle_mod, full_aos, name):
    """256Mi particles in the bench's launch configuration; windows at the
    start, middle and end checked against the oracle."""
    n = W.NBODY_MOVE_N
    aos, src = full_aos
    dm = llama.Mapping.from_spec(W.PARTICLE7, [n], _spec(name))
    db = dm.alloc("cuda")
    ab = aos.alloc("cuda")
    llama.copy(aos, src, dm, db)
    llama.nbody_move(dm, db, DT)
    llama.copy(dm, db, aos, ab)
    torch.cuda.synchronize()
    for a in (0, n // 2 - 777, n - 4099):
        w = 4099
        v = W.particle_values(w, seed=42, i0=a)
        om = oracle_mod.Mapping(W.PARTICLE7, [w], "aos")
        exp = oracle_mod.nbody_move(om, [np.frombuffer(v.tobytes(), np.uint8).copy()], DT)[0]
        got = ab[0][a * 28:(a + w) * 28].cpu().numpy()
        assert np.array_equal(got, exp), (name, a)
    del db, ab
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n", [127, 128 * 37 + 5, 300_001])
def test_move_aos_lsu_variant(llama, oracle_mod, n):
    """The warp-staged LSU AoS kernel (path AOS_LSU) against the oracle."""
    vals = W.particle_values(n, seed=8)
    om = oracle_mod.Mapping(W.PARTICLE7, [n], "aos")
    exp = oracle_mod.nbody_move(om, [np.frombuffer(vals.tobytes(), np.uint8).copy()], DT)
    dm, db, _, _ = _device_view(llama, oracle_mod, "aos", n, vals)
    assert llama.nbody_move(dm, db, DT, path="aos_lsu") == "aos_lsu"
    torch.cuda.synchronize()
    assert np.array_equal(db[0].cpu().numpy(), exp[0])


@pytest.mark.parametrize("cap", [4096, 1 << 20])
@pytest.mark.parametrize("name", ["aos", "soa_mb", "aosoa8"])
def test_move_staged_host(llama, oracle_mod, name, cap):
    """llama_nbody_move_staged on pinned host blobs: many slabs, a partial last one."""
    n = 10_007
    vals = W.particle_values(n, seed=12)
    om = oracle_mod.mapping_from_spec(W.PARTICLE7, [n], _spec(name))
    ob = oracle_mod.copy(oracle_mod.Mapping(W.PARTICLE7, [n], "aos"),
                         [np.frombuffer(vals.tobytes(), np.uint8).copy()], om)
    host = [torch.from_numpy(b.copy()).pin_memory() for b in ob]
    exp = oracle_mod.nbody_move(om, ob, DT)
    dm = llama.Mapping.from_spec(W.PARTICLE7, [n], _spec(name))
    llama.nbody_move_staged(llama.Stager(cap), dm, host, DT)
    torch.cuda.synchronize()
    for j, h in enumerate(host):
        assert np.array_equal(h.numpy(), exp[j]), (name, cap, j)
