"""Pins of the oracle's n-body move (Listing P:643-645): the exact
value p + v*dt rounded ONCE to f32 (reading #25: the paper's builds contract
the multiply-add, -ffast-math -mfma P:593, nvcc --use_fast_math P:597),
computed here in exact rational arithmetic; closed forms, untouched bytes,
and layout commutation."""
from fractions import Fraction

import numpy as np
import pytest

import workloads as W

SPECS = ["aos", "soa_mb", "soa_sb", "aosoa8", "aosoa32", "split_p7"]
DT = np.float32(W.NBODY_TIMESTEP)


def _view(oracle, name, n, values):
    """The particles `values` ((n,7) f32) in mapping `name` (oracle copy from packed AoS)."""
    aos = oracle.Mapping(W.PARTICLE7, [n], "aos")
    m = oracle.mapping_from_spec(W.PARTICLE7, [n], W.resolve_spec(name))
    return m, oracle.copy(aos, [np.frombuffer(values.tobytes(), np.uint8).copy()], m)


def _values(oracle, m, blobs):
    aos = oracle.Mapping(W.PARTICLE7, [m.record_count], "aos")
    return np.frombuffer(oracle.copy(m, blobs, aos)[0].tobytes(), np.float32).reshape(-1, 7)


def round_f32(q):
    """The f32 nearest to the rational q, ties to even (IEEE 754 round to
    nearest), decided exactly: candidates around float(q), compared as
    Fractions."""
    f = np.float32(float(q))
    cands = {f, np.nextafter(f, np.float32(np.inf)), np.nextafter(f, np.float32(-np.inf))}
    cands = [c for c in cands if np.isfinite(c)]
    best = min(abs(Fraction(float(c)) - q) for c in cands)
    near = [c for c in cands if abs(Fraction(float(c)) - q) == best]
    if len(near) > 1:  # a tie: the even significand
        near = [c for c in near if (int(np.array(c, np.float32).view(np.uint32)) & 1) == 0]
    return np.float32(near[0])


def fused_ref(p, v, dt):
    """p + v*dt, exact, then one rounding to f32."""
    return round_f32(Fraction(float(p)) + Fraction(float(v)) * Fraction(float(dt)))


def test_round_f32_helper():
    # exact values stay; halfway cases go to the even neighbour
    assert round_f32(Fraction(3, 4)) == np.float32(0.75)
    one_up = np.nextafter(np.float32(1), np.float32(2))
    assert round_f32(Fraction(1) + Fraction(1, 2 ** 24)) == np.float32(1)  # tie -> even (1.0)
    assert round_f32(Fraction(1) + Fraction(3, 2 ** 24)) == np.nextafter(one_up, np.float32(2))  # tie -> even
    assert round_f32(Fraction(1) + Fraction(1, 2 ** 23) - Fraction(1, 2 ** 40)) == one_up


@pytest.mark.parametrize("name", SPECS)
@pytest.mark.parametrize("n", [1, 33, 1000])
def test_move_equals_exact_single_rounding(oracle_mod, name, n):
    vals = W.particle_values(n, seed=42)
    m, blobs = _view(oracle_mod, name, n, vals)
    oracle_mod.nbody_move(m, blobs, float(DT))
    got = _values(oracle_mod, m, blobs)
    exp = vals.copy()
    for i in range(n):
        for c in range(3):
            exp[i, c] = fused_ref(vals[i, c], vals[i, 3 + c], DT)
    assert got.tobytes() == exp.tobytes()


def test_single_rounding_reading(oracle_mod):
    """Reading #25: one rounding (fused multiply-add, P:593 -ffast-math -mfma,
    P:597 --use_fast_math).  (1 + 2^-12)^2 - 1 = 2^-11 + 2^-24 exactly and is
    representable; two roundings would lose the 2^-24 term (the product alone
    rounds, tie to even, to 1 + 2^-11)."""
    e = np.float32(1 + 2.0 ** -12)
    vals = np.zeros((1, 7), np.float32)
    vals[0, 0] = -1.0
    vals[0, 3] = e
    m, blobs = _view(oracle_mod, "soa_mb", 1, vals)
    oracle_mod.nbody_move(m, blobs, float(e))
    got = _values(oracle_mod, m, blobs)[0, 0]
    assert float(np.float32(2.0 ** -11 + 2.0 ** -24)) == 2.0 ** -11 + 2.0 ** -24
    assert got == np.float32(2.0 ** -11 + 2.0 ** -24)    # one rounding (exact here)
    assert got != np.float32(2.0 ** -11)                 # what two roundings would give


def test_closed_forms(oracle_mod):
    """S:655 Vel = 0 -> Pos unchanged; dt = 0 -> nothing changes; dt = 1/2 on
    small integers is exact: Pos + Vel/2."""
    n = 64
    vals = W.particle_values(n, seed=3)
    v0 = vals.copy()
    v0[:, 3:6] = 0
    m, blobs = _view(oracle_mod, "aosoa8", n, v0)
    before = [b.copy() for b in blobs]
    oracle_mod.nbody_move(m, blobs, 0.25)
    assert all((a == b).all() for a, b in zip(before, blobs))
    m, blobs = _view(oracle_mod, "aos", n, vals)
    before = [b.copy() for b in blobs]
    oracle_mod.nbody_move(m, blobs, 0.0)
    assert all((a == b).all() for a, b in zip(before, blobs))
    ints = np.arange(n * 7, dtype=np.float32).reshape(n, 7) - 100
    m, blobs = _view(oracle_mod, "soa_sb", n, ints)
    oracle_mod.nbody_move(m, blobs, 0.5)
    got = _values(oracle_mod, m, blobs)
    assert (got[:, :3] == ints[:, :3] + ints[:, 3:6] / 2).all()
    assert (got[:, 3:] == ints[:, 3:]).all()


@pytest.mark.parametrize("name", ["aos_aligned", "aosoa8"])
def test_only_pos_bytes_change(oracle_mod, name):
    """Vel, Mass and padding bytes are never written ("Mass untouched")."""
    n = 13  # AoSoA8 tail block: 3 padding lanes
    vals = W.particle_values(n, seed=5)
    m, blobs = _view(oracle_mod, name, n, vals)
    before = [b.copy() for b in blobs]
    oracle_mod.nbody_move(m, blobs, float(DT))
    pos_bytes = set()
    for i in range(n):
        for k in range(3):
            b, o = m.addr(i, k)
            pos_bytes.update((b, o + j) for j in range(4))
    for bi, (a, b) in enumerate(zip(before, blobs)):
        diff = np.nonzero(a != b)[0]
        assert all((bi, int(o)) in pos_bytes for o in diff)


@pytest.mark.parametrize("a,b", [("aos", "soa_mb"), ("aosoa8", "split_p7"), ("soa_sb", "aosoa32")])
def test_move_commutes_with_copy(oracle_mod, a, b):
    n = 257
    vals = W.particle_values(n, seed=9)
    ma, ba = _view(oracle_mod, a, n, vals)
    mb = oracle_mod.mapping_from_spec(W.PARTICLE7, [n], W.resolve_spec(b))
    x = oracle_mod.copy(ma, oracle_mod.nbody_move(ma, [t.copy() for t in ba], float(DT)), mb)
    y = oracle_mod.nbody_move(mb, oracle_mod.copy(ma, ba, mb), float(DT))
    assert all((p == q).all() for p, q in zip(x, y))


def test_aos_useful_bandwidth_fraction():
    """of 7 floats 6 are read and 3 written; at cache-line granularity an
    AoS moves 7 + 7, so 1 - (1 + 4)/(7 + 7) = 64.3% is useful; the per-particle
    byte counts the roofline uses give the same ratio."""
    useful = (6 + 3) * 4
    aos_traffic = (7 + 7) * 4
    assert abs(1 - (1 + 4) / (7 + 7) - 0.642857) < 1e-6
    assert abs(useful / aos_traffic - (1 - (1 + 4) / (7 + 7))) < 1e-12


def test_move_validation(oracle_mod):
    m = oracle_mod.Mapping(W.LISTING1, [4], "aos")  # leaf 3 (Mass) is 8 bytes
    with pytest.raises(ValueError):
        oracle_mod.nbody_move(m, m.alloc(), 0.1, pos=(1, 2, 3), vel=(1, 2, 0))
