"""Seeded synthetic workload recipes shared by tests/ and bench.py.

This module holds only DATA (schema strings, extents, mapping-pair lists, seeds);
it contains none of the method's arithmetic and imports neither the product
package nor the oracle.  Both sides implement the same counter-based input
generator themselves (splitmix64 of seed ^ (i*K + k)).
"""

# Particle7: "7 floats"; field order Pos, Vel, Mass as in the
# n-body code.  DESIGN.md reading #11.
PARTICLE7 = "Particle{Pos{X:f32,Y:f32,Z:f32},Vel{X:f32,Y:f32,Z:f32},Mass:f32}"

# Listing 1: the paper's nested record with a static array.
LISTING1 = "Particle{Id:u16,Pos{X:f32,Y:f32},Mass:f64,Flags:bool[3]}"

# Vec of Listing 1.
VEC = "Vec{X:f32,Y:f32}"

# HEP100 stand-in for the CMS event record (P:775 is an internal dataset):
# 10 groups of 10 mixed leaves -> 100 leaves (20 f64, 30 f32, 10 i32, 20 i16,
# 20 bool); packed 380 B, aligned 480 B.  DESIGN.md reading #19.
_HEP_GROUP = "{pt:f32,eta:f32,phi:f32,mass:f64,charge:i16,pdgId:i32,nHits:i16,isGood:bool,isTight:bool,weight:f64}"
HEP100 = "Event{" + ",".join(f"G{g}{_HEP_GROUP}" for g in range(10)) + "}"

# A nesting discriminator (SURVEY §8(c) reading #3): flattened per-leaf
# alignment gives 16 B, C nested-struct rules would give 24 B.
OUTER = "Outer{A{d:f64,b:bool},c:bool}"

SCHEMAS = {"particle7": PARTICLE7, "listing1": LISTING1, "vec": VEC, "hep100": HEP100}

# Mapping descriptors: (kind, lanes, aligned).  CLI names follow S:341.
MAPPINGS = {
    "aos": ("aos", 1, False),            # packed AoS  (reading #10: "AoS" := packed)
    "aos_aligned": ("aos", 1, True),     # aligned AoS
    "soa_mb": ("soa_mb", 1, False),      # SoA multi-blob (reading #10: "SoA" := MB)
    "soa_sb": ("soa_sb", 1, False),      # SoA single-blob
    "soa_sb_aligned": ("soa_sb", 1, True),  # sub-array starts rounded up to the leaf size (reading #9)
    "aosoa4": ("aosoa", 4, False),
    "aosoa8": ("aosoa", 8, False),
    "aosoa32": ("aosoa", 32, False),
    "aosoa4_aligned": ("aosoa", 4, True),  # aligned offsets x L, aligned record size (reading #6)
    "one": ("one", 1, True),             # One: always the aligned record
}

# Split mappings, per schema: (leaves_a, part_a, part_b), where a
# part is a MAPPINGS name or a nested split of that part's leaves; leaves_a
# index the (sub-)record's DFS leaf list.
SPLITS = {
    # Listing-1 Particle, Pos -> SoA MB, the rest packed AoS
    "split_pos": ("listing1", ([1, 2], "soa_mb", "aos")),
    # Listing P:499-509 (MappingC): Pos -> SoA MB; of the rest {Id, Mass,
    # Flags[3]}, Mass -> One and {Id, Flags[3]} -> aligned AoS
    "mapping_c": ("listing1", ([1, 2], "soa_mb", ([1], "one", "aos_aligned"))),
    # Particle7: Pos -> SoA MB, {Vel, Mass} -> AoSoA8 (the hot/cold split of P:479)
    "split_p7": ("particle7", ([0, 1, 2], "soa_mb", "aosoa8")),
    # HEP100: the 4-momenta of all 10 objects -> SoA MB, the rest aligned AoS
    "split_hep": ("hep100", ([g * 10 + j for g in range(10) for j in range(4)], "soa_mb", "aos_aligned")),
}

SEEDS = (42, 1, 2)  # seed 42 default

# BASELINE.json configs.
C1 = dict(name="C1", schema="particle7", extents=(4096,), pairs=[("aos", "soa_mb")])
_C2_KINDS = ["aos", "soa_mb", "aosoa8", "aosoa32"]
C2 = dict(name="C2", schema="particle7", extents=(16_777_216,),
          pairs=[(a, b) for a in _C2_KINDS for b in _C2_KINDS])
C3 = dict(name="C3", schema="hep100", extents=(67_108_864,),
          pairs=[(a, b) for a in ("aos", "aos_aligned", "soa_mb")
                 for b in ("aos", "aos_aligned", "soa_mb") if a != b])
C4 = dict(name="C4", schema="listing1", extents=(8192, 8192), pairs=[("aosoa32", "soa_sb")])
C5 = dict(name="C5", schema="particle7", extents=(1 << 27,), pairs=[("aos", "soa_mb")])
CONFIGS = {"C1": C1, "C2": C2, "C3": C3, "C4": C4, "C5": C5}


def resolve_spec(spec):
    """A MAPPINGS name / split tree with MAPPINGS names -> the same tree with
    (kind, lanes, aligned) tuples at the leaves (no layout arithmetic)."""
    if isinstance(spec, str):
        if spec in SPLITS:
            return resolve_spec(SPLITS[spec][1])
        return MAPPINGS[spec]
    if len(spec) == 3 and isinstance(spec[0], str):
        return spec
    leaves_a, a, b = spec
    return (list(leaves_a), resolve_spec(a), resolve_spec(b))


# ------------------------------------------------------------- n-body (f3)
# Listing P:617-619: FP = float, TIMESTEP = 0.0001f.  Initial state (S:685,
# the paper gives none): Pos, Vel uniform in [-1, 1), Mass in (0, 1], drawn
# from splitmix64 hashes as u = (h >> 40) * 2^-24, exact in f32.
NBODY_TIMESTEP = 0.0001
NBODY_MOVE_N = 1 << 28  # "Move with 256Mi particles"


def _splitmix64_np(x):
    import numpy as np
    z = (x + np.uint64(0x9E3779B97F4A7C15)).astype(np.uint64)
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)).astype(np.uint64)
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)).astype(np.uint64)
    return z ^ (z >> np.uint64(31))


def particle_values(n, seed=42, i0=0):
    """(n, 7) float32: Pos.X..Z, Vel.X..Z, Mass of particles i0 .. i0+n-1 (Particle7 leaf order)."""
    import numpy as np
    with np.errstate(over="ignore"):
        i = np.arange(i0, i0 + n, dtype=np.uint64)[:, None] * np.uint64(7) + np.arange(7, dtype=np.uint64)[None, :]
        h = _splitmix64_np(i ^ np.uint64(seed))
    u = (h >> np.uint64(40)).astype(np.float64) * 2.0 ** -24
    out = np.empty((n, 7), dtype=np.float32)
    out[:, :6] = (2.0 * u[:, :6] - 1.0).astype(np.float32)
    out[:, 6] = (1.0 - u[:, 6]).astype(np.float32)
    return out
