"""Parity oracle for the layout-aware copy -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference legs) may import this package.  The product package
(paper_2106_04284_b200) never imports it and shares no code with it.

Thin ctypes wrapper over oracle/oracle.c (plain C, see oracle.h for the
definitions and citations) plus the schema flattener in oracle/schema.py.
"""
import ctypes
import os
import subprocess

import numpy as np

from .schema import SCALAR_SIZE, SchemaError, flatten, leaf_sizes  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

KINDS = {"aos": 0, "soa_sb": 1, "soa_mb": 2, "aosoa": 3, "one": 4, "split": 5}
LINS = {"row": 0, "col": 1, "morton": 2}


def build(force=False):
    """Compiles oracle.c (g++/gcc -O3, OpenMP; no -march=native so the .so runs
    on any x86-64 host it travels to)."""
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-O3", "-std=c11", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
                           "-Wall", "-Wextra", "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, _LIB)
    return _LIB


class _CMapping(ctypes.Structure):
    pass


_CMapping._fields_ = [
        ("n_leaves", ctypes.c_int32),
        ("leaf_size", ctypes.POINTER(ctypes.c_int32)),
        ("rank", ctypes.c_int32),
        ("extents", ctypes.POINTER(ctypes.c_int64)),
        ("kind", ctypes.c_int32),
        ("lanes", ctypes.c_int64),
        ("aligned", ctypes.c_int32),
        ("inner_a", ctypes.POINTER(_CMapping)),
        ("inner_b", ctypes.POINTER(_CMapping)),
        ("leaves_a", ctypes.POINTER(ctypes.c_int32)),
        ("n_a", ctypes.c_int32),
        ("lin", ctypes.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER
        M = P(_CMapping)
        u8pp = P(P(ctypes.c_uint8))
        _lib.oracle_validate.argtypes = [M]
        _lib.oracle_record_count.argtypes = [M]
        _lib.oracle_record_count.restype = ctypes.c_int64
        _lib.oracle_linearize.argtypes = [M, P(ctypes.c_int64)]
        _lib.oracle_linearize.restype = ctypes.c_int64
        _lib.oracle_packed_offsets.argtypes = [M, P(ctypes.c_uint64)]
        _lib.oracle_packed_offsets.restype = ctypes.c_uint64
        _lib.oracle_aligned_offsets.argtypes = [M, P(ctypes.c_uint64)]
        _lib.oracle_aligned_offsets.restype = ctypes.c_uint64
        _lib.oracle_blob_count.argtypes = [M]
        _lib.oracle_blob_sizes.argtypes = [M, P(ctypes.c_uint64)]
        _lib.oracle_blob_nr_and_offset.argtypes = [M, ctypes.c_int64, ctypes.c_int32,
                                                   P(ctypes.c_int32), P(ctypes.c_uint64)]
        _lib.oracle_splitmix64.argtypes = [ctypes.c_uint64]
        _lib.oracle_splitmix64.restype = ctypes.c_uint64
        _lib.oracle_generate.argtypes = [M, u8pp, P(ctypes.c_uint64), ctypes.c_uint64,
                                         ctypes.c_int64, ctypes.c_int64]
        _lib.oracle_copy_range.argtypes = [M, u8pp, P(ctypes.c_uint64), M, u8pp,
                                           P(ctypes.c_uint64), ctypes.c_int64, ctypes.c_int64]
        _lib.oracle_copy.argtypes = [M, u8pp, M, u8pp, ctypes.c_int32]
        _lib.oracle_nbody_move.argtypes = [M, u8pp, P(ctypes.c_int32), P(ctypes.c_int32), ctypes.c_float,
                                           ctypes.c_int64, ctypes.c_int64]
        u32pp = P(P(ctypes.c_uint32))
        _lib.oracle_copy_counted.argtypes = [M, u8pp, M, u8pp, P(ctypes.c_uint64), P(ctypes.c_uint64), u32pp, u32pp]
        _lib.oracle_nbody_move_counted.argtypes = [M, u8pp, P(ctypes.c_int32), P(ctypes.c_int32), ctypes.c_float,
                                                   P(ctypes.c_uint64), u32pp]
    return _lib


def _u8pp(arrays):
    ptrs = (ctypes.POINTER(ctypes.c_uint8) * len(arrays))()
    for j, a in enumerate(arrays):
        assert a.dtype == np.uint8 and a.flags["C_CONTIGUOUS"]
        ptrs[j] = a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    return ptrs


def _u64p(vals):
    if vals is None:
        return None
    return (ctypes.c_uint64 * len(vals))(*[int(v) for v in vals])


class Mapping:
    """A mapping as the oracle sees it: flattened leaf sizes, extents, kind,
    AoSoA lanes and packed/aligned."""

    def __init__(self, schema, extents, kind, lanes=1, aligned=False, lin="row"):
        if isinstance(schema, str):
            self.schema = schema
            self.sizes = leaf_sizes(schema)
        else:
            self.schema = None
            self.sizes = [int(s) for s in schema]
        self.extents = [int(e) for e in extents]
        self.kind_name = kind
        self.lanes = int(lanes)
        self.aligned = bool(aligned)
        self.lin = lin
        self._sizes_c = (ctypes.c_int32 * len(self.sizes))(*self.sizes)
        self._ext_c = (ctypes.c_int64 * len(self.extents))(*self.extents)
        self.c = _CMapping(len(self.sizes), self._sizes_c, len(self.extents), self._ext_c,
                           KINDS[kind], self.lanes, int(self.aligned), None, None, None, 0, LINS[lin])
        if lib().oracle_validate(ctypes.byref(self.c)) != 0:
            raise ValueError(f"invalid oracle mapping {kind} {self.sizes} {self.extents}")

    @classmethod
    def split(cls, schema, leaves_a, a, b):
        """Split: the leaves of the full record listed in
        leaves_a (increasing) are mapped by a, the others by b; a and b are
        mappings of those sub-records over the same extents."""
        self = cls.__new__(cls)
        self.schema = schema if isinstance(schema, str) else None
        self.sizes = leaf_sizes(schema) if isinstance(schema, str) else [int(s) for s in schema]
        self.extents = list(a.extents)
        self.kind_name = "split"
        self.lanes = 1
        self.aligned = False
        self.lin = "row"
        self.inner = (a, b)
        self.leaves_a = [int(k) for k in leaves_a]
        self._sizes_c = (ctypes.c_int32 * len(self.sizes))(*self.sizes)
        self._ext_c = (ctypes.c_int64 * len(self.extents))(*self.extents)
        self._la_c = (ctypes.c_int32 * max(1, len(self.leaves_a)))(*self.leaves_a)
        self.c = _CMapping(len(self.sizes), self._sizes_c, len(self.extents), self._ext_c,
                           KINDS["split"], 1, 0, ctypes.pointer(a.c), ctypes.pointer(b.c),
                           self._la_c, len(self.leaves_a), 0)
        if lib().oracle_validate(ctypes.byref(self.c)) != 0:
            raise ValueError(f"invalid oracle split {self.sizes} leaves_a={self.leaves_a}")
        return self

    def __repr__(self):
        if self.kind_name == "split":
            return f"oracle.Split({self.leaves_a}: {self.inner[0]!r} | {self.inner[1]!r})"
        return f"oracle.Mapping({self.kind_name}, L={self.lanes}, aligned={self.aligned}, ext={self.extents})"

    @property
    def ref(self):
        return ctypes.byref(self.c)

    @property
    def n_leaves(self):
        return len(self.sizes)

    @property
    def record_count(self):
        return int(lib().oracle_record_count(self.ref))

    def linearize(self, index):
        idx = (ctypes.c_int64 * len(index))(*index)
        return int(lib().oracle_linearize(self.ref, idx))

    def packed_offsets(self):
        out = (ctypes.c_uint64 * self.n_leaves)()
        size = lib().oracle_packed_offsets(self.ref, out)
        return list(out), int(size)

    def aligned_offsets(self):
        out = (ctypes.c_uint64 * self.n_leaves)()
        size = lib().oracle_aligned_offsets(self.ref, out)
        return list(out), int(size)

    @property
    def blob_count(self):
        return int(lib().oracle_blob_count(self.ref))

    def blob_sizes(self):
        out = (ctypes.c_uint64 * self.blob_count)()
        lib().oracle_blob_sizes(self.ref, out)
        return [int(v) for v in out]

    def addr(self, i, k):
        b = ctypes.c_int32()
        o = ctypes.c_uint64()
        rc = lib().oracle_blob_nr_and_offset(self.ref, int(i), int(k), ctypes.byref(b), ctypes.byref(o))
        if rc != 0:
            raise IndexError((i, k))
        return int(b.value), int(o.value)

    def alloc(self, fill=0):
        return [np.full(s, fill, dtype=np.uint8) for s in self.blob_sizes()]


def mapping_from_spec(schema_or_sizes, extents, spec, lin="row"):
    """A mapping from a workloads.MAPPINGS tuple (kind, lanes, aligned) or a
    split tree (leaves_a, part_a, part_b) whose parts are such tuples or trees
    (P:479-481); `resolve` names are looked up by the caller."""
    sizes = leaf_sizes(schema_or_sizes) if isinstance(schema_or_sizes, str) else list(schema_or_sizes)
    if len(spec) == 3 and isinstance(spec[0], str):
        kind, lanes, aligned = spec
        return Mapping(sizes, extents, kind, lanes, aligned, lin)
    leaves_a, spec_a, spec_b = spec
    sel = set(leaves_a)
    a = mapping_from_spec([sizes[k] for k in leaves_a], extents, spec_a, lin)
    b = mapping_from_spec([sizes[k] for k in range(len(sizes)) if k not in sel], extents, spec_b, lin)
    return Mapping.split(sizes, leaves_a, a, b)


def splitmix64(x):
    return int(lib().oracle_splitmix64(ctypes.c_uint64(x & 0xFFFFFFFFFFFFFFFF)))


def generate(m, blobs, seed, i0=0, i1=None, base=None):
    """Writes the seeded leaf bytes of records [i0,i1) through m's address
    function; padding bytes are left as they are."""
    if i1 is None:
        i1 = m.record_count
    lib().oracle_generate(m.ref, _u8pp(blobs), _u64p(base), ctypes.c_uint64(seed), int(i0), int(i1))


def make_view(m, seed, pad_fill=0):
    blobs = m.alloc(pad_fill)
    generate(m, blobs, seed)
    return blobs


def copy(src, src_blobs, dst, dst_blobs=None, nthreads=1):
    """Whole-view naive copy; dst padding := 0.  Returns dst blobs."""
    if dst_blobs is None:
        dst_blobs = dst.alloc()
    rc = lib().oracle_copy(src.ref, _u8pp(src_blobs), dst.ref, _u8pp(dst_blobs), int(nthreads))
    if rc != 0:
        raise ValueError(f"oracle_copy failed rc={rc}")
    return dst_blobs


def copy_range(src, src_blobs, src_base, dst, dst_blobs, dst_base, i0, i1):
    rc = lib().oracle_copy_range(src.ref, _u8pp(src_blobs), _u64p(src_base), dst.ref,
                                 _u8pp(dst_blobs), _u64p(dst_base), int(i0), int(i1))
    if rc != 0:
        raise ValueError(f"oracle_copy_range failed rc={rc}")
    return rc


def nbody_move(m, blobs, dt, pos=(0, 1, 2), vel=(3, 4, 5), i0=0, i1=None):
    """n-body move (Listing P:643-645) in place on m's blobs: Pos += Vel * dt
    in f32 (one rounding: fmaf, reading #25).  Default leaves: Particle7's Pos.X..Z, Vel.X..Z."""
    if i1 is None:
        i1 = m.record_count
    p3 = (ctypes.c_int32 * 3)(*pos)
    v3 = (ctypes.c_int32 * 3)(*vel)
    rc = lib().oracle_nbody_move(m.ref, _u8pp(blobs), p3, v3, ctypes.c_float(dt), int(i0), int(i1))
    if rc != 0:
        raise ValueError(f"oracle_nbody_move failed rc={rc}")
    return blobs


def _u32pp(arrays):
    ptrs = (ctypes.POINTER(ctypes.c_uint32) * len(arrays))()
    for j, a in enumerate(arrays):
        assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]
        ptrs[j] = a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))
    return ptrs


def copy_counted(src, src_blobs, dst):
    """The copy with Trace / Heatmap counters on both sides:
    returns (dst_blobs, src_hits, dst_hits, src_heat, dst_heat)."""
    dst_blobs = dst.alloc()
    sh = np.zeros(src.n_leaves, np.uint64)
    dh = np.zeros(dst.n_leaves, np.uint64)
    sheat = [np.zeros(max(1, s), np.uint32) for s in src.blob_sizes()]
    dheat = [np.zeros(max(1, s), np.uint32) for s in dst.blob_sizes()]
    u64 = ctypes.POINTER(ctypes.c_uint64)
    rc = lib().oracle_copy_counted(src.ref, _u8pp(src_blobs), dst.ref, _u8pp(dst_blobs),
                                   sh.ctypes.data_as(u64), dh.ctypes.data_as(u64), _u32pp(sheat), _u32pp(dheat))
    if rc != 0:
        raise ValueError(f"oracle_copy_counted failed rc={rc}")
    return dst_blobs, sh, dh, sheat, dheat


def nbody_move_counted(m, blobs, dt, pos=(0, 1, 2), vel=(3, 4, 5)):
    """The move with Trace / Heatmap counters: returns (hits, heat)."""
    hits = np.zeros(m.n_leaves, np.uint64)
    heat = [np.zeros(max(1, s), np.uint32) for s in m.blob_sizes()]
    p3 = (ctypes.c_int32 * 3)(*pos)
    v3 = (ctypes.c_int32 * 3)(*vel)
    rc = lib().oracle_nbody_move_counted(m.ref, _u8pp(blobs), p3, v3, ctypes.c_float(dt),
                                         hits.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), _u32pp(heat))
    if rc != 0:
        raise ValueError(f"oracle_nbody_move_counted failed rc={rc}")
    return hits, heat
