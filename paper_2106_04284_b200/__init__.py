"""B200-native layout-aware copy (LLAMA, arXiv 2106.04284) -- Python binding.

Thin ctypes marshalling over the C ABI in include/llama_b200.h (the in-tree
libllama_b200.so, sm_100a kernels).  Every step of the copy runs in the
library's CUDA kernels; this module only converts arguments.  There is no CPU
fallback: if the library cannot be loaded, import fails loudly.

PyTorch provides device memory (torch.uint8 tensors as blobs) and
streams; it is plumbing, not the product.

    import paper_2106_04284_b200 as llama
    src = llama.Mapping("Particle{Pos{X:f32,Y:f32,Z:f32},Vel{X:f32,Y:f32,Z:f32},Mass:f32}",
                        [1 << 20], "aos")
    dst = llama.Mapping(src.schema, [1 << 20], "soa_mb")
    a, b = src.alloc("cuda"), dst.alloc("cuda")
    llama.generate(src, a, seed=42)
    llama.copy(src, a, dst, b)
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libllama_b200.so")

KINDS = {"aos": 0, "soa_sb": 1, "soa_mb": 2, "aosoa": 3, "one": 4}
LINS = {"row": 0, "col": 1, "morton": 2}
PATHS = {"auto": 0, "naive": 1, "blobcopy": 2, "run": 3, "permute": 4, "transpose": 5}
PATH_NAMES = {v: k for k, v in PATHS.items()}
STATUS = {0: "LLAMA_OK", -1: "LLAMA_ERR_INVALID_ARGUMENT", -2: "LLAMA_ERR_SHAPE_MISMATCH",
          -3: "LLAMA_ERR_RECORD_MISMATCH", -4: "LLAMA_ERR_UNSUPPORTED", -5: "LLAMA_ERR_ALIGNMENT",
          -6: "LLAMA_ERR_OVERLAP", -7: "LLAMA_ERR_CUDA", -8: "LLAMA_ERR_OOM"}

# Symbols declared in include/llama_b200.h (checked by tests/test_capi_host.py).
EXPORTS = ["llama_mapping_create", "llama_mapping_create_from_schema", "llama_mapping_create_split",
           "llama_mapping_with_linearizer", "llama_mapping_create_traced", "llama_trace_field_hits",
           "llama_trace_byte_hits", "llama_trace_reset",
           "llama_mapping_destroy",
           "llama_blob_count", "llama_blob_sizes", "llama_record_count", "llama_leaf_types",
           "llama_blob_nr_and_offset", "llama_copy", "llama_copy_ex", "llama_plan", "llama_plan_source",
           "llama_generate",
           "llama_launch_count", "llama_status_string", "llama_last_error_message", "llama_version",
           "llama_stager_create", "llama_stager_destroy", "llama_copy_staged", "llama_copy_staged_batch",
           "llama_nbody_move_staged", "llama_nbody_move",
           "llama_nbody_move_ex"]
MOVE_PATHS = {"auto": 0, "generic": 1, "runs": 2, "aos": 3, "aos_lsu": 4}
MOVE_PATH_NAMES = {v: k for k, v in MOVE_PATHS.items()}


class LlamaError(RuntimeError):
    def __init__(self, status, message):
        self.status = status
        self.status_name = STATUS.get(status, str(status))
        super().__init__(f"{self.status_name}: {message}")


class _Desc(ctypes.Structure):
    _fields_ = [("leaf_types", ctypes.POINTER(ctypes.c_int)), ("n_leaves", ctypes.c_int32),
                ("extents", ctypes.POINTER(ctypes.c_int64)), ("rank", ctypes.c_int32),
                ("kind", ctypes.c_int), ("lanes", ctypes.c_int64), ("aligned", ctypes.c_int32)]


class _Options(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int), ("tile_records", ctypes.c_int32),
                ("knobs", ctypes.POINTER(ctypes.c_int64))]


# llama_knob (include/llama_b200.h): explicit overrides of the planner's defaults
KNOBS = ["tile_bytes", "smem_budget", "stages", "dst_bufs", "ws_order", "no_tma", "permute_v1", "no_pdl",
         "word_mode", "direct", "direct_stages", "direct_async", "direct_phase", "direct_staging",
         "direct_chunks", "direct_mix", "bulk_chunk", "bulk_stages", "blobcopy_lsu", "transpose_raw",
         "transpose_linear", "transpose_raw1", "transpose_fixed", "transpose_table", "transpose_raw_typed",
         "jit", "jit_tile", "jit_stages", "jit_dst_bufs", "jit_chunks", "jit_lanes", "jit_soa_tma", "jit_pad", "jit_block", "jit_bmap", "jit_torder", "jit_dst_lsu", "jit_swizzle", "jit_group", "jit_ctas", "jit_ablate", "wide", "wide_group", "wide_stage", "wide_chunk4", "wide_torder", "wide_tma", "wide_async", "wide_aosoa_img"]


class _PlanInfo(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int), ("tile_records", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("moves", ctypes.c_int32), ("tma", ctypes.c_int32), ("src_bytes", ctypes.c_uint64),
                ("dst_bytes", ctypes.c_uint64), ("word_moves", ctypes.c_int32),
                ("direct", ctypes.c_int32), ("jit", ctypes.c_int32), ("wide", ctypes.c_int32)]


def _load():
    from . import _build
    if not _build.up_to_date():  # missing, or built from other sources: rebuild (fails loudly)
        _build.build()
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    vpp = P(ctypes.c_void_p)
    lib.llama_mapping_create.argtypes = [P(_Desc), P(ctypes.c_void_p)]
    lib.llama_mapping_create_from_schema.argtypes = [ctypes.c_char_p, P(ctypes.c_int64), ctypes.c_int32,
                                                     ctypes.c_int, ctypes.c_int64, ctypes.c_int32,
                                                     P(ctypes.c_void_p)]
    lib.llama_mapping_create_split.argtypes = [ctypes.c_void_p, ctypes.c_void_p, P(ctypes.c_int32),
                                                ctypes.c_int32, P(ctypes.c_void_p)]
    lib.llama_mapping_with_linearizer.argtypes = [ctypes.c_void_p, ctypes.c_int, P(ctypes.c_void_p)]
    lib.llama_mapping_create_traced.argtypes = [ctypes.c_void_p, ctypes.c_int32, P(ctypes.c_void_p)]
    lib.llama_trace_field_hits.argtypes = [ctypes.c_void_p, P(ctypes.c_uint64), ctypes.c_int32]
    lib.llama_trace_byte_hits.argtypes = [ctypes.c_void_p, ctypes.c_int32, P(ctypes.c_uint32), ctypes.c_uint64]
    lib.llama_trace_reset.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.llama_mapping_destroy.argtypes = [ctypes.c_void_p]
    lib.llama_mapping_destroy.restype = None
    lib.llama_blob_count.argtypes = [ctypes.c_void_p]
    lib.llama_blob_sizes.argtypes = [ctypes.c_void_p, P(ctypes.c_uint64), ctypes.c_int32]
    lib.llama_record_count.argtypes = [ctypes.c_void_p]
    lib.llama_record_count.restype = ctypes.c_int64
    lib.llama_leaf_types.argtypes = [ctypes.c_void_p, P(ctypes.c_int), ctypes.c_int32]
    lib.llama_blob_nr_and_offset.argtypes = [ctypes.c_void_p, P(ctypes.c_int64), ctypes.c_int32,
                                             P(ctypes.c_int32), P(ctypes.c_uint64)]
    lib.llama_copy.argtypes = [ctypes.c_void_p, vpp, ctypes.c_void_p, vpp, ctypes.c_void_p]
    lib.llama_copy_ex.argtypes = [ctypes.c_void_p, vpp, ctypes.c_void_p, vpp, ctypes.c_void_p, P(_Options)]
    lib.llama_plan.argtypes = [ctypes.c_void_p, ctypes.c_void_p, P(_Options), P(_PlanInfo)]
    lib.llama_plan_source.argtypes = [ctypes.c_void_p, ctypes.c_void_p, P(_Options), ctypes.c_char_p, ctypes.c_uint64,
                                      P(ctypes.c_uint64)]
    lib.llama_generate.argtypes = [ctypes.c_void_p, vpp, ctypes.c_uint64, ctypes.c_uint8, ctypes.c_void_p]
    lib.llama_stager_create.argtypes = [ctypes.c_uint64, P(ctypes.c_void_p)]
    lib.llama_stager_destroy.argtypes = [ctypes.c_void_p]
    lib.llama_stager_destroy.restype = None
    lib.llama_copy_staged.argtypes = [ctypes.c_void_p, ctypes.c_void_p, vpp, ctypes.c_void_p, vpp, ctypes.c_void_p]
    lib.llama_nbody_move_staged.argtypes = [ctypes.c_void_p, ctypes.c_void_p, vpp, P(ctypes.c_int32),
                                            P(ctypes.c_int32), ctypes.c_float, ctypes.c_void_p]
    lib.llama_copy_staged_batch.argtypes = [ctypes.c_void_p, ctypes.c_int32, P(ctypes.c_void_p), P(vpp),
                                            P(ctypes.c_void_p), P(vpp), ctypes.c_void_p]
    lib.llama_launch_count.restype = ctypes.c_uint64
    lib.llama_status_string.restype = ctypes.c_char_p
    lib.llama_nbody_move.argtypes = [ctypes.c_void_p, vpp, P(ctypes.c_int32), P(ctypes.c_int32), ctypes.c_float,
                                     ctypes.c_void_p]
    lib.llama_nbody_move_ex.argtypes = [ctypes.c_void_p, vpp, P(ctypes.c_int32), P(ctypes.c_int32), ctypes.c_float,
                                        ctypes.c_int, P(ctypes.c_int), ctypes.c_void_p]
    lib.llama_status_string.argtypes = [ctypes.c_int]
    lib.llama_last_error_message.restype = ctypes.c_char_p
    lib.llama_version.restype = ctypes.c_char_p
    return lib


_lib = _load()


def lib():
    return _lib


def _check(status):
    if status != 0:
        raise LlamaError(status, _lib.llama_last_error_message().decode())


class Mapping:
    """A mapping of a record dimension (schema string, S:122-126,
    or a list of llama_scalar leaf type codes) over array extents.
    kind: 'aos' | 'soa_sb' | 'soa_mb' | 'aosoa' | 'one'; splits come from
    Mapping.split / Mapping.from_spec."""

    def __init__(self, schema, extents, kind="aos", lanes=1, aligned=False):
        self.schema = schema
        self.extents = [int(e) for e in extents]
        self.kind = kind
        self.lanes = int(lanes)
        self.aligned = bool(aligned)
        self.lin = "row"
        if kind not in KINDS:
            raise ValueError(f"unknown mapping kind {kind!r}")
        ext = (ctypes.c_int64 * len(self.extents))(*self.extents)
        h = ctypes.c_void_p()
        if isinstance(schema, str):
            _check(_lib.llama_mapping_create_from_schema(schema.encode(), ext, len(self.extents), KINDS[kind],
                                                         self.lanes, int(self.aligned), ctypes.byref(h)))
        else:
            types = (ctypes.c_int * len(schema))(*[int(t) for t in schema])
            d = _Desc(types, len(schema), ext, len(self.extents), KINDS[kind], self.lanes, int(self.aligned))
            _check(_lib.llama_mapping_create(ctypes.byref(d), ctypes.byref(h)))
        self._h = h

    @classmethod
    def split(cls, a, b, leaves_a):
        """Split: leaves_a (increasing DFS leaf indices of the full
        record) are mapped by `a`, the others by `b`; blobs are a's then b's."""
        self = cls.__new__(cls)
        la = (ctypes.c_int32 * max(1, len(leaves_a)))(*[int(k) for k in leaves_a])
        h = ctypes.c_void_p()
        _check(_lib.llama_mapping_create_split(a.handle, b.handle, la, len(leaves_a), ctypes.byref(h)))
        self._h = h
        self.schema = None
        self.extents = list(a.extents)
        self.kind = "split"
        self.lanes = 1
        self.aligned = False
        self.lin = a.lin
        self.parts = (a, b, [int(k) for k in leaves_a])
        return self

    def with_linearizer(self, lin):
        """A copy with storage order lin: 'row' | 'col' | 'morton'."""
        c = self.__class__.__new__(self.__class__)
        h = ctypes.c_void_p()
        _check(_lib.llama_mapping_with_linearizer(self._h, LINS[lin], ctypes.byref(h)))
        c.__dict__.update({k: v for k, v in self.__dict__.items() if k != "_h"})
        c._h = h
        c.lin = lin
        return c

    def traced(self, fields=True, bytes=False):
        """Trace (per-leaf counters) and/or Heatmap (per-byte counters) of this
        mapping: a new mapping owning device counters."""
        c = self.__class__.__new__(self.__class__)
        h = ctypes.c_void_p()
        _check(_lib.llama_mapping_create_traced(self._h, (1 if fields else 0) | (2 if bytes else 0), ctypes.byref(h)))
        c.__dict__.update({k: v for k, v in self.__dict__.items() if k != "_h"})
        c._h = h
        return c

    def field_hits(self):
        n = self.leaf_count
        out = (ctypes.c_uint64 * n)()
        _check(_lib.llama_trace_field_hits(self._h, out, n))
        return [int(v) for v in out]

    def byte_hits(self, blob):
        import numpy as np
        n = self.blob_sizes()[blob]
        out = np.zeros(max(1, n), np.uint32)
        _check(_lib.llama_trace_byte_hits(self._h, int(blob), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), n))
        return out[:n]

    def reset_trace(self, stream=None):
        _check(_lib.llama_trace_reset(self._h, _stream(stream)))

    @classmethod
    def from_spec(cls, schema, extents, spec, lin="row"):
        """A mapping from (kind, lanes, aligned) or a split tree
        (leaves_a, spec_a, spec_b) (argument marshalling: the parts' leaf
        type lists are selected from the full record's)."""
        if len(spec) == 3 and isinstance(spec[0], str):
            kind, lanes, aligned = spec
            m = cls(schema, extents, kind, lanes, aligned)
            return m if lin == "row" else m.with_linearizer(lin)
        types = schema if not isinstance(schema, str) else cls(schema, [0]).leaf_types()
        leaves_a, spec_a, spec_b = spec
        sel = set(int(k) for k in leaves_a)
        a = cls.from_spec([types[k] for k in sorted(sel)], extents, spec_a, lin)
        b = cls.from_spec([t for k, t in enumerate(types) if k not in sel], extents, spec_b, lin)
        return cls.split(a, b, sorted(sel))

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.llama_mapping_destroy(h)
            self._h = None

    def __repr__(self):
        if self.kind == "split":
            return f"Mapping(split {self.parts[2]}: {self.parts[0]!r} | {self.parts[1]!r})"
        return f"Mapping({self.kind}, lanes={self.lanes}, aligned={self.aligned}, extents={self.extents})"

    @property
    def blob_count(self):
        return int(_lib.llama_blob_count(self._h))

    def blob_sizes(self):
        n = self.blob_count
        out = (ctypes.c_uint64 * n)()
        _check(_lib.llama_blob_sizes(self._h, out, n))
        return [int(v) for v in out]

    @property
    def record_count(self):
        return int(_lib.llama_record_count(self._h))

    @property
    def leaf_count(self):
        return int(_lib.llama_leaf_types(self._h, None, 0))

    def leaf_types(self):
        n = self.leaf_count
        out = (ctypes.c_int * n)()
        _lib.llama_leaf_types(self._h, out, n)
        return list(out)

    def blob_nr_and_offset(self, index, leaf):
        if isinstance(index, int):
            index = [index]
        idx = (ctypes.c_int64 * len(index))(*[int(i) for i in index])
        b = ctypes.c_int32()
        o = ctypes.c_uint64()
        _check(_lib.llama_blob_nr_and_offset(self._h, idx, int(leaf), ctypes.byref(b), ctypes.byref(o)))
        return int(b.value), int(o.value)

    def footprint(self):
        return sum(self.blob_sizes())

    def alloc(self, device="cuda"):
        """One torch.uint8 tensor per blob (torch allocations are >= 256-B aligned)."""
        import torch
        return [torch.empty(max(s, 1), dtype=torch.uint8, device=device)[:s] if s else
                torch.empty(16, dtype=torch.uint8, device=device) for s in self.blob_sizes()]


class Stager:
    """Device staging memory + streams for llama_copy_staged:
    slab_bytes per side per buffer (3 buffers x 2 sides), 0 = 64 MiB."""

    def __init__(self, slab_bytes=0):
        h = ctypes.c_void_p()
        _check(_lib.llama_stager_create(int(slab_bytes), ctypes.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.llama_stager_destroy(h)
            self._h = None


def _ptrs(blobs, sizes, what, device_only=True):
    if len(blobs) < len(sizes):
        raise LlamaError(-1, f"{what}: {len(sizes)} blobs needed, {len(blobs)} given")
    arr = (ctypes.c_void_p * max(1, len(blobs)))()
    for j, b in enumerate(blobs):
        if isinstance(b, int):
            arr[j] = b
            continue
        if j < len(sizes) and b.numel() * b.element_size() < sizes[j]:
            raise LlamaError(-1, f"{what}[{j}] holds {b.numel() * b.element_size()} bytes, needs {sizes[j]}")
        if device_only and not b.is_cuda:
            raise LlamaError(-1, f"{what}[{j}] is not a CUDA tensor")
        arr[j] = b.data_ptr()
    return arr


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _options(path, tile_records, knobs=None):
    opt = _Options(PATHS[path or "auto"], int(tile_records), None)
    if knobs:
        vals = [-1] * len(KNOBS)
        for k, v in knobs.items():
            vals[KNOBS.index(k)] = int(v)
        opt._keep = (ctypes.c_int64 * len(KNOBS))(*vals)
        opt.knobs = opt._keep
    return opt


def copy(src_map, src_blobs, dst_map, dst_blobs, stream=None, path=None, tile_records=0, knobs=None):
    """The layout-aware copy (llama_copy / llama_copy_ex), enqueued on `stream`
    (default: torch's current stream).  knobs: {name: value} overrides of the
    planner's tuning defaults (KNOBS)."""
    s = _ptrs(src_blobs, src_map.blob_sizes(), "src_blobs")
    d = _ptrs(dst_blobs, dst_map.blob_sizes(), "dst_blobs")
    opt = _options(path, tile_records, knobs)
    _check(_lib.llama_copy_ex(src_map.handle, s, dst_map.handle, d, _stream(stream), ctypes.byref(opt)))


def copy_staged(stager, src_map, src_blobs, dst_map, dst_blobs, stream=None):
    """Staged copy between host (pinned) and/or device blobs (llama_copy_staged):
    slab DMA in, relayout on the device, DMA out, overlapped on three streams."""
    s = _ptrs(src_blobs, src_map.blob_sizes(), "src_blobs", device_only=False)
    d = _ptrs(dst_blobs, dst_map.blob_sizes(), "dst_blobs", device_only=False)
    _check(_lib.llama_copy_staged(stager.handle, src_map.handle, s, dst_map.handle, d, _stream(stream)))



def copy_staged_batch(stager, copies, stream=None):
    """Several staged copies as one pipeline (llama_copy_staged_batch):
    copies = [(src_map, src_blobs, dst_map, dst_blobs), ...]."""
    n = len(copies)
    vp = ctypes.POINTER(ctypes.c_void_p)
    sm = (ctypes.c_void_p * n)(*[c[0].handle for c in copies])
    dm = (ctypes.c_void_p * n)(*[c[2].handle for c in copies])
    keep = [(_ptrs(c[1], c[0].blob_sizes(), "src_blobs", device_only=False),
             _ptrs(c[3], c[2].blob_sizes(), "dst_blobs", device_only=False)) for c in copies]
    sb = (vp * n)(*[ctypes.cast(k[0], vp) for k in keep])
    db = (vp * n)(*[ctypes.cast(k[1], vp) for k in keep])
    _check(_lib.llama_copy_staged_batch(stager.handle, n, sm, sb, dm, db, _stream(stream)))

def plan(src_map, dst_map, path=None, tile_records=0, knobs=None):
    """The planner's decision for a pair (no device work)."""
    info = _PlanInfo()
    opt = _options(path, tile_records, knobs)
    _check(_lib.llama_plan(src_map.handle, dst_map.handle, ctypes.byref(opt), ctypes.byref(info)))
    return {"path": PATH_NAMES[info.path], "tile_records": info.tile_records, "smem_bytes": info.smem_bytes,
            "moves": info.moves, "tma": bool(info.tma), "src_bytes": int(info.src_bytes),
            "dst_bytes": int(info.dst_bytes), "word_moves": int(info.word_moves), "direct": bool(info.direct),
            "jit": bool(info.jit), "wide": bool(info.wide)}


def plan_source(src_map, dst_map, path=None, tile_records=0, knobs=None):
    """The generated CUDA source of the pair's plan-time specialised kernel."""
    opt = _options(path, tile_records, knobs)
    n = ctypes.c_uint64(0)
    _check(_lib.llama_plan_source(src_map.handle, dst_map.handle, ctypes.byref(opt), None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    _check(_lib.llama_plan_source(src_map.handle, dst_map.handle, ctypes.byref(opt), buf, n.value + 1, None))
    return buf.value.decode()


def generate(m, blobs, seed=42, pad_byte=0, stream=None):
    """Seeded synthetic input (llama_generate): padding := pad_byte, leaf bytes
    from splitmix64(seed ^ (i*K + k))."""
    p = _ptrs(blobs, m.blob_sizes(), "blobs")
    _check(_lib.llama_generate(m.handle, p, ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), int(pad_byte) & 0xFF,
                               _stream(stream)))


def launch_count():
    """Kernels launched by the library in this process."""
    return int(_lib.llama_launch_count())


def version():
    return _lib.llama_version().decode()


def nbody_move(m, blobs, dt, pos=(0, 1, 2), vel=(3, 4, 5), path="auto", stream=None):
    """n-body move in place (llama_nbody_move_ex; Listing P:643-645):
    Pos += Vel * dt in f32 on device blobs.  Default leaves: Particle7's
    Pos.X..Z and Vel.X..Z.  Returns the path that ran."""
    ptrs = _ptrs(blobs, m.blob_sizes(), "blobs")
    p3 = (ctypes.c_int32 * 3)(*pos)
    v3 = (ctypes.c_int32 * 3)(*vel)
    used = ctypes.c_int(0)
    _check(_lib.llama_nbody_move_ex(m.handle, ptrs, p3, v3, ctypes.c_float(dt), MOVE_PATHS[path],
                                    ctypes.byref(used), _stream(stream)))
    return MOVE_PATH_NAMES[used.value]


def nbody_move_staged(stager, m, blobs, dt, pos=(0, 1, 2), vel=(3, 4, 5), stream=None):
    """n-body move of a view in host (pinned) or device memory through the
    stager's slab pipeline (llama_nbody_move_staged)."""
    ptrs = _ptrs(blobs, m.blob_sizes(), "blobs", device_only=False)
    p3 = (ctypes.c_int32 * 3)(*pos)
    v3 = (ctypes.c_int32 * 3)(*vel)
    _check(_lib.llama_nbody_move_staged(stager.handle, m.handle, ptrs, p3, v3, ctypes.c_float(dt), _stream(stream)))
