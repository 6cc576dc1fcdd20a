/*
 * llama_b200.h -- C ABI of the B200-native layout-aware copy.
 *
 * Implements the hot path of LLAMA (Gruber et al., arXiv 2106.04284): copying
 * an N-dimensional array of nested records between two *views* of the same
 * data space that use different *mappings* (§3.1 "layout-aware copy
 * operations between instances of the same data space but with different
 * mappings"; §3.9; §4.2).
 *
 * Citation convention: P:n = PAPER.md line n, S:n = SPEC.md line n (the
 * reference texts of the paper).
 *
 * Conventions for every function:
 *   - Thread safety: all functions are thread-safe (plan and launch caches
 *     are mutex-protected), except that one llama_stager runs one staged call
 *     at a time.  Mappings are immutable after creation and may be shared
 *     between threads and devices.
 *   - Ownership: the library owns llama_mapping objects (create/destroy).  The
 *     caller owns all blob memory ("LLAMA ... function[s] orthogonally to
 *     memory allocation"); the library never allocates or frees blobs.  Arrays
 *     passed in (descriptors, blob pointer arrays, sizes) are read during the
 *     call only.
 *   - Errors: a function returns LLAMA_OK or a negative llama_status.  All
 *     validation happens synchronously before any device work is enqueued,
 *     and a failed call does no partial work.  llama_last_error_message()
 *     returns a thread-local description of the last failure.  No C++
 *     exception crosses this ABI.
 *   - Streams: `stream` is a cudaStream_t passed as void* (NULL = the legacy
 *     default stream) that belongs to the calling thread's current device.
 *     Device functions enqueue and return; ordering follows CUDA stream
 *     semantics.  Blobs must stay alive until the enqueued work completes.
 */
#ifndef LLAMA_B200_H
#define LLAMA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LLAMA_OK = 0,
  LLAMA_ERR_INVALID_ARGUMENT = -1, /* NULL pointer, bad enum, too few blobs, ... */
  LLAMA_ERR_SHAPE_MISMATCH = -2,   /* different array extents */
  LLAMA_ERR_RECORD_MISMATCH = -3,  /* different leaf type lists */
  LLAMA_ERR_UNSUPPORTED = -4,      /* beyond the implemented limits (see below) */
  LLAMA_ERR_ALIGNMENT = -5,        /* a blob base address not 16-byte aligned */
  LLAMA_ERR_OVERLAP = -6,          /* src and dst byte ranges overlap (in-situ is out of scope) */
  LLAMA_ERR_CUDA = -7,             /* a CUDA launch / runtime call failed */
  LLAMA_ERR_OOM = -8               /* host allocation failed */
} llama_status;

/* Leaf scalar types.  Size = alignment; bool is one
 * byte.  Leaf bytes are copied verbatim: no bool normalisation, no
 * floating-point canonicalisation (NaN payloads survive). */
typedef enum {
  LLAMA_BOOL = 0, LLAMA_I8, LLAMA_U8, LLAMA_I16, LLAMA_U16, LLAMA_I32, LLAMA_U32,
  LLAMA_I64, LLAMA_U64, LLAMA_F32, LLAMA_F64
} llama_scalar;

/* Mapping kinds. */
typedef enum {
  LLAMA_AOS = 0,             /* P:460-463 fields after each other, repeated per record */
  LLAMA_SOA_SINGLE_BLOB = 1, /* P:465-468 one sub-array per leaf, all in one blob */
  LLAMA_SOA_MULTI_BLOB = 2,  /* P:465-468 one blob per leaf ("SoA MB") */
  LLAMA_AOSOA = 3,           /* P:470-473 AoS of blocks that repeat each field L times */
  LLAMA_ONE = 4,             /* P:475-477 the whole array collapsed onto one (aligned) record */
  LLAMA_SPLIT = 5            /* P:479-481 composite, from llama_mapping_create_split only */
} llama_kind;

/* A mapping description (a mapping is configured on the array and
 * record dimensions).
 *   leaf_types/n_leaves: the record dimension flattened depth-first in
 *     declaration order, 1 <= n_leaves <= LLAMA_MAX_LEAVES.
 *   extents/rank: the array dimensions, row-major (last index fastest,
 *     P:414-416), 1 <= rank <= LLAMA_MAX_RANK, every extent >= 0.
 *   kind: see llama_kind.  lanes: AoSoA lane count L >= 1 (any L, not only
 *     powers of two; ignored for other kinds).
 *   aligned: 0 = tightly packed, 1 = each leaf at a multiple of its size and
 *     the record rounded up to the largest leaf.  For SoA
 *     single-blob, aligned=1 rounds each leaf sub-array start up to the leaf
 *     size (reading #9); for SoA multi-blob it has no effect. */
typedef struct {
  const llama_scalar* leaf_types;
  int32_t n_leaves;
  const int64_t* extents;
  int32_t rank;
  llama_kind kind;
  int64_t lanes;
  int32_t aligned;
} llama_mapping_desc;

#define LLAMA_MAX_LEAVES 128
#define LLAMA_MAX_RANK 8
#define LLAMA_MAX_BLOBS 128

typedef struct llama_mapping llama_mapping; /* opaque, immutable */

/* Creates a mapping.  *out receives a new mapping on LLAMA_OK.
 * Errors: INVALID_ARGUMENT (NULL, bad enum, extent < 0, lanes < 1),
 * UNSUPPORTED (n_leaves or rank beyond the limits, blob sizes overflowing 64
 * bits). */
llama_status llama_mapping_create(const llama_mapping_desc* desc, llama_mapping** out);

/* Convenience: parses a schema string in the grammar of S:122-126, e.g.
 * "Particle{Id:u16,Pos{X:f32,Y:f32},Mass:f64,Flags:bool[3]}" (Listing 1,
 * P:296-313); static arrays become n fields.  Same errors as
 * llama_mapping_create, plus INVALID_ARGUMENT on a malformed schema. */
llama_status llama_mapping_create_from_schema(const char* schema, const int64_t* extents,
                                              int32_t rank, llama_kind kind, int64_t lanes,
                                              int32_t aligned, llama_mapping** out);

/* Split mapping (Listing P:499-509): the leaves
 * leaves_a[0..n_a) (strictly increasing indices into the full record's DFS
 * leaf list) are mapped by `a`, the remaining leaves by `b`; a and b are
 * mappings of those sub-records (in leaf order) over the same extents.  The
 * split's blobs are a's blobs followed by b's.  a and b may themselves be
 * splits; they are copied, so they may be destroyed afterwards.
 * Errors: INVALID_ARGUMENT (NULL, bad leaf list, leaf count or extents that
 * do not add up, a and b linearised differently), UNSUPPORTED (more than
 * LLAMA_MAX_BLOBS blobs).  The split takes a's linearisation. */
llama_status llama_mapping_create_split(const llama_mapping* a, const llama_mapping* b, const int32_t* leaves_a,
                                        int32_t n_a, llama_mapping** out);

/* Linearisation of the array index into a storage position (P:140-142
 * "storage order ... row- or column-major ... Morton codes").
 * ROW_MAJOR (the default of every create call): last index fastest;
 * COL_MAJOR: first index fastest; MORTON: bit b of index[d] goes to bit
 * b*rank + (rank-1-d) (all extents equal powers of two; #26).
 * Data belongs to the array index: a copy between views of different
 * linearisations moves record (index) to record (index), i.e. it also
 * transposes / reorders (naive path only); views of equal linearisation use
 * every path.  llama_blob_nr_and_offset applies the linearisation. */
typedef enum { LLAMA_ROW_MAJOR = 0, LLAMA_COL_MAJOR = 1, LLAMA_MORTON = 2 } llama_linearizer;

/* A copy of `m` (any kind, splits included) with linearisation `lin`.
 * Errors: INVALID_ARGUMENT (NULL, bad lin, MORTON with unequal or
 * non-power-of-two extents). */
llama_status llama_mapping_with_linearizer(const llama_mapping* m, llama_linearizer lin, llama_mapping** out);

/* Instrumentation (#27): a traced mapping is
 * `inner` (copied) plus device counters owned by the new mapping, allocated
 * on the current device:
 *   LLAMA_TRACE_FIELDS  (Trace)   one uint64 counter per leaf
 *   LLAMA_TRACE_BYTES   (Heatmap) one uint32 counter per blob byte
 * (a bit mask; both may be set).  Every llama_copy / llama_nbody_move through
 * a traced view counts its address resolutions -- a copy resolves each
 * (record, leaf) once per side; the move resolves each Pos and Vel component
 * once per particle -- and therefore runs the element-wise kernels (copy:
 * NAIVE; move: GENERIC; forcing another path is UNSUPPORTED).  Counters
 * start at 0, accumulate over calls, and are read (synchronously, after all
 * work on the device) or reset (on `stream`) below.
 * Errors: INVALID_ARGUMENT, CUDA (allocation), OOM. */
typedef enum { LLAMA_TRACE_FIELDS = 1, LLAMA_TRACE_BYTES = 2 } llama_trace_kind;
llama_status llama_mapping_create_traced(const llama_mapping* inner, int32_t kinds, llama_mapping** out);
/* hits[k] for k < min(capacity, leaf count); INVALID_ARGUMENT if not traced with FIELDS. */
llama_status llama_trace_field_hits(const llama_mapping* m, uint64_t* hits, int32_t capacity);
/* counters of blob `blob` (its blob size many); INVALID_ARGUMENT if not traced with BYTES,
 * blob out of range or capacity below the blob size. */
llama_status llama_trace_byte_hits(const llama_mapping* m, int32_t blob, uint32_t* hits, uint64_t capacity);
llama_status llama_trace_reset(const llama_mapping* m, void* stream);

/* Destroys a mapping; NULL-safe.  Plans cached for pairs involving it are
 * released. */
void llama_mapping_destroy(llama_mapping* m);

/* Blob count ("a compile time blob count"): 1, or n_leaves for SoA MB.
 * Returns -1 for a NULL mapping. */
int32_t llama_blob_count(const llama_mapping* m);

/* Blob sizes in bytes.  Writes llama_blob_count(m) values into sizes;
 * capacity is the array length.  INVALID_ARGUMENT if capacity is too small. */
llama_status llama_blob_sizes(const llama_mapping* m, uint64_t* sizes, int32_t capacity);

/* Record count = product of the extents; -1 for a NULL mapping. */
int64_t llama_record_count(const llama_mapping* m);

/* Number of leaves; writes the leaf types into types[0..capacity) if non-NULL. */
int32_t llama_leaf_types(const llama_mapping* m, llama_scalar* types, int32_t capacity);

/* blobNrAndOffset: the blob number and byte offset of leaf `leaf` of
 * the record at the rank-dimensional `index`.  Host-side, for tests and tools.
 * INVALID_ARGUMENT on a NULL argument or an out-of-range index / leaf. */
llama_status llama_blob_nr_and_offset(const llama_mapping* m, const int64_t* index, int32_t leaf,
                                      int32_t* blob, uint64_t* offset);

/* The layout-aware copy.
 *   src_blobs: llama_blob_count(src_map) device pointers, each 16-byte aligned,
 *     each at least the corresponding blob size.  Never written.
 *   dst_blobs: llama_blob_count(dst_map) device (or peer-mapped) pointers,
 *     16-byte aligned.
 * Result: for every record i and leaf k the s_k bytes of the leaf land at the
 * destination mapping's blob/offset, bit-exactly; every destination byte in
 * [0, blob size) of every destination blob is written, padding bytes with 0
 * (reading #12).  Source padding never influences the result.
 * Errors (synchronous, before any launch): RECORD_MISMATCH, SHAPE_MISMATCH,
 * INVALID_ARGUMENT (NULL mapping/pointer array/pointer), ALIGNMENT, OVERLAP,
 * UNSUPPORTED (also: a destination that maps several records onto one
 * location, e.g. a One leaf with more than one record -- the result would
 * depend on the order of the writes); CUDA on a launch failure. */
llama_status llama_copy(const llama_mapping* src_map, void* const* src_blobs,
                        const llama_mapping* dst_map, void* const* dst_blobs, void* stream);

/* Copy paths. */
typedef enum {
  LLAMA_PATH_AUTO = 0,     /* planner's choice */
  LLAMA_PATH_NAIVE = 1,    /* element-wise: thread per record, leaf loop */
  LLAMA_PATH_BLOBCOPY = 2, /* identical layout without padding: raw blob copy */
  LLAMA_PATH_RUN = 3,      /* field-run copy: common contiguous runs >= 16 B */
  LLAMA_PATH_PERMUTE = 4,  /* TMA-staged tile permute through shared memory */
  LLAMA_PATH_TRANSPOSE = 5 /* 2-d views of different linearisations: record tiles through
                              shared memory, read in source and written in destination storage order --
                              the plan-time specialised JIT transpose (TY x 32 tiles), the 32x32 tile kernel,
                              or for records too wide for those (HEP100) the wide-record kernel
                              (AoS / AoSoA sides as tensor-map TMA box images, SoA sides element-wise) */
} llama_path;

/* Tuning knobs: explicit overrides of the planner's measured defaults (for
 * sweeps and ablations).  The library never reads
 * the environment: a plan depends only on the two mappings and the options,
 * and the plan cache keys on every knob value. */
typedef enum {
  LLAMA_KNOB_TILE_BYTES = 0,   /* PERMUTE: src + dst image bytes per tile (64 KB small records, 48 KB wide) */
  LLAMA_KNOB_SMEM_BUDGET,      /* PERMUTE: shared memory per CTA the ring may use (230 KB / 112 KB) */
  LLAMA_KNOB_STAGES,           /* PERMUTE: source stages 2..4 (4 small records, 2 wide) */
  LLAMA_KNOB_DST_BUFS,         /* PERMUTE: destination buffers 2..4 (3 small records, 2 wide) */
  LLAMA_KNOB_WS_ORDER,         /* PERMUTE: producer order 0 stores first / 1 release first / 2 refill first (2) */
  LLAMA_KNOB_NO_TMA,           /* PERMUTE: 1 = LSU segment copies (0) */
  LLAMA_KNOB_PERMUTE_V1,       /* PERMUTE: 1 = barrier-synchronised kernel (0) */
  LLAMA_KNOB_NO_PDL,           /* PERMUTE: 1 = no programmatic dependent launch (0) */
  LLAMA_KNOB_WORD_MODE,        /* PERMUTE: AoS <-> AoS word mode for wide records (1) */
  LLAMA_KNOB_DIRECT,           /* PERMUTE: direct AoS <-> SoA variant: 0 off, 1 many leaves, 2 any leaf count (1) */
  LLAMA_KNOB_DIRECT_STAGES,    /* direct: ring stages (3 AoS -> SoA, 2 SoA -> AoS) */
  LLAMA_KNOB_DIRECT_ASYNC,     /* direct SoA -> AoS: aligned 4- / 8-byte classes by cp.async (1) */
  LLAMA_KNOB_DIRECT_PHASE,     /* direct: compile-time word phases of misaligned classes (1) */
  LLAMA_KNOB_DIRECT_STAGING,   /* direct SoA -> AoS: misaligned 4- / 8-byte classes staged by cp.async (1) */
  LLAMA_KNOB_DIRECT_CHUNKS,    /* direct SoA -> AoS: 1- / 2-byte classes staged as 16-byte chunks (1) */
  LLAMA_KNOB_DIRECT_MIX,       /* direct: 4 leaves x 8 records per warp access for even word strides (1) */
  LLAMA_KNOB_BULK_CHUNK,       /* BLOBCOPY: TMA chunk bytes (65536) */
  LLAMA_KNOB_BULK_STAGES,      /* BLOBCOPY: TMA ring stages (3) */
  LLAMA_KNOB_BLOBCOPY_LSU,     /* BLOBCOPY: 1 = 16-byte LSU vector copy instead of TMA (0) */
  LLAMA_KNOB_TRANSPOSE_RAW,    /* TRANSPOSE: raw 16-byte AoS tiles (1) */
  LLAMA_KNOB_TRANSPOSE_LINEAR, /* TRANSPOSE: linear-side element addressing (1) */
  LLAMA_KNOB_TRANSPOSE_RAW1,   /* TRANSPOSE: one raw AoS side next to an element-wise side (1) */
  LLAMA_KNOB_TRANSPOSE_FIXED,  /* TRANSPOSE: two-leaf load pass for one 4- / 8-byte leaf size (1) */
  LLAMA_KNOB_TRANSPOSE_TABLE,  /* TRANSPOSE: per-CTA shared-memory leaf table (1) */
  LLAMA_KNOB_TRANSPOSE_RAW_TYPED, /* TRANSPOSE: typed 4-byte raw passes (1) */
  LLAMA_KNOB_JIT,              /* PERMUTE: plan-time specialised kernel (NVRTC): 0 off, 1 wide records (> 16
                                  leaves) and splits, 2 every eligible pair (1) */
  LLAMA_KNOB_JIT_TILE,         /* JIT: records per tile, 32 / 64 / 128 / 256 / 512 (<= 64 KB of images per tile) */
  LLAMA_KNOB_JIT_STAGES,       /* JIT: source stages 2..6 (3 while the ring fits 180 KB, else 2) */
  LLAMA_KNOB_JIT_DST_BUFS,     /* JIT: destination image buffers 2..4 (3 while <= 180 KB, else 2) */
  LLAMA_KNOB_JIT_CHUNKS,       /* JIT transpose: AoS source segments as 16-byte cp.async chunks (1) or TMA (0) */
  LLAMA_KNOB_JIT_LANES,        /* JIT transpose: lanes along x (0), y (1), Morton codes (2), 4 x 8 blocks (3);
                                  default: the SoA destination's order, else a Morton source's, else x */
  LLAMA_KNOB_JIT_SOA_TMA,      /* JIT permute: SoA destination leaves stored from registers (0), or staged in shared
                                  memory and TMA-stored per leaf (1) / stored as 16-byte chunks by the consumers
                                  (2; the default when every destination part is SoA) */
  LLAMA_KNOB_JIT_PAD,          /* JIT permute: shared-memory images of AoS parts whose record-group stride is a
                                  multiple of 32 bytes get a 16-byte pad per group (bank conflicts), moved as
                                  16-byte chunks instead of one TMA op: 0 never, 1 strides multiple of 128 B
                                  (1), 2 every even 16-byte multiple */
  LLAMA_KNOB_JIT_BLOCK,        /* JIT transpose: a thread moves a 4 x 4 block of records with 16-byte vector
                                  accesses (1) or one record per thread (0) */
  LLAMA_KNOB_JIT_BMAP,         /* JIT transpose, blocks: thread -> block order 0 x-fastest, 1 y-fastest, 2 / 3
                                  their diagonals, 4 Morton (default: the fewest simulated bank conflicts) */
  LLAMA_KNOB_JIT_TORDER,       /* JIT transpose: tile order over the CTAs, 0 x fastest, 1 y fastest, 2 Morton
                                  within 8 x 8-tile groups */
  LLAMA_KNOB_JIT_DST_LSU,      /* JIT transpose: AoS destination segments stored by the store warp's TMA ops (0) or
                                  as 16-byte chunks by the consumers (1; default unless the destination is Morton) */
  LLAMA_KNOB_JIT_SWIZZLE,      /* JIT transpose, blocks: source segment chunks XOR-swizzled by block row / column
                                  (1) or plain padded pitches (0) */
  LLAMA_KNOB_JIT_GROUP,        /* JIT permute: records per thread group, 1 / 2 / 4 (at least what odd record strides
                                  need; larger groups move SoA / AoSoA leaves and AoS records as wider vectors) */
  LLAMA_KNOB_JIT_CTAS,         /* JIT permute: most CTAs per SM the launch bounds promise (4; the register budget
                                  per thread shrinks with it) */
  LLAMA_KNOB_JIT_ABLATE,        /* JIT kernels, ablation only: 1 = skip the move program (tile loads and stores
                                  only; the destination is NOT the copy) to measure the data movement alone (0) */
  LLAMA_KNOB_WIDE,             /* TRANSPOSE: the wide-record transposing copy (k_transpose_wide): 0 never, 1 when
                                  the JIT / 32 x 32 transposes do not apply (HEP100-sized records), 2 first (1) */
  LLAMA_KNOB_WIDE_GROUP,       /* wide transpose, AoS <-> element-wise side: a thread moves 4 records along the
                                  element-wise side's order, one vector per leaf there (1) */
  LLAMA_KNOB_WIDE_STAGE,       /* wide transpose, element-wise -> AoS: the element-wise side lands by cp.async in a
                                  shared-memory staging area before the image is written (0: measured slower, 0.46 -> 0.39) */
  LLAMA_KNOB_WIDE_CHUNK4,      /* wide transpose: an image may take 4-byte chunks for an odd-word run pitch when that
                                  takes fewer simulated shared-memory wavefronts (0: measured slower) */
  LLAMA_KNOB_WIDE_TORDER,      /* wide transpose tile order: 0 x fastest, 1 y fastest, 2 along a column-major
                                  element-wise side (2) */
  LLAMA_KNOB_WIDE_TMA,         /* wide transpose: AoS images loaded / stored as one tensor-map TMA box per tile (1) */
  LLAMA_KNOB_WIDE_ASYNC,       /* wide transpose, element-wise -> AoS: 4- / 8-byte leaves aligned on both sides land in
                                  the image by cp.async element copies (0: measured 1-5% slower) */
  LLAMA_KNOB_WIDE_AOSOA_IMG,    /* wide transpose: AoSoA-L sides whose tile runs hold whole blocks are staged as
                                  shared-memory images (else element-wise), except an AoSoA destination of a plain AoS
                                  source (2: that too) (1) */
  LLAMA_KNOB_COUNT
} llama_knob;

typedef struct {
  llama_path path;      /* forced path; UNSUPPORTED if not applicable to the pair */
  int32_t tile_records; /* PERMUTE only: records per tile, 0 = planner's choice */
  const int64_t* knobs; /* NULL = all defaults, else LLAMA_KNOB_COUNT values (< 0 = that knob's default);
                           read during the call only */
} llama_copy_options;

/* llama_copy with options (NULL = defaults = llama_copy). */
llama_status llama_copy_ex(const llama_mapping* src_map, void* const* src_blobs,
                           const llama_mapping* dst_map, void* const* dst_blobs, void* stream,
                           const llama_copy_options* options);

/* What the planner chooses for a pair (no device work). */
typedef struct {
  llama_path path;
  int32_t tile_records;     /* PERMUTE: records per tile */
  int32_t smem_bytes;       /* PERMUTE: dynamic shared memory per CTA */
  int32_t moves;            /* PERMUTE: per-record move table length */
  int32_t tma;              /* PERMUTE: 1 if every segment is moved by TMA bulk copies */
  uint64_t src_bytes;       /* sum of source blob sizes */
  uint64_t dst_bytes;       /* sum of destination blob sizes */
  int32_t word_moves;       /* PERMUTE: > 0 if AoS <-> AoS word mode is used (words per record) */
  int32_t direct;           /* PERMUTE: 1 = direct variant (AoS side through TMA, SoA side element-wise) */
  int32_t jit;              /* PERMUTE: 1 = plan-time specialised kernel (NVRTC-compiled move program) */
  int32_t wide;             /* TRANSPOSE: 1 = wide-record transposing copy (tile_records records per tile) */
} llama_plan_info;

llama_status llama_plan(const llama_mapping* src_map, const llama_mapping* dst_map,
                        const llama_copy_options* options, llama_plan_info* out);

/* The generated CUDA source of the plan-time specialised kernel the planner
 * chose for a pair (llama_plan_info.jit == 1), for inspection and tests: the
 * NUL-terminated text is copied into buf (truncated to capacity - 1 bytes);
 * *length (may be NULL) receives the full length.  INVALID_ARGUMENT when the
 * plan is not a JIT plan.  No device work. */
llama_status llama_plan_source(const llama_mapping* src_map, const llama_mapping* dst_map,
                               const llama_copy_options* options, char* buf, uint64_t capacity, uint64_t* length);

/* Seeded synthetic input (an input recipe, not the method): fills every blob
 * byte with pad_byte, then writes byte b of leaf k of record i as byte b
 * (little endian) of splitmix64(seed ^ (i*K + k)), K = n_leaves.  Same blob
 * requirements as llama_copy's dst_blobs. */
llama_status llama_generate(const llama_mapping* m, void* const* blobs, uint64_t seed,
                            uint8_t pad_byte, void* stream);

/* ------------------------------------------------------------------------
 * Staged cross-address-space copy (§3.9: "use smaller intermediate
 * views to shuffle a chunk from one mapping to the other and then perform a
 * copy of that chunk into the other address space, potentially overlapping
 * shuffles and copies in an asynchronous workflow").
 *
 * A stager owns device staging memory and three streams of the device that
 * is current when it is created.  llama_copy_staged cuts the copy into slabs
 * of records whose bytes are contiguous ranges of every blob; per slab it
 * DMAs the source ranges into staging memory (cudaMemcpyAsync), relayouts
 * the slab there with the copy kernels (llama_copy on 1-D views of the slab),
 * and DMAs the destination ranges back, overlapping the three steps of
 * consecutive slabs.  Source and destination blobs may be host memory
 * (pinned for full PCIe speed; pageable works but serialises) or device
 * memory.  Same result contract as llama_copy (destination padding := 0).
 */
typedef struct llama_stager llama_stager; /* opaque; not thread-safe: one copy at a time */

/* Creates a stager with `slab_bytes` of staging memory per side and buffer
 * (3 buffers x 2 sides are allocated with cudaMalloc).  0 = 64 MiB.
 * Errors: INVALID_ARGUMENT, CUDA (no device / allocation failed). */
llama_status llama_stager_create(uint64_t slab_bytes, llama_stager** out);
void llama_stager_destroy(llama_stager* st); /* NULL-safe; synchronises its streams */

/* Enqueues the staged copy after all work already enqueued on `stream`;
 * `stream` waits for its completion.  Errors as llama_copy, plus UNSUPPORTED
 * when one slab of whole AoSoA blocks does not fit the staging memory. */
llama_status llama_copy_staged(llama_stager* st, const llama_mapping* src_map, void* const* src_blobs,
                               const llama_mapping* dst_map, void* const* dst_blobs, void* stream);

/* `count` staged copies as one pipeline: the staging buffers rotate from one
 * copy's slabs straight into the next's, so the DMA engines do not drain
 * between copies (one fill / drain per batch instead of per copy).  Every copy
 * is validated before anything is enqueued; same contract as
 * llama_copy_staged per copy.  src_blobs[i] / dst_blobs[i]: copy i's blob
 * pointer arrays. */
llama_status llama_copy_staged_batch(llama_stager* st, int32_t count, const llama_mapping* const* src_maps,
                                     void* const* const* src_blobs, const llama_mapping* const* dst_maps,
                                     void* const* const* dst_blobs, void* stream);

/* ------------------------------------------------------------------------
 * n-body move (Listing P:643-645, §4.1, §4.2
 * P:698-743): in place on one view, for every particle i and c in {X,Y,Z}
 *     Pos_c(i) = Pos_c(i) + Vel_c(i) * dt
 * in f32 with one rounding (fused multiply-add, as the paper's -ffast-math
 * -mfma / --use_fast_math builds contracted it; DESIGN.md
 * reading #25).
 * pos_leaves[3] / vel_leaves[3]: leaf indices (DFS order) of Pos.{X,Y,Z} and
 * Vel.{X,Y,Z}; all six must be 4-byte leaves (f32).  Only Pos bytes change
 * value (the AoS kernel rewrites whole records with their own bytes).
 * Paths (llama_move_path): GENERIC = thread per particle through the
 * mapping's address function (any mapping); RUNS = 4 consecutive particles
 * per thread as 16-byte vectors of each leaf (every Pos/Vel leaf laid out in
 * 16-byte aligned runs of >= 4 records: SoA, AoSoA with L % 4 == 0, splits of
 * those); AOS = records of one packed/aligned AoS part staged through shared
 * memory with coalesced 16-byte accesses (record size a multiple of 4).
 * Blobs: device memory, 16-byte aligned (as llama_copy).
 * Errors: INVALID_ARGUMENT (NULL, bad leaf index, non-4-byte leaf, a leaf
 * listed twice), UNSUPPORTED (forced path not applicable; a mapping that maps
 * several particles onto one place), ALIGNMENT, CUDA. */
typedef enum {
  LLAMA_MOVE_AUTO = 0, LLAMA_MOVE_GENERIC = 1, LLAMA_MOVE_RUNS = 2, LLAMA_MOVE_AOS = 3,
  LLAMA_MOVE_AOS_LSU = 4 /* as AOS, through the warp-staged LSU kernel instead of the TMA ring (comparison) */
} llama_move_path;
llama_status llama_nbody_move(const llama_mapping* m, void* const* blobs, const int32_t* pos_leaves,
                              const int32_t* vel_leaves, float dt, void* stream);
/* The same with a forced path (AUTO = planner's choice); *path_used (may be
 * NULL) receives the path that ran. */
llama_status llama_nbody_move_ex(const llama_mapping* m, void* const* blobs, const int32_t* pos_leaves,
                                 const int32_t* vel_leaves, float dt, llama_move_path path,
                                 llama_move_path* path_used, void* stream);

/* The n-body move on a view whose blobs may live in host memory (pinned for
 * full PCIe speed): slabs are DMA'd into staging memory, moved in place there
 * (llama_nbody_move on the slab's 1-D view) and DMA'd back, the three steps of
 * consecutive slabs overlapped (the f2 pipeline applied to f3).  Errors as
 * llama_nbody_move and llama_copy_staged. */
llama_status llama_nbody_move_staged(llama_stager* st, const llama_mapping* m, void* const* blobs,
                                     const int32_t* pos_leaves, const int32_t* vel_leaves, float dt, void* stream);

/* Number of kernels this library has launched in this process (monotonic). */
uint64_t llama_launch_count(void);

const char* llama_status_string(llama_status s);
const char* llama_last_error_message(void); /* thread-local, never NULL */
const char* llama_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LLAMA_B200_H */
