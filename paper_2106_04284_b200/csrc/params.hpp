// params.hpp -- kernel parameter blocks shared by the host planner (plan.cpp)
// and the sm_100a kernels (*.cu).  Plain C++ (no CUDA types) so g++ and nvcc
// both compile it.  Every kernel receives one of these by value as a
// __grid_constant__ parameter (<= 32 KB kernel parameter space, CUDA >= 12.1).
#pragma once
#include <cuda.h>  // CUtensorMap (a plain C struct)
#include <stdint.h>

#include "llama_b200.h"

namespace llb {

constexpr int kMaxLeaves = LLAMA_MAX_LEAVES;
constexpr int kMaxBlobs = LLAMA_MAX_BLOBS;
constexpr int kMaxMoves = 512;
constexpr int kMaxRank = LLAMA_MAX_RANK;
constexpr uint32_t kNoShift = 0xFFFFFFFFu;

// One side's mapping in the AoSoA normal form:
//   off(i,k) = base_k + (i / L) * B + F_k + (i % L) * s_k   in blob blob_k
// AoS: L=1, B=S; AoSoA: L=lanes, B=L*S, F_k=L*off_k; SoA: L>=N (one block), B=0.
struct DevSide {
  uint64_t L;       // lanes per block
  uint64_t B;       // block stride in bytes
  uint32_t lshift;  // log2(L) when L is a power of two, else kNoShift
  uint32_t pad_;
};

// Linearisation of the array index: the storage position of the
// record whose array index has row-major rank i (kind 0: i itself).
struct DevLin {
  uint32_t kind;   // llama_linearizer
  uint32_t rank;
  uint32_t bits;   // MORTON: log2 of the (equal) extents
  uint32_t pad_;
  uint64_t ext[kMaxRank];
};

// One leaf's normal form (per leaf, so composite Split mappings and One fit):
//   off(i) = base + (i / L) * B + F + (i % L) * size     in blob `blob`
struct DevLeaf {
  uint64_t base;
  uint64_t F;
  uint64_t L;
  uint64_t B;
  uint32_t blob;
  uint32_t size;
  uint32_t lshift;  // log2(L) when L is a power of two (63 for a single-block SoA leaf), else kNoShift
  uint32_t pad_;
};

// ---------------------------------------------------------------- naive / gen
// Trace / Heatmap counters of one side: hits[k] per leaf, heat
// per blob byte at heat + heat_base[blob] (NULL: not counted).
struct DevTrace {
  unsigned long long* hits;
  uint32_t* heat;
  uint64_t heat_base[kMaxBlobs];
};

struct NaiveParams {
  uint64_t N;
  int32_t K;
  int32_t relin;      // 1: the sides are linearised differently (records located per side)
  DevLin slin, dlin;
  int32_t traced;     // 1: count address resolutions (tr[0] = src, tr[1] = dst)
  uint32_t tsmem;     // TRANSPOSE: shared-memory bytes of a 32x32-record tile
  DevTrace tr[2];
  uint64_t H, W;      // TRANSPOSE: the 2-d extents
  uint32_t tbase[kMaxLeaves];  // TRANSPOSE: leaf k's 32x33-element tile at smem + tbase[k]
  uint32_t taligned;           // TRANSPOSE: every element of both sides naturally aligned
  uint32_t tuniform;           // TRANSPOSE: both sides share one L and B over all leaves
  uint32_t tlinear;            // TRANSPOSE: every leaf of both sides at base + F + f * (L == 1 ? B : size),
                               // f < 2^32: 0 = no, else the one leaf size of all leaves (4 or 8) or 1 (mixed)
  uint32_t sraw, draw;         // TRANSPOSE: that side is a plain AoS moved as raw 16-byte vectors
  uint32_t rawoff;             // TRANSPOSE: shared-memory offset of the raw record buffer
  uint32_t sS, dS;             // TRANSPOSE: record strides of the raw sides
  uint32_t dpad;               // TRANSPOSE: the raw destination has padding bytes (zero the buffer)
  uint32_t linoff;             // TRANSPOSE, linear sides: shared-memory offset of the per-CTA leaf table
  uint32_t raw_typed;          // TRANSPOSE: raw passes as typed 4-byte moves when every leaf is 4 bytes
  DevLeaf sl[kMaxLeaves];
  DevLeaf dl[kMaxLeaves];
  const uint8_t* sb[kMaxBlobs];
  uint8_t* db[kMaxBlobs];
};

struct GenParams {
  uint64_t N;
  uint64_t seed;
  int32_t K;
  int32_t pad_;
  DevLin lin;
  DevLeaf dl[kMaxLeaves];
  uint8_t* db[kMaxBlobs];
};

// Fill every byte of nb blobs with one value (padding pre-fill).
struct FillParams {
  int32_t nb;
  uint32_t value;  // byte replicated
  uint64_t vstart[kMaxBlobs + 1];  // prefix of 16-byte vectors per blob
  uint64_t bytes[kMaxBlobs];
  uint8_t* ptr[kMaxBlobs];
};

// Identity copy of whole blobs ("trivial" copy).
struct BlobCopyParams {
  int32_t nb;
  int32_t pad_;
  uint64_t vstart[kMaxBlobs + 1];
  uint64_t bytes[kMaxBlobs];
  const uint8_t* src[kMaxBlobs];
  uint8_t* dst[kMaxBlobs];
};

// Identity copy through TMA: each blob is cut into chunks of CH bytes that
// one thread per CTA streams global -> shared -> global with a ring of NS
// stages (cp.async.bulk load on an mbarrier, cp.async.bulk store).
struct BulkCopyParams {
  int32_t nb;
  uint32_t CH;                       // chunk bytes (16-B multiple)
  uint32_t NS;                       // ring stages
  uint32_t pad_;
  uint64_t cstart[kMaxBlobs + 1];    // prefix of chunks per blob
  uint64_t bytes[kMaxBlobs];
  const uint8_t* src[kMaxBlobs];
  uint8_t* dst[kMaxBlobs];
  // segments (seg = 1): range j is leaf j's single contiguous run on both
  // sides, src[j] = src blob sblob[j] + soff[j] (patched per call)
  int32_t seg;
  int32_t sblob[kMaxBlobs], dblob[kMaxBlobs];
  uint64_t soff[kMaxBlobs], doff[kMaxBlobs];
};

// ------------------------------------------------------------------ run copy
// Field-run copy: per leaf, records come in runs of
// g = gcd(L_s, L_d) that are contiguous on both sides; g*s_k % 16 == 0 and all
// offsets are 16-byte aligned, so one 16-byte vector never straddles a run.
struct RunParams {
  uint64_t N;
  uint64_t C;        // records per chunk: a CTA moves every leaf of a chunk together
  uint64_t n_chunks;
  uint32_t chunk_vecs;  // 16-byte vectors in a full chunk (sum over leaves)
  int32_t K;
  DevLeaf sl[kMaxLeaves];
  DevLeaf dl[kMaxLeaves];
  uint32_t cvstart[kMaxLeaves + 1];  // prefix of C*s_k/16 vectors per leaf in a chunk
  const uint8_t* sb[kMaxBlobs];
  uint8_t* db[kMaxBlobs];
};

// ------------------------------------------------------------ tile permute
// A tile is T consecutive records.  Each side keeps one shared-memory image
// per tile, made of the images of its parts (one part for the classic kinds,
// one per inner mapping of a Split): an "AoS-like" part (L divides T) as the
// single contiguous byte range of its T/L blocks; a "SoA-like" part (T
// divides L, or SoA) as one segment of T*s_k bytes per leaf.  Inside the
// image, leaf k (of part P) of tile record r sits at
//   (r / Limg_P) * Bimg_P + imgF_k + (r % Limg_P) * s_k.
struct PermPart {
  DevSide g;          // the part's global normal form (segment addresses)
  uint64_t E;         // records the part's blobs cover (padded block extent / N)
  uint32_t soa_like;  // 1: per-leaf segments
  uint32_t pad_;
};

struct PermGeo {      // image geometry shared by one or more parts of a side
  uint32_t Limg;      // image lanes (AoS-like: L; SoA-like: T)
  uint32_t limg_shift;
  uint32_t Bimg;      // image block stride
  uint32_t pad_;
};
constexpr int kMaxParts = 8;

struct PermSeg {      // segment j of a side: part, leaf (AoS-like: any leaf of the part), image offset
  uint16_t part;
  uint16_t leaf;
  uint32_t soff;
};

struct PermSide {
  uint64_t E;         // records the side's blobs cover (max over its parts)
  uint32_t n_parts;
  uint32_t n_geo;     // distinct image geometries (1: the permute hoists one record offset)
  uint32_t n_segs;
  uint32_t linear;    // 1: a full tile's segment addresses are linear in the tile index
  uint32_t img_bytes; // image bytes of a full tile
};

struct Move {        // one unit move of the per-record permutation
  uint32_t soff;     // src image offset of leaf part for r = 0
  uint32_t doff;     // dst image offset
  uint16_t size;     // leaf size s_k (multiplies r % Limg)
  uint8_t unit;      // bytes moved: 1, 2, 4 or 8
  uint8_t pad_;
};

// Word move (AoS <-> AoS word mode): destination word doff of a record is
// built from the 12-byte source window at soff (4-aligned):
//   t = prmt(w0, w1, sel1); v = prmt(t, w2, sel2) & mask   (w2 read only if sel2 != 0x3210)
struct WordMove {
  uint16_t doff, soff;
  uint16_t sel1, sel2;
  uint32_t mask;
};
constexpr int kMaxWordMoves = 128;  // 4 per lane

struct MoveClass {    // moves [m0, m1) share unit, leaf size and the parts on both sides
  uint32_t m0, m1;
  uint16_t unit, size;
  uint16_t sp, dp;    // src / dst image geometry
};
constexpr int kMaxClasses = 32;

struct PermParams {
  uint64_t N;         // records
  uint64_t n_tiles;   // ceil(R / T), R = records the dst image must cover
  uint32_t T;         // records per tile (multiple of 32)
  uint32_t n_moves;
  uint32_t K;
  uint32_t tma;       // 1: segment starts 16-B aligned for every tile -> TMA bulk
  uint32_t src_stage; // bytes of one src image buffer (16-B multiple)
  uint32_t dst_stage; // bytes of one dst image buffer
  uint32_t ns, nd;    // src stages, dst buffers
  uint32_t order;     // producer: 1 = release the dst buffer before the refill load
  uint32_t src_tile_tma;  // TMA bytes of a full tile's source segments
  uint32_t n_classes;
  MoveClass classes[kMaxClasses];
  uint32_t n_wmoves;     // > 0: AoS <-> AoS word mode (move-parallel) instead of the move classes
  WordMove wmoves[kMaxWordMoves];
  uint32_t tab_bytes;     // shared-memory bytes of the segment tables (16-B multiple)
  uint32_t pad2_;
  PermSide side[2];   // 0 = src, 1 = dst
  PermPart part[2][kMaxParts];
  PermGeo geo[2][kMaxParts];
  PermSeg seg[2][kMaxLeaves];
  DevLeaf leaf[2][kMaxLeaves];
  Move moves[kMaxMoves];
  // destination padding outside every tile segment (gaps between the leaf
  // sub-arrays of an aligned SoA single blob): zeroed by CTA 0
  uint32_t n_gaps;
  uint32_t gap_blob[kMaxLeaves];
  uint32_t gap_len[kMaxLeaves];
  uint64_t gap_off[kMaxLeaves];
  uint8_t* blobs[2][kMaxBlobs];
};

// ---------------------------------------------------------- n-body move
// Listing P:643-645: Pos_c += Vel_c * dt for c in X, Y, Z (f32, two roundings).
struct MoveParams {
  uint64_t N;
  float dt;
  uint32_t S;          // AOS path: record stride in bytes
  uint32_t g;          // AOS path: records per thread (g * S % 16 == 0)
  uint32_t aligned;    // GENERIC path: every Pos/Vel access is 4-byte aligned
  uint64_t base;       // AOS path: byte offset of record 0 in blob `blob`
  uint32_t blob;       // AOS path
  uint32_t fpos[3], fvel[3];  // AOS path: leaf offsets inside a record
  uint32_t tile, ns;          // AOS path, TMA kernel: records per tile, ring stages (tile = 0: LSU kernel)
  DevLeaf pos[3], vel[3];     // GENERIC / RUNS paths
  uint8_t* blobs[kMaxBlobs];
  uint32_t traced;            // GENERIC path: count resolutions into tr
  uint32_t lpos[3], lvel[3];  // leaf indices of Pos / Vel (trace counters)
  DevTrace tr;
};

// ------------------------------------------------------- direct permute
// AoS <-> SoA with many leaves (HEP100): the AoS side moves as one TMA op per
// tile through a shared-memory ring, the SoA side element by element with
// coalesced global accesses (a warp = 32 consecutive records of one leaf) --
// no per-leaf TMA segments of T * s_k bytes.
struct DirectLeaf {
  uint64_t gbase;    // SoA side: byte offset of record 0's element in its blob
  uint8_t* gptr;     // SoA side: blob + gbase (filled per launch)
  uint32_t F;        // AoS side: offset of the leaf inside a record
  uint32_t blob;     // SoA side blob
  uint16_t size;
  uint8_t a_img;     // alignment of every (r * S + F) in the AoS image (1, 2, 4, 8)
  uint8_t a_glob;    // alignment of every SoA element address
  uint32_t stg;      // SoA -> AoS, staged class: offset of the leaf's T elements in the staging area
};

// Leaves of equal size and alignment classes, handled by one specialised loop:
// kind = size | 16 (image accesses aligned) | 32 (global accesses aligned).
struct DirectClass {
  uint16_t k0, k1;   // range in DirectParams::order
  uint32_t kind;
};

struct DirectParams {
  uint64_t N, n_tiles;
  uint32_t T, K, S;  // S: AoS record stride
  uint32_t a2s;      // 1: AoS -> SoA (ring holds source tiles); 0: SoA -> AoS (ring holds destination tiles)
  uint32_t ns, stage;
  uint32_t mix;      // 1: aligned-image classes use the 4-leaves x 8-records warp mapping
  uint32_t async;    // SoA -> AoS: 4- / 8-byte classes aligned on both sides land by cp.async
  uint32_t stg_bytes; // SoA -> AoS with async: staging area of the misaligned 4- / 8-byte (phase) classes
  uint64_t abase;    // AoS side: byte offset of record 0 in blob `ablob`
  uint32_t ablob;
  uint32_t n_gaps;   // AoS -> aligned SoA SB: padding between sub-arrays, zeroed by CTA 0
  uint32_t gap_blob[kMaxLeaves];
  uint32_t gap_len[kMaxLeaves];
  uint64_t gap_off[kMaxLeaves];
  DirectLeaf leaf[kMaxLeaves];
  uint32_t n_cls;
  uint32_t cat_end[3];  // SoA -> AoS with async: class ranges [0, e0) chunk-staged, [e0, e1) staged, [e1, e2) cp.async
  DirectClass cls[16];
  uint16_t order[kMaxLeaves];  // leaf ids grouped by class
  uint8_t* blobs[2][kMaxBlobs];
};
static_assert(sizeof(DirectParams) <= 32764, "DirectParams exceeds the kernel parameter limit");

// ------------------------------------------------- wide transposing copy
// Rank-2 views of different storage orders whose records are too
// wide for the JIT transpose's TY x 32-record tiles (HEP100: 380 / 480 B).
// A tile is 2^lty x 2^ltx records; each side is either an "A" side (plain
// AoS, record stride S % 4 == 0) staged as a shared-memory image of the
// tile's storage runs (row: 2^ltx records, column: 2^lty, Morton: the whole
// tile, which is Morton-contiguous), or an "E" side (SoA / AoSoA) accessed
// element by element with the warp's lanes along that side's storage order.
struct WideSide {
  uint32_t A;       // 1: AoS image side
  uint32_t lin;     // llama_linearizer
  uint32_t S;       // A: record stride
  uint32_t blob;    // A: the blob
  uint64_t base;    // A: byte offset of record 0
  uint32_t chunk;   // A: bytes per cp.async / vector access of a run (16, 8 or 4)
  uint32_t pitch;   // A: image bytes per run (a multiple of chunk)
  uint32_t lrun;    // A: log2 records per run
  uint32_t img;     // A: shared-memory offset of the image
  uint32_t img_bytes;
  uint32_t uni;     // E: every leaf shares L / B below (the block split is hoisted out of the leaf loop)
  uint64_t L, B;    // E, uni: lanes per block, block stride (A: block stride too)
  uint32_t lshift;  // E, uni: log2(L) or kNoShift
  uint32_t mshift;  // E, uni, L not a power of two: ceil(log2 L); q = (t + ((p - t) >> 1)) >> (mshift - 1),
  uint64_t magic;   //   t = umulhi(p, magic), magic = floor(2^64 (2^mshift - L) / L) + 1
  // A, tensor-map TMA (knob wide_tma): the tile's runs are one box of the
  // side's blob viewed as a 2-d (row-major: [H][W * S]) or 3-d (column-major:
  // [W][H / g][g * S]) array of elsz-byte elements; the image is the dense box
  uint32_t lL;      // A: log2 of the lanes per block (AoSoA-L images: record t of a run sits in block
  uint32_t pad5_;   //   (t >> lL) at B bytes per block (the B above), lane t & (L - 1); plain AoS: lL = 0, B = S)
  uint32_t tma;     // 0 cp.async / vector copies, 2 / 3: box dimensions
  uint32_t elsz;    // element bytes of the tensor map (1, 2, 4, 8)
  uint32_t g;       // 3-d: records per innermost row of the box
  uint32_t box_bytes;
};

// Leaf j of the class order (positions, not leaf ids: the kernel walks them in order).
struct WideLeaf {
  uint8_t* sp;          // E source (uniform): blob + base + F (patched per launch)
  uint8_t* dp;          // E destination (uniform)
  uint32_t soff, doff;  // A sides: leaf offset inside a record
  uint16_t size, unit;  // unit: widest access valid at every address on both sides (1, 2, 4, 8)
  uint32_t buf;         // E -> E: offset of the leaf's element buffer inside the batch area
  uint32_t vec;         // E -> E, grp: bit 0 / 1 = every 4-element group of the source / destination
                        // is one 4 * s_k-byte range aligned to min(16, 4 * s_k)
};

struct WideClass {      // positions [j0, j1) share size, unit and (grp) the E-side vector flag
  uint16_t j0, j1;
  uint16_t size, unit;  // unit | 256: every 4-record group of the E side is one aligned vector
};

struct WideParams {
  CUtensorMap tmap[2];  // per side when side[X].tma (encoded per launch: the blob address is part of it)
  uint64_t H, W;
  uint64_t ntx;         // tiles along x
  uint64_t nty;         // tiles along y
  uint32_t yfast;       // tile order: y fastest (along a column-major side)
  uint32_t pad3_;
  uint64_t n_items;     // tiles (x nbatch for E -> E)
  uint32_t lty, ltx;    // log2 tile rows / columns
  uint32_t mode;        // 0 A -> E, 1 E -> A, 2 A -> A (leaf moves), 3 A -> A (same record layout), 4 E -> E
  uint32_t K;
  uint32_t nbatch;      // E -> E: leaf batches per tile
  uint32_t dzero;       // the destination image has padding bytes: zeroed once per CTA
  uint32_t smem;        // dynamic shared memory per CTA
  uint32_t buf;         // E -> E: shared-memory offset of the batch area
  uint32_t n_cls;
  uint32_t u3;          // mode 3: bytes per access of a record copy (16, 8, 4)
  uint32_t bar;         // shared-memory offset of the TMA mbarrier (8 bytes)
  uint32_t async;       // mode 1, grp: 4- / 8-byte elements aligned on both sides move by cp.async
  uint32_t grp;         // modes 0 / 1 / 4: threads move 4-record groups along the E side's order
  uint32_t stage;       // mode 1, grp: the E side lands by cp.async in a staging area at buf first
  uint16_t bstart[kMaxLeaves + 1];   // E -> E: batch b = positions [bstart[b], bstart[b+1])
  uint16_t order[kMaxLeaves];        // leaf id at each position
  WideClass cls[16];
  WideSide side[2];
  WideLeaf leaf[kMaxLeaves];
  DevLeaf sl[kMaxLeaves];            // by position: E sides that are not uniform
  DevLeaf dl[kMaxLeaves];
  const uint8_t* sb[kMaxBlobs];
  uint8_t* db[kMaxBlobs];
};
static_assert(sizeof(WideParams) <= 32764, "WideParams exceeds the kernel parameter limit");

// kernel parameter blocks travel as __grid_constant__ arguments (<= 32764 B)
static_assert(sizeof(PermParams) <= 32764, "PermParams exceeds the kernel parameter limit");
static_assert(sizeof(NaiveParams) <= 32764, "NaiveParams exceeds the kernel parameter limit");
static_assert(sizeof(RunParams) <= 32764, "RunParams exceeds the kernel parameter limit");
}  // namespace llb
