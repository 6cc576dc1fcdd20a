// permute_common.cuh -- tile geometry and the shared-memory permutation used
// by both tile-permute kernels (k_permute.cu: barrier-synchronised, any
// alignment; k_permute_ws.cu: warp-specialised TMA pipeline).
//
// A tile is T consecutive records.  Each side
// keeps one shared-memory image per tile, the images of its parts one after
// another (a Split has one part per inner mapping): an AoS-like part (L
// divides T) as the single contiguous byte range of its T/L blocks, a
// SoA-like part as one segment of T*s_k bytes per leaf.  Inside an image,
// leaf k of tile record r sits at (r / Limg) * Bimg + imgF_k + (r % Limg) * s_k
// with its part's Limg / Bimg.
#pragma once
#include "device.cuh"

namespace llb {

constexpr int kPermThreads = 256;  // threads that permute (consumer warps)

struct Seg {
  uint8_t* g;     // global address of the segment for this tile
  uint32_t soff;  // offset inside the side's image
  uint32_t len;   // bytes
};

// Segment j of side X for the tile starting at record t0 (any tile, clipped
// to the side's record extent E).
__device__ __forceinline__ Seg tile_seg(const PermParams& p, int X, uint64_t t0, int j) {
  const PermSeg sg = p.seg[X][j];
  const PermPart& P = p.part[X][sg.part];
  const uint64_t end = t0 + p.T < P.E ? t0 + p.T : P.E;
  const uint64_t nrec = end > t0 ? end - t0 : 0;
  const DevLeaf& l = p.leaf[X][sg.leaf];
  Seg s;
  s.soff = sg.soff;
  if (!P.soa_like) {  // AoS-like: the tile's T/L whole blocks are one range
    const uint64_t blk0 = block_of(t0, P.g);
    s.g = p.blobs[X][l.blob] + l.base + blk0 * P.g.B;
    s.len = (uint32_t)(block_of(nrec, P.g) * P.g.B);
  } else {            // SoA-like: the leaf's T consecutive elements
    s.g = p.blobs[X][l.blob] + nf_offset(t0, P.g, l);
    s.len = (uint32_t)(nrec * l.size);
  }
  return s;
}

__device__ __forceinline__ int n_segs(const PermParams& p, int X) { return (int)p.side[X].n_segs; }

__device__ __forceinline__ uint32_t tile_nrec(const PermParams& p, uint64_t t0) {
  if (t0 >= p.N) return 0;
  const uint64_t n = p.N - t0;
  return n < p.T ? (uint32_t)n : p.T;
}

// Segment address table for sides whose full-tile segment starts are linear
// in the tile index (AoS-like and SoA sides): start = g0 + tile * tstride.
struct SSeg {
  uint8_t* g0;
  uint64_t tstride;
  uint32_t soff;
  uint32_t len;
};

__device__ __forceinline__ Seg full_seg(const PermParams& p, const SSeg* __restrict__ st, int X, uint64_t tile,
                                        int j) {
  if (p.side[X].linear) {
    const SSeg& e = st[j];
    return Seg{e.g0 + tile * e.tstride, e.soff, e.len};
  }
  return tile_seg(p, X, tile * p.T, j);
}

// Fills the per-CTA segment tables (threads tid of nt).
__device__ __forceinline__ void build_seg_tables(const PermParams& p, SSeg* sseg, SSeg* dseg, int tid, int nt) {
  for (uint32_t j = tid; j < 2 * p.K; j += nt) {
    const int X = j < p.K ? 0 : 1, k = j < p.K ? (int)j : (int)(j - p.K);
    if (p.side[X].linear && k < n_segs(p, X)) {
      const Seg s0 = tile_seg(p, X, 0, k);
      const Seg s1 = tile_seg(p, X, p.T, k);  // tile 1 - tile 0 = per-tile stride
      (X == 0 ? sseg : dseg)[k] = SSeg{s0.g, (uint64_t)(s1.g - s0.g), s0.soff, s0.len};
    }
  }
}

// Cooperative byte-exact copy for segments that are not TMA-eligible (any
// alignment): 16-byte vectors when both sides are congruent mod 16, else
// 4-byte words when congruent mod 4, else bytes.
__device__ inline void coop_copy(uint8_t* d, const uint8_t* s, uint32_t len, int tid, int nt) {
  const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(d) ^ reinterpret_cast<uintptr_t>(s)) & 15);
  uint32_t head = 0, body = 0;
  if (mis == 0 || (mis & 3) == 0) {
    const uint32_t w = mis == 0 ? 16 : 4;
    head = (uint32_t)((w - (reinterpret_cast<uintptr_t>(d) & (w - 1))) & (w - 1));
    if (head > len) head = len;
    body = (len - head) / w * w;
    if (w == 16) {
      for (uint32_t o = head + 16 * tid; o < head + body; o += 16 * nt)
        *reinterpret_cast<uint4*>(d + o) = *reinterpret_cast<const uint4*>(s + o);
    } else {
      for (uint32_t o = head + 4 * tid; o < head + body; o += 4 * nt)
        *reinterpret_cast<uint32_t*>(d + o) = *reinterpret_cast<const uint32_t*>(s + o);
    }
  }
  for (uint32_t o = tid; o < head; o += nt) d[o] = s[o];
  for (uint32_t o = head + body + tid; o < len; o += nt) d[o] = s[o];
}

// ------------------------------------------------------------ the permute
// Record-dependent part of an image offset of record r on one side:
// base = (r / Limg) * Bimg, mul = r % Limg (multiplies the leaf size).
__device__ __forceinline__ void rec_addr(const PermGeo& S, uint32_t r, uint32_t& base, uint32_t& mul) {
  const uint32_t q = S.limg_shift != kNoShift ? (r >> S.limg_shift) : r / S.Limg;
  mul = r - q * S.Limg;
  base = q * S.Bimg;
}

// One move class (same unit and leaf size) for the R records this thread
// owns.  The record-dependent offsets are hoisted out of the move loop; a move
// is one load and one store at a warp-uniform offset (read from the parameter
// bank with a uniform index), and the R loads of a move are independent.
template <typename U, int R>
__device__ __forceinline__ void move_class(const PermParams& p, const MoveClass& mc, uint32_t G, uint32_t grp,
                                           const uint8_t* __restrict__ simg, uint8_t* __restrict__ dimg,
                                           const uint32_t (&sb)[R], const uint32_t (&sm)[R],
                                           const uint32_t (&db)[R], const uint32_t (&dm)[R],
                                           const bool (&ok)[R], bool all) {
  uint32_t rs[R], rd[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    rs[j] = sb[j] + sm[j] * mc.size;
    rd[j] = db[j] + dm[j] * mc.size;
  }
  if (all) {
#pragma unroll 2
    for (uint32_t m = mc.m0 + grp; m < mc.m1; m += G) {
      const uint32_t so = p.moves[m].soff, dof = p.moves[m].doff;
      U v[R];
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = *reinterpret_cast<const U*>(simg + rs[j] + so);
#pragma unroll
      for (int j = 0; j < R; ++j) *reinterpret_cast<U*>(dimg + rd[j] + dof) = v[j];
    }
  } else {
    for (uint32_t m = mc.m0 + grp; m < mc.m1; m += G) {
      const uint32_t so = p.moves[m].soff, dof = p.moves[m].doff;
#pragma unroll
      for (int j = 0; j < R; ++j)
        if (ok[j]) *reinterpret_cast<U*>(dimg + rd[j] + dof) = *reinterpret_cast<const U*>(simg + rs[j] + so);
    }
  }
}

// Records r0 + lane_r + j*Tp (j < R) of the tile; for T < 256 the thread
// groups beyond the first Tp threads split the move table instead (G groups).
// kParts: a side has several image geometries (Split parts of different
// kinds), so the record-dependent offsets are recomputed when the class's
// geometries differ from the previous class's (classes are ordered by them).
template <int R, bool kParts, int NT>
__device__ __forceinline__ void permute_pass(const PermParams& p, const uint8_t* __restrict__ simg,
                                             uint8_t* __restrict__ dimg, uint32_t nrec, uint32_t r0, int tid) {
  const uint32_t Tp = p.T < (uint32_t)NT ? p.T : (uint32_t)NT;
  const uint32_t G = (uint32_t)NT / Tp;
  const uint32_t lane_r = (uint32_t)tid % Tp, grp = (uint32_t)tid / Tp;
  uint32_t sb[R], sm[R], db[R], dm[R];
  bool ok[R];
  bool all = true;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const uint32_t r = r0 + lane_r + j * Tp;
    ok[j] = r < nrec;
    all = all && ok[j];
    rec_addr(p.geo[0][0], r, sb[j], sm[j]);
    rec_addr(p.geo[1][0], r, db[j], dm[j]);
  }
  uint32_t cur_sp = 0, cur_dp = 0;
  for (uint32_t c = 0; c < p.n_classes; ++c) {
    const MoveClass mc = p.classes[c];
    if (kParts && mc.sp != cur_sp) {
      cur_sp = mc.sp;
#pragma unroll
      for (int j = 0; j < R; ++j) rec_addr(p.geo[0][cur_sp], r0 + lane_r + j * Tp, sb[j], sm[j]);
    }
    if (kParts && mc.dp != cur_dp) {
      cur_dp = mc.dp;
#pragma unroll
      for (int j = 0; j < R; ++j) rec_addr(p.geo[1][cur_dp], r0 + lane_r + j * Tp, db[j], dm[j]);
    }
    switch (mc.unit) {
      case 8: move_class<unsigned long long, R>(p, mc, G, grp, simg, dimg, sb, sm, db, dm, ok, all); break;
      case 4: move_class<uint32_t, R>(p, mc, G, grp, simg, dimg, sb, sm, db, dm, ok, all); break;
      case 2: move_class<unsigned short, R>(p, mc, G, grp, simg, dimg, sb, sm, db, dm, ok, all); break;
      default: move_class<unsigned char, R>(p, mc, G, grp, simg, dimg, sb, sm, db, dm, ok, all); break;
    }
  }
}

// AoS <-> AoS word mode: lane j owns destination words j, j+32, ... of a
// record (table in registers); warps take records in turn.  Both images are
// accessed as consecutive words within a record: no bank conflicts at any
// record stride (the 480-B aligned HEP record gives 8-way conflicts in the
// record-parallel mapping).
// (table: the per-CTA shared copy, see word_table())
template <int NT>
__device__ __forceinline__ void permute_words(const PermParams& p, const WordMove* __restrict__ wt,
                                              const uint8_t* __restrict__ simg, uint8_t* __restrict__ dimg,
                                              uint32_t nrec, int tid) {
  const int warp = tid >> 5, lane = tid & 31;
  WordMove w[4];
  bool has[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t m = lane + 32 * i;
    has[i] = m < p.n_wmoves;
    w[i] = has[i] ? wt[m] : WordMove{0, 0, 0x3210, 0x3210, 0};
  }
  const uint32_t Bs = p.geo[0][0].Bimg, Bd = p.geo[1][0].Bimg;
  for (uint32_t r = warp; r < nrec; r += NT / 32) {
    const uint8_t* sr = simg + r * Bs;
    uint8_t* dr = dimg + r * Bd;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (!has[i]) continue;
      const uint32_t a = *reinterpret_cast<const uint32_t*>(sr + w[i].soff);
      const uint32_t b = *reinterpret_cast<const uint32_t*>(sr + w[i].soff + 4);
      uint32_t v = __byte_perm(a, b, w[i].sel1);
      if (w[i].sel2 != 0x3210) v = __byte_perm(v, *reinterpret_cast<const uint32_t*>(sr + w[i].soff + 8), w[i].sel2);
      *reinterpret_cast<uint32_t*>(dr + w[i].doff) = v & w[i].mask;
    }
  }
}

// The whole tile, threads tid in [0, 256): T <= 256 or a multiple of 256
// (planner), in passes of 4, 2 or 1 x 256 records.
// Per-CTA shared copy of the word-move table: it lives after the segment
// tables (lane-indexed reads of the parameter bank would serialise).
__device__ __forceinline__ WordMove* word_table(uint8_t* tables, const PermParams& p) {
  return reinterpret_cast<WordMove*>(tables + ((2u * 32u * p.K + 15u) & ~15u));
}

__device__ __forceinline__ void copy_word_table(const PermParams& p, WordMove* wt, int tid, int nt) {
  for (uint32_t m = tid; m < p.n_wmoves; m += nt) wt[m] = p.wmoves[m];
}

// kParts: instantiated separately (its own kernel), so the single-geometry
// kernel keeps its register allocation and code size (measured: a shared
// kernel with both paths ran 4.5% slower on the C2 pairs).
template <bool kParts, int NT = kPermThreads>
__device__ __forceinline__ void permute_records(const PermParams& p, const WordMove* wt, const uint8_t* simg,
                                                uint8_t* dimg, uint32_t nrec, int tid) {
  if (!kParts && p.n_wmoves) {
    permute_words<NT>(p, wt, simg, dimg, nrec, tid);
    return;
  }
  uint32_t r0 = 0;
  for (; r0 + 4 * NT <= p.T; r0 += 4 * NT) permute_pass<4, kParts, NT>(p, simg, dimg, nrec, r0, tid);
  if (r0 + 2 * NT <= p.T) {
    permute_pass<2, kParts, NT>(p, simg, dimg, nrec, r0, tid);
    r0 += 2 * NT;
  }
  if (r0 < p.T) permute_pass<1, kParts, NT>(p, simg, dimg, nrec, r0, tid);
}

// Several image geometries on a side (planner: n_geo > 1)?
__host__ __device__ __forceinline__ bool multi_geo(const PermParams& p) {
  return p.side[0].n_geo > 1 || p.side[1].n_geo > 1;
}

}  // namespace llb
