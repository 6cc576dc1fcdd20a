// k_permute.cu -- the staged tile permute: AoS <-> SoA / AoSoA transposes,
// packed <-> aligned relayouts, sub-word and misaligned leaves, padding.
//
// Per tile of T records:
//   1. TMA bulk copies (cp.async.bulk, one per contiguous segment) bring the
//      tile's source bytes into a shared-memory source image; an mbarrier
//      counts the bytes ("large, contiguous memory chunks").
//   2. The CTA permutes source image -> destination image with a per-record
//      move table of 1/2/4/8-byte units (every leaf of every record
//      lands at the destination mapping's offset).  Destination padding is
//      never written by a move; the image was zeroed once, so padding goes out
//      as 0 (reading #12).
//   3. TMA bulk stores write the destination image's segments (full sectors).
// Persistent CTAs loop over tiles; the next tiles' loads are in flight
// (ns-stage ring) while a tile is permuted, and stores drain asynchronously
// (2 destination buffers).  Both HBM sides move as whole contiguous segments.
#include "device.cuh"
#include "launch.hpp"

namespace llb {

namespace {
constexpr int kThreads = 256;
constexpr int kBarBytes = 128;  // mbarrier area at the start of dynamic smem
}  // namespace

// Phase timers (debug bit 4, experiments only): cycles thread 0 spends per
// phase of the tile loop, summed over CTAs.
__device__ unsigned long long g_perm_prof[8];

// Per-CTA shared copies of the tables the tile loop reads with a dynamic
// index (kernel parameters live in the constant bank; dynamic-index reads of
// a 20 KB parameter block miss the constant cache).
struct SMove {
  uint32_t soff, doff, size;
};
struct SSeg {         // segment j of a side whose tile segments are linear in the tile index
  uint8_t* g0;        // address for tile 0
  uint64_t tstride;   // bytes per tile
  uint32_t soff;      // offset in the image
  uint32_t len;       // bytes in a full tile
};

struct Seg {
  uint8_t* g;     // global address of the segment for this tile
  uint32_t soff;  // offset inside the side's image
  uint32_t len;   // bytes
};

// Segment j of side X for the tile starting at record t0.
__device__ __forceinline__ Seg tile_seg(const PermParams& p, int X, uint64_t t0, int j) {
  const PermSide& S = p.side[X];
  const uint64_t end = t0 + p.T < S.E ? t0 + p.T : S.E;
  const uint64_t nrec = end > t0 ? end - t0 : 0;
  Seg s;
  if (!S.soa_like) {  // AoS-like: the tile's T/L whole blocks are one range
    const DevLeaf& l0 = p.leaf[X][0];
    const uint64_t blk0 = block_of(t0, S.g);
    s.g = p.blobs[X][l0.blob] + l0.base + blk0 * S.g.B;
    s.soff = 0;
    s.len = (uint32_t)(block_of(nrec, S.g) * S.g.B);
  } else {            // SoA-like: leaf j's T consecutive elements
    const DevLeaf& l = p.leaf[X][j];
    s.g = p.blobs[X][l.blob] + nf_offset(t0, S.g, l);
    s.soff = p.imgF[X][j];
    s.len = (uint32_t)(nrec * l.size);
  }
  return s;
}

__device__ __forceinline__ int n_segs(const PermParams& p, int X) { return p.side[X].soa_like ? (int)p.K : 1; }

// Cooperative byte-exact copy for segments that are not TMA-eligible (any
// alignment): 16-byte vectors when both sides are congruent mod 16, else
// 4-byte words when congruent mod 4, else bytes.
__device__ void coop_copy(uint8_t* d, const uint8_t* s, uint32_t len, int tid, int nt) {
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

// ---- shared-memory unit accesses on 32-bit shared addresses
template <int W> struct Unit;
template <> struct Unit<8> {
  using T = unsigned long long;
  static __device__ __forceinline__ T ld(uint32_t a) { T v; asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a)); return v; }
  static __device__ __forceinline__ void st(uint32_t a, T v) { asm volatile("st.shared.b64 [%0], %1;" :: "r"(a), "l"(v)); }
};
template <> struct Unit<4> {
  using T = uint32_t;
  static __device__ __forceinline__ T ld(uint32_t a) { T v; asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a)); return v; }
  static __device__ __forceinline__ void st(uint32_t a, T v) { asm volatile("st.shared.b32 [%0], %1;" :: "r"(a), "r"(v)); }
};
template <> struct Unit<2> {
  using T = unsigned short;
  static __device__ __forceinline__ T ld(uint32_t a) { T v; asm volatile("ld.shared.b16 %0, [%1];" : "=h"(v) : "r"(a)); return v; }
  static __device__ __forceinline__ void st(uint32_t a, T v) { asm volatile("st.shared.b16 [%0], %1;" :: "r"(a), "h"(v)); }
};
template <> struct Unit<1> {
  using T = unsigned short;
  static __device__ __forceinline__ T ld(uint32_t a) { T v; asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a)); return v; }
  static __device__ __forceinline__ void st(uint32_t a, T v) { asm volatile("st.shared.u8 [%0], %1;" :: "r"(a), "h"(v)); }
};

// Record-dependent part of the image addresses of record r on one side:
// base = image + (r / Limg) * Bimg, mul = r % Limg (multiplies the leaf size).
__device__ __forceinline__ void rec_addr(const PermSide& S, uint32_t img, uint32_t r, uint32_t& base, uint32_t& mul) {
  const uint32_t q = S.limg_shift != kNoShift ? (r >> S.limg_shift) : r / S.Limg;
  mul = r - q * S.Limg;
  base = img + q * S.Bimg;
}

// One move class for the R records this thread owns.  The record-dependent
// offsets (block base + (r % Limg) * size) are hoisted out of the move loop;
// a move is then one load and one store at a warp-uniform offset (soff/doff
// read from the parameter bank with a uniform index), so the compiler can use
// [reg + ureg] addressing and batch the R independent loads.
template <typename U, int R>
__device__ __forceinline__ void move_class_fast(const PermParams& p, const MoveClass& mc, uint32_t G, uint32_t grp,
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

template <int R>
__device__ __forceinline__ void permute_pass(const PermParams& p, const uint8_t* __restrict__ simg,
                                             uint8_t* __restrict__ dimg, uint32_t nrec, uint32_t r0, int tid) {
  const uint32_t Tp = p.T < (uint32_t)kThreads ? p.T : (uint32_t)kThreads;  // records per pass
  const uint32_t G = (uint32_t)kThreads / Tp;                               // move groups
  const uint32_t lane_r = (uint32_t)tid % Tp, grp = (uint32_t)tid / Tp;
  uint32_t sb[R], sm[R], db[R], dm[R];
  bool ok[R];
  bool all = true;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const uint32_t r = r0 + lane_r + j * Tp;
    ok[j] = r < nrec;
    all = all && ok[j];
    rec_addr(p.side[0], 0u, r, sb[j], sm[j]);
    rec_addr(p.side[1], 0u, r, db[j], dm[j]);
  }
  for (uint32_t c = 0; c < p.n_classes; ++c) {
    const MoveClass mc = p.classes[c];
    switch (mc.unit) {
      case 8: move_class_fast<unsigned long long, R>(p, mc, G, grp, simg, dimg, sb, sm, db, dm, ok, all); break;
      case 4: move_class_fast<uint32_t, R>(p, mc, G, grp, simg, dimg, sb, sm, db, dm, ok, all); break;
      case 2: move_class_fast<unsigned short, R>(p, mc, G, grp, simg, dimg, sb, sm, db, dm, ok, all); break;
      default: move_class_fast<unsigned char, R>(p, mc, G, grp, simg, dimg, sb, sm, db, dm, ok, all); break;
    }
  }
}

// Wide records (few records per tile, many moves): 32 x 32 blocks of
// (record, move) pairs per warp; at step t lane j moves record rb+j's move
// mb + ((j+t) & 31).  Lanes hit distinct records AND distinct moves, so both
// images see spread banks (a record-parallel warp would hit one leaf of 32
// records at the record stride: 8-way conflicts for 480-B aligned records).
template <int W>
__device__ __forceinline__ void diag_class(const PermParams& p, const SMove* __restrict__ mt, uint32_t c0, uint32_t c1,
                                           uint32_t simg, uint32_t dimg, uint32_t nrec, int warp, int lane,
                                           uint32_t& turn) {
  using U = Unit<W>;
  const uint32_t nrb = (nrec + 31) / 32;
  const uint32_t nmb = (c1 - c0 + 31) / 32;
  for (uint32_t b = 0; b < nrb * nmb; ++b, ++turn) {
    if ((int)(turn % (kThreads / 32)) != warp) continue;
    const uint32_t rb = (b / nmb) * 32, mb = c0 + (b % nmb) * 32;
    const uint32_t r = rb + lane;
    uint32_t sa, sm, da, dm;
    rec_addr(p.side[0], simg, r, sa, sm);
    rec_addr(p.side[1], dimg, r, da, dm);
    const bool rok = r < nrec;
#pragma unroll 4
    for (uint32_t t = 0; t < 32; ++t) {
      const uint32_t m = mb + ((lane + t) & 31);
      if (rok && m < c1) {
        const SMove mv = mt[m];
        U::st(da + mv.doff + dm * mv.size, U::ld(sa + mv.soff + sm * mv.size));
      }
    }
  }
}

__device__ __forceinline__ void permute_any(const PermParams& p, const SMove* mt, uint8_t* simg_p, uint8_t* dimg_p,
                                            uint32_t nrec, int tid) {
  if (p.diag) {
    const uint32_t simg = smem_u32(simg_p), dimg = smem_u32(dimg_p);
    const int warp = tid >> 5, lane = tid & 31;
    uint32_t turn = 0;
    diag_class<8>(p, mt, 0, p.unit_end[0], simg, dimg, nrec, warp, lane, turn);
    diag_class<4>(p, mt, p.unit_end[0], p.unit_end[1], simg, dimg, nrec, warp, lane, turn);
    diag_class<2>(p, mt, p.unit_end[1], p.unit_end[2], simg, dimg, nrec, warp, lane, turn);
    diag_class<1>(p, mt, p.unit_end[2], p.unit_end[3], simg, dimg, nrec, warp, lane, turn);
    return;
  }
  // passes of 4, 2 or 1 x 256 records (T <= 256 or a multiple of 256)
  uint32_t r0 = 0;
  for (; r0 + 4 * kThreads <= p.T; r0 += 4 * kThreads) permute_pass<4>(p, simg_p, dimg_p, nrec, r0, tid);
  if (r0 + 2 * kThreads <= p.T) {
    permute_pass<2>(p, simg_p, dimg_p, nrec, r0, tid);
    r0 += 2 * kThreads;
  }
  if (r0 < p.T) permute_pass<1>(p, simg_p, dimg_p, nrec, r0, tid);
}

// Segment j of side X for a full tile, from the shared table (linear sides)
// or computed (large-block AoSoA sides).
__device__ __forceinline__ Seg full_seg(const PermParams& p, const SSeg* __restrict__ st, int X, uint64_t tile,
                                        int j) {
  if (p.side[X].linear) {
    const SSeg& e = st[j];
    return Seg{e.g0 + tile * e.tstride, e.soff, e.len};
  }
  return tile_seg(p, X, tile * p.T, j);
}

__device__ __forceinline__ uint32_t tile_nrec(const PermParams& p, uint64_t t0) {
  if (t0 >= p.N) return 0;
  const uint64_t n = p.N - t0;
  return n < p.T ? (uint32_t)n : p.T;
}

// ---- LSU transfers for sides with many small segments (SoA with many leaves):
// every thread moves 16-byte chunks (cp.async for loads, arriving on the
// stage mbarrier; LDS.128 + STG.128 for stores) instead of ~K tiny TMA ops.
__device__ __forceinline__ void cp_async16(uint32_t sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Chunk c of a full tile -> (segment j, byte offset), j advancing monotonically.
__device__ __forceinline__ uint32_t chunk_seg(const uint32_t* __restrict__ cst, uint32_t c, int& j) {
  while (c >= cst[j + 1]) ++j;
  return (c - cst[j]) * 16;
}

__device__ __forceinline__ void issue_loads_lsu(const PermParams& p, const SSeg* sseg, const uint32_t* cst,
                                                uint64_t tile, bool full, uint8_t* img, uint64_t* bar, int tid) {
  const uint32_t simg = smem_u32(img);
  if (full) {
    int j = 0;
    for (uint32_t c = tid; c < cst[n_segs(p, 0)]; c += kThreads) {
      const uint32_t o = chunk_seg(cst, c, j);
      cp_async16(simg + sseg[j].soff + o, sseg[j].g0 + tile * sseg[j].tstride + o);
    }
  } else {
    for (int j = 0; j < n_segs(p, 0); ++j) {
      const Seg sg = tile_seg(p, 0, tile * p.T, j);
      for (uint32_t o = 16 * tid; o + 16 <= sg.len; o += 16 * kThreads) cp_async16(simg + sg.soff + o, sg.g + o);
    }
  }
  cp_async_arrive_noinc(bar);  // every thread arrives once per phase (count = kThreads)
}

__device__ __forceinline__ void store_lsu(const PermParams& p, const SSeg* dseg, const uint32_t* cst, uint64_t tile,
                                          bool full, const uint8_t* dimg, int tid) {
  if (full) {
    int j = 0;
    for (uint32_t c = tid; c < cst[n_segs(p, 1)]; c += kThreads) {
      const uint32_t o = chunk_seg(cst, c, j);
      const uint4 v = *reinterpret_cast<const uint4*>(dimg + dseg[j].soff + o);
      __stcs(reinterpret_cast<uint4*>(dseg[j].g0 + tile * dseg[j].tstride + o), v);
    }
  } else {
    for (int j = 0; j < n_segs(p, 1); ++j) {
      const Seg sg = tile_seg(p, 1, tile * p.T, j);
      uint32_t o = 16 * tid;
      for (; o + 16 <= sg.len; o += 16 * kThreads)
        __stcs(reinterpret_cast<uint4*>(sg.g + o), *reinterpret_cast<const uint4*>(dimg + sg.soff + o));
      for (uint32_t q = (sg.len & ~15u) + tid; q < sg.len; q += kThreads) sg.g[q] = dimg[sg.soff + q];
    }
  }
}

// Issues the TMA loads of a tile's source segments into one stage (warp 0):
// lane 0 arms the stage's mbarrier with the byte count, the lanes issue one
// cp.async.bulk per segment.
__device__ __forceinline__ void issue_loads(const PermParams& p, const SSeg* sseg, uint64_t tile, bool full,
                                            uint8_t* img, uint64_t* bar, int lane) {
  const int ns = n_segs(p, 0);
  const uint64_t t0 = tile * p.T;
  uint32_t total = p.src_tile_tma;
  if (!full) {
    total = 0;
    for (int j = 0; j < ns; ++j) total += tile_seg(p, 0, t0, j).len & ~15u;
  }
  if (lane == 0) mbar_arrive_expect_tx(bar, total);
  __syncwarp();
  for (int j = lane; j < ns; j += 32) {
    const Seg s = full ? full_seg(p, sseg, 0, tile, j) : tile_seg(p, 0, t0, j);
    const uint32_t body = s.len & ~15u;
    if (body) bulk_g2s(img + s.soff, s.g, body, bar);
  }
}

template <bool kTma>
__global__ void __launch_bounds__(kThreads, 4) k_permute(const __grid_constant__ PermParams p) {
  // dynamic smem: [mbarriers | move table | src seg table | dst seg table |
  //                src chunk prefix | dst chunk prefix | src ring | dst buffers]
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  SMove* mt = reinterpret_cast<SMove*>(smem + kBarBytes);
  SSeg* sseg = reinterpret_cast<SSeg*>(smem + kBarBytes + p.tab_moves);
  SSeg* dseg = sseg + p.K;
  uint32_t* scst = reinterpret_cast<uint32_t*>(dseg + p.K);
  uint32_t* dcst = scst + (p.K + 1);
  uint8_t* sbuf = smem + kBarBytes + p.tab_bytes;
  uint8_t* dbuf = sbuf + (size_t)p.ns * p.src_stage;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const bool lsu_s = kTma && p.lsu[0], lsu_d = kTma && p.lsu[1];

  // Zero both destination images once: padding positions are never written
  // by a move, so they stay 0 for every tile.
  for (uint32_t o = 16 * tid; o < p.nd * p.dst_stage; o += 16 * kThreads)
    *reinterpret_cast<uint4*>(dbuf + o) = make_uint4(0, 0, 0, 0);
  for (uint32_t m = tid; m < p.n_moves; m += kThreads) mt[m] = SMove{p.moves[m].soff, p.moves[m].doff, p.moves[m].size};
  for (uint32_t j = tid; j < 2 * p.K; j += kThreads) {
    const int X = j < p.K ? 0 : 1, k = j < p.K ? (int)j : (int)(j - p.K);
    if (p.side[X].linear && k < n_segs(p, X)) {
      const Seg s0 = tile_seg(p, X, 0, k);
      const Seg s1 = tile_seg(p, X, p.T, k);  // linear: tile 1 - tile 0 = per-tile stride
      (X == 0 ? sseg : dseg)[k] = SSeg{s0.g, (uint64_t)(s1.g - s0.g), s0.soff, s0.len};
    }
  }
  if (tid == 0) {  // 16-byte chunk prefixes of the full-tile segments (LSU sides)
    uint32_t a = 0, b = 0;
    scst[0] = dcst[0] = 0;
    for (uint32_t k = 0; k < p.K; ++k) {
      if (p.lsu[0] && (int)k < n_segs(p, 0)) a += tile_seg(p, 0, 0, (int)k).len / 16;
      if (p.lsu[1] && (int)k < n_segs(p, 1)) b += tile_seg(p, 1, 0, (int)k).len / 16;
      scst[k + 1] = a;
      dcst[k + 1] = b;
    }
  }
  if (kTma && tid == 0) {
    for (uint32_t s = 0; s < p.ns; ++s) mbar_init(&bars[s], lsu_s ? kThreads : 1);
    fence_mbar_init();
  }
  __syncthreads();

  if (blockIdx.x == 0)
    for (uint32_t g = 0; g < p.n_gaps; ++g)
      for (uint32_t o = tid; o < p.gap_len[g]; o += kThreads) p.blobs[1][p.gap_blob[g]][p.gap_off[g] + o] = 0;

  const uint64_t first = blockIdx.x, stride = gridDim.x;
  const uint64_t n_full = p.N / p.T;  // tiles [0, n_full) are full: no tails, no clipping
  const bool only_permute = p.debug & 16;
  if (kTma && !only_permute) {
    for (uint32_t s = 0; s < p.ns; ++s) {
      const uint64_t tile = first + s * stride;
      if (tile >= p.n_tiles) break;
      uint8_t* img = sbuf + (size_t)s * p.src_stage;
      if (lsu_s) issue_loads_lsu(p, sseg, scst, tile, tile < n_full, img, &bars[s], tid);
      else if (warp == 0) issue_loads(p, sseg, tile, tile < n_full, img, &bars[s], lane);
    }
  }

  uint32_t it = 0;
  for (uint64_t tile = first; tile < p.n_tiles; tile += stride, ++it) {
    const uint32_t s = it % p.ns, d = it & 1;
    uint8_t* simg = sbuf + (size_t)s * p.src_stage;
    uint8_t* dimg = dbuf + (size_t)d * p.dst_stage;
    const uint64_t t0 = tile * p.T;
    const bool full = tile < n_full;
    const uint32_t nrec = full ? p.T : tile_nrec(p, t0);

    const bool prof = (p.debug & 4) && tid == 0;
    long long c0 = prof ? clock64() : 0, c1 = 0, c2 = 0, c3 = 0, c4 = 0;
    if (only_permute) {
      // experiment: permute the stage's stale bytes, no memory traffic
    } else if (kTma) {
      if (warp == 0) {  // one warp waits; the others sleep in the barrier below
        if (lane == 0) mbar_wait(&bars[s], (it / p.ns) & 1);
        if (prof) c1 = clock64();
        if (!lsu_d && it >= 2) bulk_wait_read<1>();  // dst buffer d (tile it-2) has been read out
        __syncwarp();
      }
      if (!full) {  // sub-16-byte tails of the last tile's segments
        __syncthreads();
        for (int j = 0; j < n_segs(p, 0); ++j) {
          const Seg sg = tile_seg(p, 0, t0, j);
          for (uint32_t o = (sg.len & ~15u) + tid; o < sg.len; o += kThreads) simg[sg.soff + o] = sg.g[o];
        }
      }
    } else {
      __syncthreads();
      for (int j = 0; j < n_segs(p, 0); ++j) {
        const Seg sg = tile_seg(p, 0, t0, j);
        coop_copy(simg + sg.soff, sg.g, sg.len, tid, kThreads);
      }
    }
    __syncthreads();

    if (!full) {  // records beyond N are padding in the dst image
      for (uint32_t o = 16 * tid; o < p.dst_stage; o += 16 * kThreads)
        *reinterpret_cast<uint4*>(dimg + o) = make_uint4(0, 0, 0, 0);
      __syncthreads();
    }
    if (prof) c2 = clock64();
    if (!(p.debug & 1)) permute_any(p, mt, simg, dimg, nrec, tid);
    long long cf = prof ? clock64() : 0;
    if (kTma && !lsu_d) fence_proxy_async_smem();
    if (prof) c3 = clock64();
    __syncthreads();
    if (prof) c4 = clock64();

    const int nds = n_segs(p, 1);
    if (only_permute) {
    } else if (kTma) {
      const uint64_t next = tile + (uint64_t)p.ns * stride;
      if (lsu_d) {
        if (!(p.debug & 2)) store_lsu(p, dseg, dcst, tile, full, dimg, tid);
      } else if (warp == 0) {
        for (int j = lane; j < nds; j += 32) {
          const Seg sg = full ? full_seg(p, dseg, 1, tile, j) : tile_seg(p, 1, t0, j);
          const uint32_t body = sg.len & ~15u;
          if (body && !(p.debug & 2)) bulk_s2g(sg.g, dimg + sg.soff, body);
        }
        bulk_commit();
      }
      // ring slot s is free again (every thread passed the barrier): prefetch
      if (next < p.n_tiles) {
        if (lsu_s) issue_loads_lsu(p, sseg, scst, next, next < n_full, simg, &bars[s], tid);
        else if (warp == 0) issue_loads(p, sseg, next, next < n_full, simg, &bars[s], lane);
      }
      if (!full && !lsu_d) {
        for (int j = 0; j < nds; ++j) {
          const Seg sg = tile_seg(p, 1, t0, j);
          for (uint32_t o = (sg.len & ~15u) + tid; o < sg.len; o += kThreads) sg.g[o] = dimg[sg.soff + o];
        }
      }
      if (prof) {
        const long long c5 = clock64();
        atomicAdd(&g_perm_prof[0], (unsigned long long)(c1 - c0));  // mbarrier wait (TMA load)
        atomicAdd(&g_perm_prof[1], (unsigned long long)(c2 - c1));  // store drain + barrier A
        atomicAdd(&g_perm_prof[2], (unsigned long long)(c3 - c2));  // permute (thread 0) + fence
        atomicAdd(&g_perm_prof[3], (unsigned long long)(c4 - c3));  // barrier B (slowest thread)
        atomicAdd(&g_perm_prof[4], (unsigned long long)(c5 - c4));  // issue stores + next loads
        atomicAdd(&g_perm_prof[5], 1ull);                           // tiles
        atomicAdd(&g_perm_prof[6], (unsigned long long)(c3 - cf));  // fence.proxy.async alone
      }
    } else {
      for (int j = 0; j < nds; ++j) {
        const Seg sg = tile_seg(p, 1, t0, j);
        coop_copy(sg.g, dimg + sg.soff, sg.len, tid, kThreads);
      }
    }
  }
  if (kTma && warp == 0 && !only_permute) bulk_wait_all();
}

// Debug hook (not in the public header): read and optionally reset the phase timers.
extern "C" int llama_debug_permute_profile(unsigned long long* out8, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(out8, g_perm_prof, sizeof(g_perm_prof));
  if (e == cudaSuccess && reset) {
    unsigned long long z[8] = {0};
    e = cudaMemcpyToSymbol(g_perm_prof, z, sizeof(z));
  }
  return (int)e;
}

int launch_permute(const PermParams& p, int smem_bytes, void* stream) {
  if (p.n_tiles == 0) return 0;
  cudaError_t e;
  int sms = 148;
  current_device_sms(&sms);
  int per_sm = 1;
  if (p.tma) {
    e = cudaFuncSetAttribute(k_permute<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return (int)e;
    cudaFuncSetAttribute(k_permute<true>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_permute<true>, kThreads, smem_bytes);
  } else {
    e = cudaFuncSetAttribute(k_permute<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return (int)e;
    cudaFuncSetAttribute(k_permute<false>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_permute<false>, kThreads, smem_bytes);
  }
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)sms * (uint64_t)per_sm;
  if (grid > p.n_tiles) grid = p.n_tiles;
  if (p.tma)
    k_permute<true><<<(unsigned)grid, kThreads, smem_bytes, (cudaStream_t)stream>>>(p);
  else
    k_permute<false><<<(unsigned)grid, kThreads, smem_bytes, (cudaStream_t)stream>>>(p);
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace llb
