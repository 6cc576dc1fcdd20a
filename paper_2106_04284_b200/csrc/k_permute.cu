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

// Full tile: every record exists, so no guards.  A thread owns records
// lane_r + j*Tp (j < R); M moves x R records of independent loads are
// issued before their stores.
template <int W, int R, int M>
__device__ __forceinline__ void move_class_full(const SMove* __restrict__ mt, uint32_t m0, uint32_t m1, uint32_t G,
                                                const uint32_t (&sa)[R], const uint32_t (&sm)[R],
                                                const uint32_t (&da)[R], const uint32_t (&dm)[R]) {
  using U = Unit<W>;
  uint32_t m = m0;
  for (; m + (M - 1) * G < m1; m += M * G) {
    SMove mv[M];
#pragma unroll
    for (int i = 0; i < M; ++i) mv[i] = mt[m + i * G];
    typename U::T v[M][R];
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
      for (int j = 0; j < R; ++j) v[i][j] = U::ld(sa[j] + mv[i].soff + sm[j] * mv[i].size);
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
      for (int j = 0; j < R; ++j) U::st(da[j] + mv[i].doff + dm[j] * mv[i].size, v[i][j]);
  }
  for (; m < m1; m += G) {
    const SMove mv = mt[m];
    typename U::T v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = U::ld(sa[j] + mv.soff + sm[j] * mv.size);
#pragma unroll
    for (int j = 0; j < R; ++j) U::st(da[j] + mv.doff + dm[j] * mv.size, v[j]);
  }
}

template <int R>
__device__ __forceinline__ void permute_full(const PermParams& p, const SMove* __restrict__ mt, uint32_t simg,
                                             uint32_t dimg, uint32_t r0, int tid) {
  const uint32_t Tp = p.T < (uint32_t)kThreads ? p.T : (uint32_t)kThreads;  // records per pass
  const uint32_t G = (uint32_t)kThreads / Tp;                               // move groups
  const uint32_t lane_r = (uint32_t)tid % Tp, grp = (uint32_t)tid / Tp;
  uint32_t sa[R], sm[R], da[R], dm[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const uint32_t r = r0 + lane_r + j * Tp;
    rec_addr(p.side[0], simg, r, sa[j], sm[j]);
    rec_addr(p.side[1], dimg, r, da[j], dm[j]);
  }
  constexpr int M = R >= 4 ? 1 : 4 / R;  // <= 4 loads in flight per thread
  move_class_full<8, R, M>(mt, grp, p.unit_end[0], G, sa, sm, da, dm);
  move_class_full<4, R, M>(mt, p.unit_end[0] + grp, p.unit_end[1], G, sa, sm, da, dm);
  move_class_full<2, R, M>(mt, p.unit_end[1] + grp, p.unit_end[2], G, sa, sm, da, dm);
  move_class_full<1, R, M>(mt, p.unit_end[2] + grp, p.unit_end[3], G, sa, sm, da, dm);
}

// Partial (last) tile: records r < nrec only; simple guarded loops.
template <int W>
__device__ __forceinline__ void move_class_part(const SMove* __restrict__ mt, uint32_t m0, uint32_t m1, uint32_t G,
                                                uint32_t sa, uint32_t sm, uint32_t da, uint32_t dm) {
  for (uint32_t m = m0; m < m1; m += G) {
    const SMove mv = mt[m];
    Unit<W>::st(da + mv.doff + dm * mv.size, Unit<W>::ld(sa + mv.soff + sm * mv.size));
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
  const uint32_t simg = smem_u32(simg_p), dimg = smem_u32(dimg_p);
  if (p.diag) {
    const int warp = tid >> 5, lane = tid & 31;
    uint32_t turn = 0;
    diag_class<8>(p, mt, 0, p.unit_end[0], simg, dimg, nrec, warp, lane, turn);
    diag_class<4>(p, mt, p.unit_end[0], p.unit_end[1], simg, dimg, nrec, warp, lane, turn);
    diag_class<2>(p, mt, p.unit_end[1], p.unit_end[2], simg, dimg, nrec, warp, lane, turn);
    diag_class<1>(p, mt, p.unit_end[2], p.unit_end[3], simg, dimg, nrec, warp, lane, turn);
    return;
  }
  if (nrec == p.T) {  // full tile: passes of 4, 2 or 1 x 256 records (T <= 256 or a multiple of 256)
    uint32_t r0 = 0;
    for (; r0 + 4 * kThreads <= p.T; r0 += 4 * kThreads) permute_full<4>(p, mt, simg, dimg, r0, tid);
    if (r0 + 2 * kThreads <= p.T) {
      permute_full<2>(p, mt, simg, dimg, r0, tid);
      r0 += 2 * kThreads;
    }
    if (r0 < p.T) permute_full<1>(p, mt, simg, dimg, r0, tid);
    return;
  }
  const uint32_t Tp = p.T < (uint32_t)kThreads ? p.T : (uint32_t)kThreads;
  const uint32_t G = (uint32_t)kThreads / Tp;
  const uint32_t grp = (uint32_t)tid / Tp;
  for (uint32_t r = (uint32_t)tid % Tp; r < nrec; r += Tp) {
    uint32_t sa, sm, da, dm;
    rec_addr(p.side[0], simg, r, sa, sm);
    rec_addr(p.side[1], dimg, r, da, dm);
    move_class_part<8>(mt, grp, p.unit_end[0], G, sa, sm, da, dm);
    move_class_part<4>(mt, p.unit_end[0] + grp, p.unit_end[1], G, sa, sm, da, dm);
    move_class_part<2>(mt, p.unit_end[1] + grp, p.unit_end[2], G, sa, sm, da, dm);
    move_class_part<1>(mt, p.unit_end[2] + grp, p.unit_end[3], G, sa, sm, da, dm);
  }
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
  // dynamic smem: [mbarriers | move table | src seg table | dst seg table | src ring | dst buffers]
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  SMove* mt = reinterpret_cast<SMove*>(smem + kBarBytes);
  SSeg* sseg = reinterpret_cast<SSeg*>(smem + kBarBytes + p.tab_moves);
  SSeg* dseg = sseg + p.K;
  uint8_t* sbuf = smem + kBarBytes + p.tab_bytes;
  uint8_t* dbuf = sbuf + (size_t)p.ns * p.src_stage;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

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
  if (kTma && tid == 0) {
    for (uint32_t s = 0; s < p.ns; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  if (blockIdx.x == 0)
    for (uint32_t g = 0; g < p.n_gaps; ++g)
      for (uint32_t o = tid; o < p.gap_len[g]; o += kThreads) p.blobs[1][p.gap_blob[g]][p.gap_off[g] + o] = 0;

  const uint64_t first = blockIdx.x, stride = gridDim.x;
  const uint64_t n_full = p.N / p.T;  // tiles [0, n_full) are full: no tails, no clipping
  if (kTma && warp == 0) {
    for (uint32_t s = 0; s < p.ns; ++s) {
      const uint64_t tile = first + s * stride;
      if (tile < p.n_tiles) issue_loads(p, sseg, tile, tile < n_full, sbuf + (size_t)s * p.src_stage, &bars[s], lane);
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

    if (kTma) {
      if (warp == 0) {  // one warp waits; the others sleep in the barrier below
        if (lane == 0) mbar_wait(&bars[s], (it / p.ns) & 1);
        if (it >= 2) bulk_wait_read<1>();  // dst buffer d (tile it-2) has been read out
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
    if (!(p.debug & 1)) permute_any(p, mt, simg, dimg, nrec, tid);
    if (kTma) fence_proxy_async_smem();
    __syncthreads();

    const int nds = n_segs(p, 1);
    if (kTma) {
      if (warp == 0) {
        for (int j = lane; j < nds; j += 32) {
          const Seg sg = full ? full_seg(p, dseg, 1, tile, j) : tile_seg(p, 1, t0, j);
          const uint32_t body = sg.len & ~15u;
          if (body && !(p.debug & 2)) bulk_s2g(sg.g, dimg + sg.soff, body);
        }
        bulk_commit();
        // ring slot s is free again (every thread passed the barrier): prefetch
        const uint64_t next = tile + (uint64_t)p.ns * stride;
        if (next < p.n_tiles) issue_loads(p, sseg, next, next < n_full, simg, &bars[s], lane);
      }
      if (!full) {
        for (int j = 0; j < nds; ++j) {
          const Seg sg = tile_seg(p, 1, t0, j);
          for (uint32_t o = (sg.len & ~15u) + tid; o < sg.len; o += kThreads) sg.g[o] = dimg[sg.soff + o];
        }
      }
    } else {
      for (int j = 0; j < nds; ++j) {
        const Seg sg = tile_seg(p, 1, t0, j);
        coop_copy(sg.g, dimg + sg.soff, sg.len, tid, kThreads);
      }
    }
  }
  if (kTma && warp == 0) bulk_wait_all();
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
