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

// The per-record permutation src image -> dst image.
__device__ __forceinline__ void permute_tile(const PermParams& p, const uint8_t* __restrict__ simg,
                                             uint8_t* __restrict__ dimg, uint32_t nrec, int tid) {
  const uint32_t Tp = p.T < (uint32_t)kThreads ? p.T : (uint32_t)kThreads;  // records per pass
  const uint32_t G = (uint32_t)kThreads / Tp;                               // move groups
  const uint32_t lane_r = (uint32_t)tid % Tp, grp = (uint32_t)tid / Tp;
  const PermSide& S = p.side[0];
  const PermSide& D = p.side[1];
  for (uint32_t r = lane_r; r < nrec; r += Tp) {
    const uint32_t qs = S.limg_shift != kNoShift ? (r >> S.limg_shift) : r / S.Limg;
    const uint32_t ms = r - qs * S.Limg;
    const uint32_t qd = D.limg_shift != kNoShift ? (r >> D.limg_shift) : r / D.Limg;
    const uint32_t md = r - qd * D.Limg;
    const uint32_t sb = qs * S.Bimg, db = qd * D.Bimg;
    for (uint32_t m = grp; m < p.n_moves; m += G) {
      const Move mv = p.moves[m];
      const uint32_t so = sb + mv.soff + ms * mv.size;
      const uint32_t dof = db + mv.doff + md * mv.size;
      switch (mv.unit) {
        case 8: *reinterpret_cast<uint64_t*>(dimg + dof) = *reinterpret_cast<const uint64_t*>(simg + so); break;
        case 4: *reinterpret_cast<uint32_t*>(dimg + dof) = *reinterpret_cast<const uint32_t*>(simg + so); break;
        case 2: *reinterpret_cast<uint16_t*>(dimg + dof) = *reinterpret_cast<const uint16_t*>(simg + so); break;
        default: dimg[dof] = simg[so]; break;
      }
    }
  }
}

__device__ __forceinline__ uint32_t tile_nrec(const PermParams& p, uint64_t t0) {
  if (t0 >= p.N) return 0;
  const uint64_t n = p.N - t0;
  return n < p.T ? (uint32_t)n : p.T;
}

// Issues the TMA loads of a tile's source segments into one stage (warp 0):
// lane 0 arms the stage's mbarrier with the byte count, the lanes issue one
// cp.async.bulk per segment.
__device__ __forceinline__ void issue_loads(const PermParams& p, uint64_t t0, bool full, uint8_t* img,
                                            uint64_t* bar, int lane) {
  const int ns = n_segs(p, 0);
  uint32_t total = p.src_tile_tma;
  if (!full) {
    total = 0;
    for (int j = 0; j < ns; ++j) total += tile_seg(p, 0, t0, j).len & ~15u;
  }
  if (lane == 0) mbar_arrive_expect_tx(bar, total);
  __syncwarp();
  for (int j = lane; j < ns; j += 32) {
    const Seg s = tile_seg(p, 0, t0, j);
    const uint32_t body = s.len & ~15u;
    if (body) bulk_g2s(img + s.soff, s.g, body, bar);
  }
}

template <bool kTma>
__global__ void __launch_bounds__(kThreads) k_permute(const __grid_constant__ PermParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint8_t* sbuf = smem + kBarBytes;
  uint8_t* dbuf = sbuf + (size_t)p.ns * p.src_stage;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  // Zero both destination images once: padding positions are never written
  // by a move, so they stay 0 for every tile.
  for (uint32_t o = 16 * tid; o < p.nd * p.dst_stage; o += 16 * kThreads)
    *reinterpret_cast<uint4*>(dbuf + o) = make_uint4(0, 0, 0, 0);
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
      if (tile < p.n_tiles)
        issue_loads(p, tile * p.T, tile < n_full, sbuf + (size_t)s * p.src_stage, &bars[s], lane);
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
    permute_tile(p, simg, dimg, nrec, tid);
    if (kTma) fence_proxy_async_smem();
    __syncthreads();

    const int nds = n_segs(p, 1);
    if (kTma) {
      if (warp == 0) {
        for (int j = lane; j < nds; j += 32) {
          const Seg sg = tile_seg(p, 1, t0, j);
          const uint32_t body = sg.len & ~15u;
          if (body) bulk_s2g(sg.g, dimg + sg.soff, body);
        }
        bulk_commit();
        // ring slot s is free again (every thread passed the barrier): prefetch
        const uint64_t next = tile + (uint64_t)p.ns * stride;
        if (next < p.n_tiles) issue_loads(p, next * p.T, next < n_full, simg, &bars[s], lane);
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
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_permute<true>, kThreads, smem_bytes);
  } else {
    e = cudaFuncSetAttribute(k_permute<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (e != cudaSuccess) return (int)e;
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
