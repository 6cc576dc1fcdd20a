// k_permute.cu -- the barrier-synchronised tile permute.  Used for pairs whose
// segments are not all 16-byte aligned (any alignment: cooperative LSU copies)
// and, with TMA, as the comparison baseline of the warp-specialised kernel in
// k_permute_ws.cu (LLAMA_PERMUTE_V1=1).
//
// Per tile of T records: bring the tile's
// source segments into a shared-memory image (TMA bulk copies on an mbarrier,
// or cooperative copies), permute source image -> destination image with the
// per-record move table (every leaf of every record lands at the
// destination mapping's offset; destination padding is never written by a
// move and the image was zeroed once, so padding goes out as 0, reading #12),
// write the destination segments (TMA bulk stores or cooperative copies).
#include "launch.hpp"
#include "permute_common.cuh"

namespace llb {

namespace {
constexpr int kThreads = kPermThreads;
constexpr int kBarBytes = 128;  // mbarrier area at the start of dynamic smem
}  // namespace

// TMA loads of a tile's source segments into one stage (warp 0): lane 0 arms
// the stage's mbarrier with the byte count, the lanes issue one bulk op each.
__device__ __forceinline__ void issue_loads_v1(const PermParams& p, const SSeg* sseg, uint64_t tile, bool full,
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

template <bool kTma, bool kParts>
__global__ void __launch_bounds__(kThreads, 4) k_permute(const __grid_constant__ PermParams p) {
  // dynamic smem: [mbarriers | segment tables | src ring | dst buffers]
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  SSeg* sseg = reinterpret_cast<SSeg*>(smem + kBarBytes);
  SSeg* dseg = sseg + p.K;
  uint8_t* sbuf = smem + kBarBytes + p.tab_bytes;
  uint8_t* dbuf = sbuf + (size_t)p.ns * p.src_stage;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  // Zero both destination images once: padding positions are never written
  // by a move, so they stay 0 for every tile.
  for (uint32_t o = 16 * tid; o < p.nd * p.dst_stage; o += 16 * kThreads)
    *reinterpret_cast<uint4*>(dbuf + o) = make_uint4(0, 0, 0, 0);
  build_seg_tables(p, sseg, dseg, tid, kThreads);
  WordMove* wt = word_table(smem + kBarBytes, p);
  copy_word_table(p, wt, tid, kThreads);
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
      if (tile >= p.n_tiles) break;
      issue_loads_v1(p, sseg, tile, tile < n_full, sbuf + (size_t)s * p.src_stage, &bars[s], lane);
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
    permute_records<kParts>(p, wt, simg, dimg, nrec, tid);
    if (kTma) fence_proxy_async_smem();
    __syncthreads();

    const int nds = n_segs(p, 1);
    if (kTma) {
      if (warp == 0) {
        for (int j = lane; j < nds; j += 32) {
          const Seg sg = full ? full_seg(p, dseg, 1, tile, j) : tile_seg(p, 1, t0, j);
          const uint32_t body = sg.len & ~15u;
          if (body) bulk_s2g(sg.g, dimg + sg.soff, body);
        }
        bulk_commit();
        // ring slot s is free again (every thread passed the barrier): prefetch
        const uint64_t next = tile + (uint64_t)p.ns * stride;
        if (next < p.n_tiles) issue_loads_v1(p, sseg, next, next < n_full, simg, &bars[s], lane);
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

int launch_permute_v1(const PermParams& p, int smem_bytes, void* stream) {
  static LaunchCache cache[4][64];
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  current_device_sms(&sms);
  const int v = (p.tma ? 1 : 0) + (multi_geo(p) ? 2 : 0);
  void (*const kern[4])(PermParams) = {k_permute<false, false>, k_permute<true, false>, k_permute<false, true>,
                                       k_permute<true, true>};
  int e = prepare_kernel(kern[v], kThreads, smem_bytes, &cache[v][dev & 63], &per_sm);
  if (e) return e;
  uint64_t grid = (uint64_t)sms * (uint64_t)per_sm;
  if (grid > p.n_tiles) grid = p.n_tiles;
  kern[v]<<<(unsigned)grid, kThreads, smem_bytes, (cudaStream_t)stream>>>(p);
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace llb
