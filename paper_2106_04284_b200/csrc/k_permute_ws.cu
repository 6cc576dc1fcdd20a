// k_permute_ws.cu -- the warp-specialised TMA tile permute (the hot kernel).
//
// 8 consumer warps permute tiles back to back; 1 producer warp drives the TMA
// (cp.async.bulk loads into an ns-stage source ring, bulk stores out of nd =
// 2 or 3 destination buffers).  Four mbarrier rings replace block-wide barriers:
//   full[s]   TMA bytes of a tile landed in source stage s   (producer -> consumers)
//   empty[s]  consumers finished reading source stage s      (consumers -> producer)
//   dfull[d]  consumers finished writing destination buffer d (consumers -> producer)
//   dempty[d] the bulk store out of buffer d has read it out  (producer -> consumers)
// so the permute of tile i overlaps the stores of tile i-1 and the loads of
// tiles i+1 .. i+ns-1, and no warp waits for another's issue work.
// Producer order per tile (p.order, measured on B200): 2 = refill
// load of stage s first, then the stores of tile i (default; C2 +3-5% over
// stores-first); with nd >= 3 the buffer of tile i-1 is handed back once its
// store has been read out, keeping one store in flight.
// Requires 16-byte aligned segment starts (planner: tma = 1).
#include <cstdlib>

#include "launch.hpp"
#include "permute_common.cuh"

namespace llb {

namespace {
constexpr int kBarBytes = 128;  // 4 rings x <= 4 x 8 B
}  // namespace

// NC consumer threads (8 or 16 warps) + 1 producer warp
template <int NC>
__device__ __forceinline__ void named_sync_consumers() {
  asm volatile("bar.sync 1, %0;" ::"n"(NC) : "memory");
}

template <bool kParts, int NC>
__global__ void __launch_bounds__(NC + 32, NC == 256 ? 3 : 1) k_permute_ws(const __grid_constant__ PermParams p) {
  constexpr int kConsumerWarps = NC / 32;
  constexpr int kThreadsWS = NC + 32;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 4;
  uint64_t* dfull = full + 8;  // ns <= 4 source stages, nd <= 4 destination buffers
  uint64_t* dempty = full + 12;
  SSeg* sseg = reinterpret_cast<SSeg*>(smem + kBarBytes);
  SSeg* dseg = sseg + p.K;
  uint8_t* sbuf = smem + kBarBytes + p.tab_bytes;
  uint8_t* dbuf = sbuf + (size_t)p.ns * p.src_stage;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  // zero both destination images once (padding is never written by a move)
  for (uint32_t o = 16 * tid; o < p.nd * p.dst_stage; o += 16 * kThreadsWS)
    *reinterpret_cast<uint4*>(dbuf + o) = make_uint4(0, 0, 0, 0);
  build_seg_tables(p, sseg, dseg, tid, kThreadsWS);
  WordMove* wt = word_table(smem + kBarBytes, p);
  copy_word_table(p, wt, tid, kThreadsWS);
  if (tid == 0) {
    for (uint32_t s = 0; s < p.ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (uint32_t d = 0; d < p.nd; ++d) {
      mbar_init(&dfull[d], 1);
      mbar_init(&dempty[d], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // Programmatic dependent launch: everything above touched only shared
  // memory and parameters, so it overlapped the previous grid's tail; global
  // memory is used only after that grid has completed.  Dependents may be
  // scheduled at once (they occupy SMs only as this grid's CTAs retire).
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (blockIdx.x == 0 && warp < kConsumerWarps)
    for (uint32_t g = 0; g < p.n_gaps; ++g)
      for (uint32_t o = tid; o < p.gap_len[g]; o += NC) p.blobs[1][p.gap_blob[g]][p.gap_off[g] + o] = 0;

  const uint64_t first = blockIdx.x, stride = gridDim.x;
  const uint64_t n_full = p.N / p.T;
  const uint32_t n_my = first < p.n_tiles ? (uint32_t)((p.n_tiles - first + stride - 1) / stride) : 0;

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer
    // ring positions advance incrementally (no division by the runtime ns / nd
    // on the producer's per-tile critical path)
    auto load = [&](uint32_t i, uint32_t s) {
      const uint64_t tile = first + (uint64_t)i * stride;
      const bool fl = tile < n_full;
      uint8_t* img = sbuf + (size_t)s * p.src_stage;
      const int ns = n_segs(p, 0);
      uint32_t total = p.src_tile_tma;
      if (!fl) {
        total = 0;
        for (int j = 0; j < ns; ++j) total += tile_seg(p, 0, tile * p.T, j).len & ~15u;
      }
      if (lane == 0) mbar_arrive_expect_tx(&full[s], total);
      __syncwarp();
      for (int j = lane; j < ns; j += 32) {
        const Seg sg = fl ? full_seg(p, sseg, 0, tile, j) : tile_seg(p, 0, tile * p.T, j);
        const uint32_t body = sg.len & ~15u;
        if (body) bulk_g2s(img + sg.soff, sg.g, body, &full[s]);
      }
    };
    for (uint32_t i = 0; i < p.ns && i < n_my; ++i) load(i, i);
    const int nds = n_segs(p, 1);
    uint32_t s = 0, sph = 0, d = 0, dph = 0, dprev = p.nd - 1;
    for (uint32_t i = 0; i < n_my; ++i) {
      const uint64_t tile = first + (uint64_t)i * stride;
      const bool fl = tile < n_full;
      auto refill = [&]() {  // refill the source stage tile i used
        if (i + p.ns < n_my) {
          if (lane == 0) mbar_wait_sleep(&empty[s], sph);
          __syncwarp();
          load(i + p.ns, s);
        }
      };
      if (p.order == 2) refill();
      if (lane == 0) mbar_wait_sleep(&dfull[d], dph);
      __syncwarp();
      uint8_t* dimg = dbuf + (size_t)d * p.dst_stage;
      for (int j = lane; j < nds; j += 32) {
        const Seg sg = fl ? full_seg(p, dseg, 1, tile, j) : tile_seg(p, 1, tile * p.T, j);
        const uint32_t body = sg.len & ~15u;
        if (body) bulk_s2g(sg.g, dimg + sg.soff, body);
      }
      bulk_commit();
      if (p.order == 1 && p.nd == 2) {  // release buffer d before refilling
        bulk_wait_read<0>();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[d]);
      }
      if (p.order != 2) refill();
      if (p.order == 1 && p.nd == 2) {
      } else if (p.nd == 2) {
        // hand buffer d back as soon as the store has read it out (the
        // consumers meanwhile fill the other buffer)
        bulk_wait_read<0>();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[d]);
      } else if (i > 0) {
        // >= 3 buffers: keep this tile's store in flight, hand back the previous one's
        bulk_wait_read<1>();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[dprev]);
      }
      dprev = d;
      if (++s == p.ns) { s = 0; sph ^= 1; }
      if (++d == p.nd) { d = 0; dph ^= 1; }
    }
    bulk_wait_all();
    return;
  }

  // ------------------------------------------------------------- consumers
  uint32_t s = 0, sph = 0, d = 0, dph = 0;
  for (uint32_t i = 0; i < n_my; ++i) {
    const uint64_t tile = first + (uint64_t)i * stride;
    const uint64_t t0 = tile * p.T;
    const bool fl = tile < n_full;
    uint8_t* simg = sbuf + (size_t)s * p.src_stage;
    uint8_t* dimg = dbuf + (size_t)d * p.dst_stage;
    if (tid == 0) {  // one consumer thread waits, the others sleep in the named barrier
      mbar_wait(&full[s], sph);
      mbar_wait(&dempty[d], dph ^ 1);  // first use of each buffer passes
    }
    named_sync_consumers<NC>();
    uint32_t nrec = p.T;
    if (!fl) {  // last, partial tile: source tails, zeroed destination image
      nrec = tile_nrec(p, t0);
      for (int j = 0; j < n_segs(p, 0); ++j) {
        const Seg sg = tile_seg(p, 0, t0, j);
        for (uint32_t o = (sg.len & ~15u) + tid; o < sg.len; o += NC) simg[sg.soff + o] = sg.g[o];
      }
      for (uint32_t o = 16 * tid; o < p.dst_stage; o += 16 * NC)
        *reinterpret_cast<uint4*>(dimg + o) = make_uint4(0, 0, 0, 0);
      named_sync_consumers<NC>();
    }
    permute_records<kParts, NC>(p, wt, simg, dimg, nrec, tid);
    if (!fl) {  // destination tails (sub-16-byte) go out directly
      named_sync_consumers<NC>();
      for (int j = 0; j < n_segs(p, 1); ++j) {
        const Seg sg = tile_seg(p, 1, t0, j);
        for (uint32_t o = (sg.len & ~15u) + tid; o < sg.len; o += NC) sg.g[o] = dimg[sg.soff + o];
      }
    }
    fence_proxy_async_smem();  // generic-proxy image writes -> TMA store reads
    named_sync_consumers<NC>();
    if (tid == 0) {
      mbar_arrive(&empty[s]);
      mbar_arrive(&dfull[d]);
    }
    if (++s == p.ns) { s = 0; sph ^= 1; }
    if (++d == p.nd) { d = 0; dph ^= 1; }
  }
}

int launch_permute_ws(const PermParams& p, int smem_bytes, bool pdl, void* stream) {
  // 8 consumer warps (measured: 16 in one CTA are no faster for small
  // records and halve the speed of wide ones, which lose their 2 CTAs per SM)
  static LaunchCache cache[2][64];
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  current_device_sms(&sms);
  const int v = multi_geo(p) ? 1 : 0;
  void (*const kerns[2])(PermParams) = {k_permute_ws<false, kPermThreads>, k_permute_ws<true, kPermThreads>};
  auto kern = kerns[v];
  const int kThreadsWS = kPermThreads + 32;
  int e = prepare_kernel(kern, kThreadsWS, smem_bytes, &cache[v][dev & 63], &per_sm);
  if (e) return e;
  uint64_t grid = (uint64_t)sms * (uint64_t)per_sm;
  if (grid > p.n_tiles) grid = p.n_tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreadsWS);
  cfg.dynamicSmemBytes = (size_t)smem_bytes;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t le = cudaLaunchKernelEx(&cfg, kern, p);
  count_launch();
  return le != cudaSuccess ? (int)le : (int)cudaGetLastError();
}

int launch_permute(const PermParams& p, int smem_bytes, bool v1, bool pdl, void* stream) {
  if (p.n_tiles == 0) return 0;
  if (p.tma && p.ns <= 4 && !v1) return launch_permute_ws(p, smem_bytes, pdl, stream);
  return launch_permute_v1(p, smem_bytes, stream);
}

}  // namespace llb
