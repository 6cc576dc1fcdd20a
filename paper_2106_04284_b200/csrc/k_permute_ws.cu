// k_permute_ws.cu -- the warp-specialised TMA tile permute (the hot kernel).
//
// 8 consumer warps permute tiles back to back; 1 producer warp drives the TMA
// (cp.async.bulk loads into an ns-stage source ring, bulk stores out of two
// destination buffers).  Four mbarrier rings replace block-wide barriers:
//   full[s]   TMA bytes of a tile landed in source stage s   (producer -> consumers)
//   empty[s]  consumers finished reading source stage s      (consumers -> producer)
//   dfull[d]  consumers finished writing destination buffer d (consumers -> producer)
//   dempty[d] the bulk store out of buffer d has read it out  (producer -> consumers)
// so the permute of tile i overlaps the stores of tile i-1 and the loads of
// tiles i+1 .. i+ns-1, and no warp waits for another's issue work.
// Requires 16-byte aligned segment starts (planner: tma = 1).
#include <cstdlib>

#include "launch.hpp"
#include "permute_common.cuh"

namespace llb {

namespace {
constexpr int kConsumerWarps = kPermThreads / 32;        // 8
constexpr int kThreadsWS = kPermThreads + 32;            // + 1 producer warp
constexpr int kBarBytes = 128;                           // 4 rings x <= 4 x 8 B
}  // namespace

__device__ __forceinline__ void named_sync_consumers() {
  asm volatile("bar.sync 1, %0;" ::"n"(kPermThreads) : "memory");
}

template <bool kParts>
__global__ void __launch_bounds__(kThreadsWS, 3) k_permute_ws(const __grid_constant__ PermParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + 4;
  uint64_t* dfull = full + 8;
  uint64_t* dempty = full + 10;
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
    for (int d = 0; d < 2; ++d) {
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
      for (uint32_t o = tid; o < p.gap_len[g]; o += kPermThreads) p.blobs[1][p.gap_blob[g]][p.gap_off[g] + o] = 0;

  const uint64_t first = blockIdx.x, stride = gridDim.x;
  const uint64_t n_full = p.N / p.T;
  const uint32_t n_my = first < p.n_tiles ? (uint32_t)((p.n_tiles - first + stride - 1) / stride) : 0;

  if (warp == kConsumerWarps) {
    // ------------------------------------------------------------ producer
    auto load = [&](uint32_t i) {
      const uint64_t tile = first + (uint64_t)i * stride;
      const bool fl = tile < n_full;
      const uint32_t s = i % p.ns;
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
    for (uint32_t i = 0; i < p.ns && i < n_my; ++i) load(i);
    const int nds = n_segs(p, 1);
    for (uint32_t i = 0; i < n_my; ++i) {
      const uint64_t tile = first + (uint64_t)i * stride;
      const bool fl = tile < n_full;
      const uint32_t d = i & 1;
      if (lane == 0) mbar_wait(&dfull[d], (i >> 1) & 1);
      __syncwarp();
      uint8_t* dimg = dbuf + (size_t)d * p.dst_stage;
      for (int j = lane; j < nds; j += 32) {
        const Seg sg = fl ? full_seg(p, dseg, 1, tile, j) : tile_seg(p, 1, tile * p.T, j);
        const uint32_t body = sg.len & ~15u;
        if (body) bulk_s2g(sg.g, dimg + sg.soff, body);
      }
      bulk_commit();
      if (i + p.ns < n_my) {  // refill the source stage tile i used
        if (lane == 0) mbar_wait(&empty[i % p.ns], (i / p.ns) & 1);
        __syncwarp();
        load(i + p.ns);
      }
      // hand buffer d back as soon as the store has read it out (the
      // consumers meanwhile fill the other buffer)
      bulk_wait_read<0>();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dempty[d]);
    }
    bulk_wait_all();
    return;
  }

  // ------------------------------------------------------------- consumers
  for (uint32_t i = 0; i < n_my; ++i) {
    const uint64_t tile = first + (uint64_t)i * stride;
    const uint64_t t0 = tile * p.T;
    const bool fl = tile < n_full;
    const uint32_t s = i % p.ns, d = i & 1;
    uint8_t* simg = sbuf + (size_t)s * p.src_stage;
    uint8_t* dimg = dbuf + (size_t)d * p.dst_stage;
    if (tid == 0) {  // one consumer thread waits, the others sleep in the named barrier
      mbar_wait(&full[s], (i / p.ns) & 1);
      mbar_wait(&dempty[d], ((i >> 1) & 1) ^ 1);  // first use of each buffer passes
    }
    named_sync_consumers();
    uint32_t nrec = p.T;
    if (!fl) {  // last, partial tile: source tails, zeroed destination image
      nrec = tile_nrec(p, t0);
      for (int j = 0; j < n_segs(p, 0); ++j) {
        const Seg sg = tile_seg(p, 0, t0, j);
        for (uint32_t o = (sg.len & ~15u) + tid; o < sg.len; o += kPermThreads) simg[sg.soff + o] = sg.g[o];
      }
      for (uint32_t o = 16 * tid; o < p.dst_stage; o += 16 * kPermThreads)
        *reinterpret_cast<uint4*>(dimg + o) = make_uint4(0, 0, 0, 0);
      named_sync_consumers();
    }
    permute_records<kParts>(p, wt, simg, dimg, nrec, tid);
    if (!fl) {  // destination tails (sub-16-byte) go out directly
      named_sync_consumers();
      for (int j = 0; j < n_segs(p, 1); ++j) {
        const Seg sg = tile_seg(p, 1, t0, j);
        for (uint32_t o = (sg.len & ~15u) + tid; o < sg.len; o += kPermThreads) sg.g[o] = dimg[sg.soff + o];
      }
    }
    fence_proxy_async_smem();  // generic-proxy image writes -> TMA store reads
    named_sync_consumers();
    if (tid == 0) {
      mbar_arrive(&empty[s]);
      mbar_arrive(&dfull[d]);
    }
  }
}

int launch_permute_ws(const PermParams& p, int smem_bytes, void* stream) {
  static LaunchCache cache[2][64];
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  current_device_sms(&sms);
  const bool parts = multi_geo(p);
  auto kern = parts ? k_permute_ws<true> : k_permute_ws<false>;
  int e = prepare_kernel(kern, kThreadsWS, smem_bytes, &cache[parts][dev & 63], &per_sm);
  if (e) return e;
  uint64_t grid = (uint64_t)sms * (uint64_t)per_sm;
  if (grid > p.n_tiles) grid = p.n_tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreadsWS);
  cfg.dynamicSmemBytes = (size_t)smem_bytes;
  cfg.stream = (cudaStream_t)stream;
  static const bool no_pdl = [] {
    const char* e = std::getenv("LLAMA_NO_PDL");
    return e && *e == '1';
  }();
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = no_pdl ? 0 : 1;
  cudaError_t le = cudaLaunchKernelEx(&cfg, kern, p);
  count_launch();
  return le != cudaSuccess ? (int)le : (int)cudaGetLastError();
}

int launch_permute(const PermParams& p, int smem_bytes, void* stream) {
  if (p.n_tiles == 0) return 0;
  static const bool v1 = [] {
    const char* e = std::getenv("LLAMA_PERMUTE_V1");
    return e && *e == '1';
  }();
  if (p.tma && p.ns <= 4 && !v1) return launch_permute_ws(p, smem_bytes, stream);
  return launch_permute_v1(p, smem_bytes, stream);
}

}  // namespace llb
