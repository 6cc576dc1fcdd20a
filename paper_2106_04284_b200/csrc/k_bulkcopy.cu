// k_bulkcopy.cu -- identical layouts without padding ("copying ... if
// mapping and size are identical is trivial"): the blobs are streamed through
// shared memory by the TMA.  One thread per CTA drives a ring of NS stages:
// NS-1 chunk loads (cp.async.bulk global->shared, completion on an mbarrier)
// stay in flight while earlier chunks are stored (cp.async.bulk
// shared->global).  No thread touches the data.
#include "device.cuh"
#include "launch.hpp"

namespace llb {

namespace {
constexpr int kThreads = 32;
constexpr int kMaxStages = 8;
}  // namespace

struct Chunk {
  const uint8_t* s;
  uint8_t* d;
  uint32_t len;
};

__device__ __forceinline__ Chunk chunk_of(const BulkCopyParams& p, uint64_t c, int& b) {
  while (c >= p.cstart[b + 1]) ++b;  // c increases per CTA
  const uint64_t off = (c - p.cstart[b]) * p.CH;
  const uint64_t rem = p.bytes[b] - off;
  return Chunk{p.src[b] + off, p.dst[b] + off, (uint32_t)(rem < p.CH ? rem : p.CH)};
}

__global__ void __launch_bounds__(kThreads) k_bulkcopy(const __grid_constant__ BulkCopyParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  uint8_t* ring = smem + 128;
  if (threadIdx.x != 0) return;
  const uint64_t total = p.cstart[p.nb];
  const uint64_t n = blockIdx.x < total ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  for (uint32_t s = 0; s < p.NS; ++s) mbar_init(&bars[s], 1);
  fence_mbar_init();
  int bl = 0, bs = 0;  // blob cursors of the load and store streams
  auto load = [&](uint64_t i) {
    const Chunk c = chunk_of(p, blockIdx.x + i * gridDim.x, bl);
    uint64_t* bar = &bars[i % p.NS];
    const uint32_t body = c.len & ~15u;
    mbar_arrive_expect_tx(bar, body);
    if (body) bulk_g2s(ring + (size_t)(i % p.NS) * p.CH, c.s, body, bar);
  };
  for (uint64_t i = 0; i + 1 < p.NS && i < n; ++i) load(i);
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t s = (uint32_t)(i % p.NS);
    mbar_wait(&bars[s], (uint32_t)((i / p.NS) & 1));
    const Chunk c = chunk_of(p, blockIdx.x + i * gridDim.x, bs);
    const uint32_t body = c.len & ~15u;
    if (body) bulk_s2g(c.d, ring + (size_t)s * p.CH, body);
    bulk_commit();
    for (uint32_t q = body; q < c.len; ++q) c.d[q] = c.s[q];  // sub-16-byte blob tail
    if (i + p.NS - 1 < n) {
      bulk_wait_read<1>();  // the store of chunk i-1 has left its stage
      load(i + p.NS - 1);
    }
  }
  bulk_wait_all();
}

int launch_bulkcopy(const BulkCopyParams& p, void* stream) {
  const uint64_t total = p.cstart[p.nb];
  if (total == 0) return 0;
  const int smem = 128 + (int)(p.NS * p.CH);
  static LaunchCache cache[64];
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  int e = prepare_kernel(k_bulkcopy, kThreads, smem, &cache[dev & 63], &per_sm);
  if (e) return e;
  current_device_sms(&sms);
  uint64_t grid = (uint64_t)sms * (uint64_t)per_sm;
  if (grid > total) grid = total;
  k_bulkcopy<<<(unsigned)grid, kThreads, smem, (cudaStream_t)stream>>>(p);
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace llb
