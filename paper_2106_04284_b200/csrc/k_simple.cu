// k_simple.cu -- the element-wise kernels: the naive copy (the paper's
// comparison), the seeded input generator, the padding fill and the
// identity blob copy.
#include <atomic>

#include "device.cuh"
#include "launch.hpp"

namespace llb {

namespace {
std::atomic<uint64_t> g_launches{0};
constexpr int kThreads = 256;

int grid_for(uint64_t work, int per_sm) {
  int sms = 148;
  current_device_sms(&sms);
  uint64_t blocks = (work + kThreads - 1) / kThreads;
  uint64_t cap = (uint64_t)sms * (uint64_t)per_sm;
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : (int)blocks;
}
}  // namespace

uint64_t launch_count() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1); }

const char* cuda_error_string(int err) { return cudaGetErrorString((cudaError_t)err); }

int current_device_sms(int* sms) {
  static int cache[64] = {0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  if (dev >= 0 && dev < 64 && cache[dev] > 0) { *sms = cache[dev]; return 0; }
  int v = 0;
  e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return (int)e;
  if (dev >= 0 && dev < 64) cache[dev] = v;
  *sms = v;
  return 0;
}

int max_optin_smem(int* bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaDeviceGetAttribute(bytes, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
}

// ------------------------------------------------------------------ naive
// One thread per record, leaves in the inner loop, one s_k-byte element copy
// through both mappings' address functions.
// kTraced: also count every address resolution (Trace / Heatmap):
// each (record, leaf) is resolved once on each side.
template <bool kTraced>
__global__ void __launch_bounds__(kThreads) k_naive(const __grid_constant__ NaiveParams p) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t cnt = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.N; i += stride) {
    ++cnt;
    for (int k = 0; k < p.K; ++k) {
      const DevLeaf& sl = p.sl[k];
      const DevLeaf& dl = p.dl[k];
      // i = row-major rank of the array index; each side's storage position
      const uint64_t fs = p.relin ? lin_storage(i, p.slin) : i;
      const uint64_t fd = p.relin ? lin_storage(i, p.dlin) : i;
      const uint64_t os = leaf_offset(fs, sl), od = leaf_offset(fd, dl);
      copy_elem(p.db[dl.blob] + od, p.sb[sl.blob] + os, sl.size);
      if (kTraced) {
        trace_bytes(p.tr[0], sl.blob, os, sl.size);
        trace_bytes(p.tr[1], dl.blob, od, dl.size);
      }
    }
  }
  if (kTraced)
    for (int k = 0; k < p.K; ++k) {
      trace_hits(p.tr[0], k, cnt);
      trace_hits(p.tr[1], k, cnt);
    }
}

int launch_naive(const NaiveParams& p, void* stream) {
  if (p.N == 0) return 0;
  if (p.traced)
    k_naive<true><<<grid_for(p.N, 16), kThreads, 0, (cudaStream_t)stream>>>(p);
  else
    k_naive<false><<<grid_for(p.N, 16), kThreads, 0, (cudaStream_t)stream>>>(p);
  count_launch();
  return (int)cudaGetLastError();
}

// -------------------------------------------------------------- generator
// Input recipe (not the method): byte b of leaf k of record i is byte b of
// splitmix64(seed ^ (i*K + k)), written through the mapping's address function.
__global__ void __launch_bounds__(kThreads) k_gen(const __grid_constant__ GenParams p) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.N; i += stride) {
    for (int k = 0; k < p.K; ++k) {
      const DevLeaf& dl = p.dl[k];
      // a leaf that maps several records onto one place (One, B = 0) keeps
      // the last of them in index order, as a sequential generator would
      if (dl.B == 0 && i + dl.L < p.N) continue;
      uint64_t v = splitmix64(p.seed ^ (i * (uint64_t)p.K + (uint64_t)k));
      uint8_t* d = p.db[dl.blob] + leaf_offset(lin_storage(i, p.lin), dl);  // data follows the array index
      copy_elem(d, reinterpret_cast<const uint8_t*>(&v), dl.size);
    }
  }
}

int launch_gen(const GenParams& p, void* stream) {
  if (p.N == 0) return 0;
  k_gen<<<grid_for(p.N, 16), kThreads, 0, (cudaStream_t)stream>>>(p);
  count_launch();
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------- fill
__global__ void __launch_bounds__(kThreads) k_fill(const __grid_constant__ FillParams p) {
  const uint64_t total = p.vstart[p.nb];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t w = p.value * 0x01010101u;
  const uint4 v4 = make_uint4(w, w, w, w);
  int b = 0;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < total; v += stride) {
    while (v >= p.vstart[b + 1]) ++b;
    const uint64_t off = (v - p.vstart[b]) * 16;
    uint8_t* d = p.ptr[b] + off;
    if (off + 16 <= p.bytes[b]) {
      *reinterpret_cast<uint4*>(d) = v4;
    } else {
      for (uint64_t j = off; j < p.bytes[b]; ++j) p.ptr[b][j] = (uint8_t)p.value;
    }
  }
}

int launch_fill(const FillParams& p, void* stream) {
  if (p.vstart[p.nb] == 0) return 0;
  k_fill<<<grid_for(p.vstart[p.nb], 8), kThreads, 0, (cudaStream_t)stream>>>(p);
  count_launch();
  return (int)cudaGetLastError();
}

// -------------------------------------------------------------- blob copy
// Identical layouts without padding: each blob is copied verbatim.
// Four independent 16-byte vectors per thread in flight.
__global__ void __launch_bounds__(kThreads) k_blobcopy(const __grid_constant__ BlobCopyParams p) {
  const uint64_t total = p.vstart[p.nb];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  int b = 0;
  for (uint64_t v0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v0 < total; v0 += 4 * stride) {
    uint4 val[4];
    uint8_t* dp[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      dp[j] = nullptr;
      const uint64_t v = v0 + j * stride;
      if (v < total) {
        while (v >= p.vstart[b + 1]) ++b;
        const uint64_t off = (v - p.vstart[b]) * 16;
        if (off + 16 <= p.bytes[b]) {
          val[j] = __ldcs(reinterpret_cast<const uint4*>(p.src[b] + off));
          dp[j] = p.dst[b] + off;
        } else {
          for (uint64_t q = off; q < p.bytes[b]; ++q) p.dst[b][q] = p.src[b][q];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (dp[j]) __stcs(reinterpret_cast<uint4*>(dp[j]), val[j]);
  }
}

int launch_blobcopy(const BlobCopyParams& p, void* stream) {
  if (p.vstart[p.nb] == 0) return 0;
  k_blobcopy<<<grid_for(p.vstart[p.nb] / 4 + 1, 8), kThreads, 0, (cudaStream_t)stream>>>(p);
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace llb
