// device.cuh -- device helpers shared by the sm_100a kernels: the normal-form
// address function (P:451 blobNrAndOffset) and thin PTX wrappers for mbarrier
// and TMA bulk copies (cp.async.bulk, SASS UBLKCP).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "params.hpp"

namespace llb {

// i -> (i / L, i % L): shift/mask when L is a power of two.
__device__ __forceinline__ uint64_t block_of(uint64_t i, const DevSide& s) {
  return s.lshift != kNoShift ? (i >> s.lshift) : (i / s.L);
}

// off(i,k) = base_k + (i / L) * B + F_k + (i % L) * s_k
__device__ __forceinline__ uint64_t nf_offset(uint64_t i, const DevSide& s, const DevLeaf& l) {
  const uint64_t q = block_of(i, s);
  return l.base + q * s.B + l.F + (i - q * s.L) * l.size;
}

// Storage position of the record whose array index has row-major rank i
// (#26).
__device__ __forceinline__ uint64_t lin_storage(uint64_t i, const DevLin& l) {
  if (l.kind == LLAMA_ROW_MAJOR) return i;
  uint64_t idx[kMaxRank];
  for (int d = (int)l.rank - 1; d >= 0; --d) {
    idx[d] = i % l.ext[d];
    i /= l.ext[d];
  }
  uint64_t f = 0;
  if (l.kind == LLAMA_COL_MAJOR) {
    for (int d = (int)l.rank - 1; d >= 0; --d) f = f * l.ext[d] + idx[d];
    return f;
  }
  for (uint32_t b = 0; b < l.bits; ++b)  // MORTON
    for (uint32_t d = 0; d < l.rank; ++d) f |= ((idx[d] >> b) & 1ull) << (b * l.rank + (l.rank - 1 - d));
  return f;
}

// The same for a 2-d index (y, x) without divisions.
__device__ __forceinline__ uint64_t lin_storage2d(uint64_t y, uint64_t x, const DevLin& l) {
  if (l.kind == LLAMA_COL_MAJOR) return x * l.ext[0] + y;
  if (l.kind == LLAMA_MORTON) {
    uint64_t f = 0;
    for (uint32_t b = 0; b < l.bits; ++b) f |= (((y >> b) & 1ull) << (2 * b + 1)) | (((x >> b) & 1ull) << (2 * b));
    return f;
  }
  return y * l.ext[1] + x;
}

// Heatmap: one count per byte of a resolved range.
__device__ __forceinline__ void trace_bytes(const DevTrace& t, uint32_t blob, uint64_t off, uint32_t size) {
  if (!t.heat) return;
  uint32_t* h = t.heat + t.heat_base[blob] + off;
  for (uint32_t j = 0; j < size; ++j) atomicAdd(h + j, 1u);
}

// Trace: adds this thread's resolution count of leaf k, summed
// over the warp first (every lane of the warp must call it).
__device__ __forceinline__ void trace_hits(const DevTrace& t, int k, uint32_t cnt) {
  const uint32_t w = __reduce_add_sync(0xffffffffu, cnt);
  if (t.hits && (threadIdx.x & 31) == 0 && w) atomicAdd(t.hits + k, (unsigned long long)w);
}

// The same with the leaf's own L and B (composite Split / One mappings).
__device__ __forceinline__ uint64_t leaf_offset(uint64_t i, const DevLeaf& l) {
  const uint64_t q = l.lshift != kNoShift ? (i >> l.lshift) : (i / l.L);
  return l.base + q * l.B + l.F + (i - q * l.L) * l.size;
}

// Copies n bytes between arbitrary addresses using the widest naturally
// aligned access both pointers allow (never assumes alignment; packed
// layouts put f64 at odd offsets).
__device__ __forceinline__ void copy_elem(uint8_t* d, const uint8_t* s, uint32_t n) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(d) | reinterpret_cast<uintptr_t>(s);
  if (n == 8 && (a & 7) == 0) { *reinterpret_cast<uint64_t*>(d) = *reinterpret_cast<const uint64_t*>(s); return; }
  if (n == 4 && (a & 3) == 0) { *reinterpret_cast<uint32_t*>(d) = *reinterpret_cast<const uint32_t*>(s); return; }
  if (n == 2 && (a & 1) == 0) { *reinterpret_cast<uint16_t*>(d) = *reinterpret_cast<const uint16_t*>(s); return; }
  for (uint32_t j = 0; j < n; ++j) d[j] = s[j];
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "LLB_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra LLB_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// The same, but the waiting thread may be suspended (up to `hint_ns` per try)
// instead of spinning: for a producer lane whose spin would take issue slots
// from the consumer warps sharing its SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t hint_ns = 20000) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "LLB_WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra LLB_WAITS_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(hint_ns)
      : "memory");
}

// TMA bulk copy global -> shared, completion counted on an mbarrier.
// Requires 16-B aligned addresses and a 16-B multiple size.
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// TMA bulk copy shared -> global, tracked by the issuing thread's bulk groups.
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }

// Wait until at most N of this thread's bulk groups still read shared memory.
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Orders this thread's generic-proxy shared-memory writes before later
// async-proxy (TMA) reads of them.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Host side: per-device cache of a kernel's launch setup (these driver
// queries cost tens of microseconds; a copy should not pay them every launch).
// Thread-safe: the dynamic-smem limit is raised ONCE per kernel and device to
// the device's opt-in maximum (so no thread ever lowers it under another's
// launch), and the occupancy per shared-memory size is memoised under a mutex.
struct LaunchCache {
  std::mutex mu;
  bool attr_set = false;
  int n = 0;            // valid entries of smem / per_sm (ring replacement)
  int smem[8] = {};
  int per_sm[8] = {};
};

int max_optin_smem(int* bytes);  // k_simple.cu

template <typename K>
inline int prepare_kernel(K kernel, int threads, int smem_bytes, LaunchCache* cache, int* per_sm) {
  std::lock_guard<std::mutex> g(cache->mu);
  if (!cache->attr_set) {
    int mx = 0;
    int e = max_optin_smem(&mx);
    if (e) return e;
    cudaError_t ce = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
    if (ce != cudaSuccess) return (int)ce;
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cache->attr_set = true;
  }
  const int used = cache->n < 8 ? cache->n : 8;
  for (int j = 0; j < used; ++j)
    if (cache->smem[j] == smem_bytes) { *per_sm = cache->per_sm[j]; return 0; }
  int n = 1;
  cudaError_t ce = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem_bytes);
  if (ce != cudaSuccess) return (int)ce;
  const int slot = cache->n++ % 8;
  cache->smem[slot] = smem_bytes;
  cache->per_sm[slot] = n < 1 ? 1 : n;
  *per_sm = cache->per_sm[slot];
  return 0;
}

}  // namespace llb
