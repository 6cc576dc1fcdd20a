// tools/tma_segments.cu -- microbenchmark (not part of the library): how fast
// can a warp-specialised TMA ring move a wide-record tile when one side is K
// small SoA segments (HEP100: 100 leaves, T * s_k bytes each) and the other
// one AoS segment?  No permute: consumers only hand stages back, so this is
// the ceiling of the TMA plumbing alone for the direct / JIT permute designs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_seg tools/tma_segments.cu
//   /tmp/tma_seg
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

struct P {
  const uint8_t* soa[128];
  uint8_t* soa_w[128];
  uint32_t sz[128];
  uint8_t* aos;
  const uint8_t* aos_r;
  uint64_t N;
  uint32_t K, T, S, Sp, ns, nd, s2a, lanes;  // lanes: producer lanes issuing the segment ops
  uint32_t chunks;     // 1: SoA source segments as 16-byte cp.async chunks (all 32 lanes, mbarrier arrive.noinc)
  uint32_t pad_smem;   // extra dynamic shared memory (fewer CTAs per SM)
};

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(sa(b)), "r"(ph) : "memory");
}

extern __shared__ __align__(128) uint8_t sm[];

__global__ void __launch_bounds__(288) k(const __grid_constant__ P p) {
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 8;
  uint64_t* dfull = full + 16;
  uint64_t* dempty = full + 24;
  uint8_t* src = sm + 256;
  const uint32_t sstage = p.T * (p.s2a ? p.Sp : p.S), dstage = p.T * (p.s2a ? p.S : p.Sp);
  uint8_t* dst = src + p.ns * sstage;
  const int tid = threadIdx.x, warp = tid >> 5;
  __shared__ uint32_t segoff[128];
  if (tid == 0) {
    uint32_t off = 0;
    for (uint32_t k = 0; k < p.K; ++k) { segoff[k] = off; off += p.T * p.sz[k]; }
    for (int i = 0; i < 8; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(full + i)), "r"(p.chunks ? 32u : 1u));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(empty + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(dfull + i)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(dempty + i)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint64_t nt = p.N / p.T;
  const uint32_t my = blockIdx.x < nt ? (uint32_t)((nt - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
  if (warp == 8) {
    const uint32_t lane = tid & 31;
    if (lane >= p.lanes) return;
    // segment offsets (prefix sums, same for every tile)
    auto load = [&](uint32_t i, uint32_t s) {
      const uint64_t t0 = (blockIdx.x + (uint64_t)i * gridDim.x) * p.T;
      uint8_t* d = src + s * sstage;
      if (p.chunks) {
        for (uint32_t k = 0; k < p.K; ++k) {
          const uint32_t n = p.T * p.sz[k] / 16;
          for (uint32_t c = lane; c < n; c += 32)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa(d + segoff[k] + 16 * c)),
                         "l"(p.soa[k] + t0 * p.sz[k] + 16 * c) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(full + s)) : "memory");
        return;
      }
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(full + s)), "r"(sstage));
      __syncwarp(p.lanes >= 32 ? 0xffffffffu : ((1u << p.lanes) - 1u));
      if (p.s2a) {
        for (uint32_t k = lane; k < p.K; k += p.lanes) {
          const uint32_t b = p.T * p.sz[k];
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d + segoff[k])),
                       "l"(p.soa[k] + t0 * p.sz[k]), "r"(b), "r"(sa(full + s)) : "memory");
        }
      } else if (lane == 0) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)),
                     "l"(p.aos_r + t0 * p.S), "r"(sstage), "r"(sa(full + s)) : "memory");
      }
    };
    for (uint32_t i = 0; i < p.ns && i < my; ++i) load(i, i);
    uint32_t s = 0, sph = 0, d = 0, dph = 0;
    for (uint32_t i = 0; i < my; ++i) {
      // consumers released the source stage of tile i and filled dst buffer d
      wait(&empty[s], sph);
      if (i + p.ns < my) load(i + p.ns, s);
      wait(&dfull[d], dph);
      const uint64_t t0 = (blockIdx.x + (uint64_t)i * gridDim.x) * p.T;
      uint8_t* img = dst + d * dstage;
      if (p.s2a) {
        if (lane == 0)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p.aos + t0 * p.S), "r"(sa(img)), "r"(dstage) : "memory");
      } else {
        for (uint32_t k = lane; k < p.K; k += p.lanes) {
          const uint32_t b = p.T * p.sz[k];
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p.soa_w[k] + t0 * p.sz[k]), "r"(sa(img + segoff[k])), "r"(b) : "memory");
        }
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp(p.lanes >= 32 ? 0xffffffffu : ((1u << p.lanes) - 1u));
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(dempty + d)) : "memory");
      if (++s == p.ns) { s = 0; sph ^= 1; }
      if (++d == p.nd) { d = 0; dph ^= 1; }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    return;
  }
  uint32_t s = 0, sph = 0, d = 0, dph = 0;
  for (uint32_t i = 0; i < my; ++i) {
    if (tid == 0) {
      wait(&full[s], sph);
      if (i >= p.nd) wait(&dempty[d], dph ^ 1);
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (tid == 0) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + s)) : "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(dfull + d)) : "memory");
    }
    if (++s == p.ns) { s = 0; sph ^= 1; }
    if (++d == p.nd) { d = 0; dph ^= 1; }
  }
}

int main() {
  // HEP100 leaf sizes (workloads.HEP100): 10 x {4,4,4,8,2,4,2,1,1,8}
  std::vector<uint32_t> sz;
  for (int g = 0; g < 10; ++g)
    for (uint32_t s : {4u, 4u, 4u, 8u, 2u, 4u, 2u, 1u, 1u, 8u}) sz.push_back(s);
  const uint32_t K = 100, Sp = 380;
  const uint64_t N = 1ull << 24;
  P p = {};
  p.K = K;
  p.N = N;
  p.Sp = Sp;
  std::vector<uint8_t*> a(K), b(K);
  for (uint32_t k = 0; k < K; ++k) {
    CK(cudaMalloc(&a[k], N * sz[k]));
    CK(cudaMalloc(&b[k], N * sz[k]));
    cudaMemset(a[k], 1, N * sz[k]);
    p.soa[k] = a[k];
    p.soa_w[k] = b[k];
    p.sz[k] = sz[k];
  }
  uint8_t *aos, *aos2;
  CK(cudaMalloc(&aos, N * 480));
  CK(cudaMalloc(&aos2, N * 480));
  cudaMemset(aos2, 1, N * 480);
  p.aos = aos;
  p.aos_r = aos2;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("dir        S    T  ns nd lanes chunks pad_KB smem_KB ctas/SM   GB/s\n");
  for (uint32_t s2a : {1u})
    for (uint32_t S : {380u})
      for (uint32_t T : {32u, 64u})
        for (uint32_t ns : {2u, 3u, 4u})
          for (uint32_t lanes : {32u})
          for (uint32_t chunks : {0u, 1u})
          for (uint32_t pad : {0u, 40u, 80u, 120u})
          for (uint32_t nd : {2u}) {
            p.lanes = lanes;
            p.chunks = chunks;
            p.pad_smem = pad * 1024;
            p.S = S;
            p.T = T;
            p.ns = ns;
            p.nd = nd;
            p.s2a = s2a;
            const uint32_t smem = 256 + ns * T * (s2a ? Sp : S) + nd * T * (s2a ? S : Sp) + p.pad_smem;
            if (smem > 226 * 1024) continue;
            int per = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 288, smem);
            if (per < 1) continue;
            const int grid = sms * per;
            k<<<grid, 288, smem>>>(p);
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            for (int r = 0; r < 5; ++r) k<<<grid, 288, smem>>>(p);
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double gbs = (double)N * (Sp + S) * 5 / (ms * 1e-3) / 1e9;
            printf("%s %4u %4u %3u %2u %5u %6u %6u %8.1f %7d %7.0f\n", s2a ? "SoA->AoS" : "AoS->SoA", S, T, ns, nd, lanes, chunks, pad, smem / 1024.0, per, gbs);
          }
  return 0;
}
