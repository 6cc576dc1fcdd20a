// k_run.cu -- the field-run copy (P:759-761 aosoa_copy, generalised): between
// two mappings whose leaves share contiguous runs of >= 16 bytes (SoA <->
// AoSoA, AoSoA_M <-> AoSoA_N, SoA MB <-> SB, ...), every 16-byte vector of a
// leaf is read and written directly, global -> registers -> global, with both
// sides coalesced.  No shared memory: there is nothing to permute inside a run.
#include "device.cuh"
#include "launch.hpp"

namespace llb {

namespace {
constexpr int kThreads = 256;
constexpr int kUnroll = 4;  // independent 16-byte loads in flight per thread
}  // namespace

__global__ void __launch_bounds__(kThreads) k_run(const __grid_constant__ RunParams p) {
  const uint64_t total = p.vstart[p.K];
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  int k = 0;
  for (uint64_t v0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v0 < total; v0 += kUnroll * stride) {
    uint4 val[kUnroll];
    uint8_t* dp[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      dp[j] = nullptr;
      const uint64_t v = v0 + j * stride;
      if (v < total) {
        while (v >= p.vstart[k + 1]) ++k;  // v is increasing per thread
        const DevLeaf& sl = p.sl[k];
        const DevLeaf& dl = p.dl[k];
        const uint32_t lg = 31 - __clz(sl.size);           // log2 s_k
        const uint64_t r = (v - p.vstart[k]) << (4 - lg);  // first record of the vector
        const uint8_t* s = p.sb[sl.blob] + nf_offset(r, p.s, sl);
        uint8_t* d = p.db[dl.blob] + nf_offset(r, p.d, dl);
        if (r + (16u >> lg) <= p.N) {
          val[j] = __ldcs(reinterpret_cast<const uint4*>(s));
          dp[j] = d;
        } else {  // last, partial vector of this leaf: the records left are contiguous on both sides
          for (uint64_t q = 0; q < (p.N - r) * sl.size; ++q) d[q] = s[q];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kUnroll; ++j)
      if (dp[j]) __stcs(reinterpret_cast<uint4*>(dp[j]), val[j]);
  }
}

int launch_run(const RunParams& p, void* stream) {
  const uint64_t total = p.vstart[p.K];
  if (total == 0) return 0;
  int sms = 148;
  current_device_sms(&sms);
  uint64_t blocks = (total + (uint64_t)kThreads * kUnroll - 1) / ((uint64_t)kThreads * kUnroll);
  const uint64_t cap = (uint64_t)sms * 8;  // 8 x 256 threads = full occupancy per SM
  if (blocks > cap) blocks = cap;
  k_run<<<(int)blocks, kThreads, 0, (cudaStream_t)stream>>>(p);
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace llb
