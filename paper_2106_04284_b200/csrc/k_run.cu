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

// Work order is chunk-major: a CTA moves every leaf of one chunk of C records
// before the next chunk, so both sides' bytes of those records (runs of a few
// tens of bytes interleaved with other leaves, e.g. AoSoA8) are consumed in
// one short window -- DRAM rows and L2 lines are used whole.
__global__ void __launch_bounds__(kThreads) k_run(const __grid_constant__ RunParams p) {
  for (uint64_t c = blockIdx.x; c < p.n_chunks; c += gridDim.x) {
    const uint64_t r0 = c * p.C;
    int k = 0;
    for (uint32_t v0 = threadIdx.x; v0 < p.chunk_vecs; v0 += kUnroll * kThreads) {
      uint4 val[kUnroll];
      uint8_t* dp[kUnroll];
#pragma unroll
      for (int j = 0; j < kUnroll; ++j) {
        dp[j] = nullptr;
        const uint32_t v = v0 + j * kThreads;
        if (v < p.chunk_vecs) {
          while (v >= p.cvstart[k + 1]) ++k;  // v increases per thread
          const DevLeaf& sl = p.sl[k];
          const DevLeaf& dl = p.dl[k];
          const uint32_t lg = 31 - __clz(sl.size);  // log2 s_k
          const uint64_t r = r0 + ((uint64_t)(v - p.cvstart[k]) << (4 - lg));
          if (r < p.N) {
            const uint8_t* s = p.sb[sl.blob] + leaf_offset(r, sl);
            uint8_t* d = p.db[dl.blob] + leaf_offset(r, dl);
            if (r + (16u >> lg) <= p.N) {
              val[j] = __ldcs(reinterpret_cast<const uint4*>(s));
              dp[j] = d;
            } else {  // last, partial vector of a leaf: the records left are contiguous on both sides
              for (uint64_t q = 0; q < (p.N - r) * sl.size; ++q) d[q] = s[q];
            }
          }
        }
      }
#pragma unroll
      for (int j = 0; j < kUnroll; ++j)
        if (dp[j]) __stcs(reinterpret_cast<uint4*>(dp[j]), val[j]);
    }
  }
}

int launch_run(const RunParams& p, void* stream) {
  if (p.n_chunks == 0) return 0;
  int sms = 148;
  current_device_sms(&sms);
  uint64_t blocks = p.n_chunks;
  const uint64_t cap = (uint64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  k_run<<<(int)blocks, kThreads, 0, (cudaStream_t)stream>>>(p);
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace llb
