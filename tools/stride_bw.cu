// stride_bw.cu -- HBM efficiency of copies made of L-byte pieces at a large
// stride (the access pattern of a transposing copy's column-major side):
// 4096 x 16 KB matrix, pieces of L bytes taken row-fastest (strided) or
// column-fastest (streaming), on the read side, the write side or both.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stride_bw tools/stride_bw.cu && /tmp/stride_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr uint64_t ROWS = 4096, PITCH = 16384, BYTES = ROWS * PITCH;  // 64 MB per array

// mode bit 0: strided reads, bit 1: strided writes
__global__ void k_pieces(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, uint32_t L, int mode, int arrays) {
  const uint64_t per = BYTES / 16;  // 16-B units per array
  const uint64_t total = per * arrays;
  const uint32_t upp = L / 16;      // units per piece
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total; t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = t / per, u = t % per;
    const uint64_t p = u / upp, q = u % upp;
    // strided: piece p -> row p % ROWS, column piece p / ROWS; streaming: identity
    const uint64_t strided = ((p % ROWS) * PITCH + (p / ROWS) * L) + q * 16;
    const uint64_t linear = u * 16;
    const uint64_t so = a * BYTES + ((mode & 1) ? strided : linear);
    const uint64_t d_o = a * BYTES + ((mode & 2) ? strided : linear);
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(src + so));
    __stcs(reinterpret_cast<uint4*>(dst + d_o), v);
  }
}

int main() {
  const int arrays = 7;
  uint8_t *s, *d;
  cudaMalloc(&s, BYTES * arrays);
  cudaMalloc(&d, BYTES * arrays);
  cudaMemset(s, 1, BYTES * arrays);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode = 0; mode < 4; ++mode)
    for (uint32_t L : {32u, 64u, 128u, 256u, 512u, 1024u, 2048u}) {
      k_pieces<<<sms * 8, 256>>>(s, d, L, mode, arrays);
      cudaEventRecord(e0);
      for (int i = 0; i < 5; ++i) k_pieces<<<sms * 8, 256>>>(s, d, L, mode, arrays);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("mode %d (%s reads, %s writes) L=%5u: %.0f GB/s\n", mode, mode & 1 ? "strided" : "linear",
             mode & 2 ? "strided" : "linear", L, 2.0 * BYTES * arrays * 5 / (ms * 1e-3) / 1e9);
    }
  return 0;
}
