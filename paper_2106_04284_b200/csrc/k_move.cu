// k_move.cu -- the n-body move (Listing P:643-645):
//   Pos_c(i) = Pos_c(i) + Vel_c(i) * dt,  c in {X, Y, Z}, f32, one rounding
// (reading #25: a fused multiply-add, __fmaf_rn, as the paper's builds with
// -ffast-math -mfma / nvcc --use_fast_math contracted it).
//
// Kernels, one per layout family:
//   k_move_generic  thread per particle through the per-leaf normal form (any mapping)
//   k_move_runs     4 consecutive particles per thread, one 16-byte vector per leaf
//                   (SoA, AoSoA with L % 4 == 0, splits of those): 6 loads, 3 stores
//   k_move_aos_tma  packed / aligned AoS: tiles of whole records through a TMA
//                   ring in shared memory, Pos updated in place (default)
//   k_move_aos      the same with warp-staged coalesced 16-byte LSU accesses
//                   (LLAMA_MOVE_AOS_LSU=1; measured 17% slower)
// All are HBM-bound: algorithmic traffic 24 B read + 12 B written per particle;
// an AoS layout moves whole records (S read + S written).
#include "device.cuh"
#include "launch.hpp"

namespace llb {

namespace {
constexpr int kThreads = 256;

__device__ __forceinline__ float move1(float x, float v, float dt) { return __fmaf_rn(v, dt, x); }

__device__ __forceinline__ float load_f32(const uint8_t* a, bool aligned) {
  if (aligned) return *reinterpret_cast<const float*>(a);
  uint32_t w = (uint32_t)a[0] | ((uint32_t)a[1] << 8) | ((uint32_t)a[2] << 16) | ((uint32_t)a[3] << 24);
  return __uint_as_float(w);
}

__device__ __forceinline__ void store_f32(uint8_t* a, float x, bool aligned) {
  if (aligned) {
    *reinterpret_cast<float*>(a) = x;
    return;
  }
  const uint32_t w = __float_as_uint(x);
  a[0] = (uint8_t)w;
  a[1] = (uint8_t)(w >> 8);
  a[2] = (uint8_t)(w >> 16);
  a[3] = (uint8_t)(w >> 24);
}

int grid_for(uint64_t work, int per_sm) {
  int sms = 148;
  current_device_sms(&sms);
  uint64_t blocks = (work + kThreads - 1) / kThreads;
  const uint64_t cap = (uint64_t)sms * (uint64_t)per_sm;
  if (blocks > cap) blocks = cap;
  return blocks < 1 ? 1 : (int)blocks;
}
}  // namespace

// ---------------------------------------------------------------- generic
// Particles [i0, N) -- i0 > 0 when it finishes the tail of the AoS kernel.
// kTraced: count the resolutions (Trace / Heatmap): Pos_c once
// (the compound +=) and Vel_c once per particle.
template <bool kAligned, bool kTraced>
__global__ void __launch_bounds__(kThreads) k_move_generic(const __grid_constant__ MoveParams p, uint64_t i0) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t cnt = 0;
  for (uint64_t i = i0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.N; i += stride) {
    uint8_t* xa[3];
    float x[3], v[3];
    ++cnt;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const uint64_t op = leaf_offset(i, p.pos[c]), ov = leaf_offset(i, p.vel[c]);
      xa[c] = p.blobs[p.pos[c].blob] + op;
      x[c] = load_f32(xa[c], kAligned);
      v[c] = load_f32(p.blobs[p.vel[c].blob] + ov, kAligned);
      if (kTraced) {
        trace_bytes(p.tr, p.pos[c].blob, op, 4);
        trace_bytes(p.tr, p.vel[c].blob, ov, 4);
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) store_f32(xa[c], move1(x[c], v[c], p.dt), kAligned);
  }
  if (kTraced)
    for (int c = 0; c < 3; ++c) {
      trace_hits(p.tr, (int)p.lpos[c], cnt);
      trace_hits(p.tr, (int)p.lvel[c], cnt);
    }
}

int launch_move_generic_range(const MoveParams& p, uint64_t i0, void* stream) {
  if (p.N <= i0) return 0;
  const int grid = grid_for(p.N - i0, 16);
  if (p.traced && p.aligned)
    k_move_generic<true, true><<<grid, kThreads, 0, (cudaStream_t)stream>>>(p, i0);
  else if (p.traced)
    k_move_generic<false, true><<<grid, kThreads, 0, (cudaStream_t)stream>>>(p, i0);
  else if (p.aligned)
    k_move_generic<true, false><<<grid, kThreads, 0, (cudaStream_t)stream>>>(p, i0);
  else
    k_move_generic<false, false><<<grid, kThreads, 0, (cudaStream_t)stream>>>(p, i0);
  count_launch();
  return (int)cudaGetLastError();
}

int launch_move_generic(const MoveParams& p, void* stream) { return launch_move_generic_range(p, 0, stream); }

// ------------------------------------------------------------------- runs
// Particles 4q .. 4q+3 share one 16-byte vector of every Pos / Vel leaf
// (planner: runs of >= 4 records, 16-byte aligned).  All six vectors are
// loaded before any store (Pos and Vel may share a blob).
__global__ void __launch_bounds__(kThreads) k_move_runs(const __grid_constant__ MoveParams p) {
  const uint64_t nq = p.N / 4;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint64_t q = t; q < nq; q += stride) {
    const uint64_t i = 4 * q;
    float4* xa[3];
    float4 x[3], v[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      xa[c] = reinterpret_cast<float4*>(p.blobs[p.pos[c].blob] + leaf_offset(i, p.pos[c]));
      x[c] = __ldcs(xa[c]);
      v[c] = __ldcs(reinterpret_cast<const float4*>(p.blobs[p.vel[c].blob] + leaf_offset(i, p.vel[c])));
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float4 y;
      y.x = move1(x[c].x, v[c].x, p.dt);
      y.y = move1(x[c].y, v[c].y, p.dt);
      y.z = move1(x[c].z, v[c].z, p.dt);
      y.w = move1(x[c].w, v[c].w, p.dt);
      __stcs(xa[c], y);
    }
  }
  // the last N % 4 particles, one thread each
  if (t < p.N - 4 * nq) {
    const uint64_t i = 4 * nq + t;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      float* xp = reinterpret_cast<float*>(p.blobs[p.pos[c].blob] + leaf_offset(i, p.pos[c]));
      const float v = *reinterpret_cast<const float*>(p.blobs[p.vel[c].blob] + leaf_offset(i, p.vel[c]));
      *xp = move1(*xp, v, p.dt);
    }
  }
}

int launch_move_runs(const MoveParams& p, void* stream) {
  if (p.N == 0) return 0;
  k_move_runs<<<grid_for(p.N / 4 + 4, 8), kThreads, 0, (cudaStream_t)stream>>>(p);
  count_launch();
  return (int)cudaGetLastError();
}

// -------------------------------------------------------------------- AoS
// A warp owns chunks of 32*g whole records (W = 32*g*S bytes, a multiple of
// 512): coalesced 16-byte loads into its shared-memory slice, lane l updates
// records l, l+32, ... (record stride S: conflict-free when S/4 is odd, e.g.
// the 28-byte Particle7), coalesced 16-byte stores of the whole slice.  The
// partial last chunk is left to the generic kernel.
__global__ void __launch_bounds__(kThreads) k_move_aos(const __grid_constant__ MoveParams p) {
  extern __shared__ __align__(16) uint8_t smem_move[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t recs = 32 * p.g;              // records per chunk
  const uint32_t nvec = 2 * p.g * p.S;         // 16-byte vectors per chunk (W / 16)
  uint4* slice = reinterpret_cast<uint4*>(smem_move) + (size_t)warp * nvec;
  const uint64_t n_chunks = p.N / recs;
  const uint64_t gw = (uint64_t)blockIdx.x * (kThreads / 32) + warp, nw = (uint64_t)gridDim.x * (kThreads / 32);
  for (uint64_t c = gw; c < n_chunks; c += nw) {
    uint4* g = reinterpret_cast<uint4*>(p.blobs[p.blob] + p.base + c * (uint64_t)recs * p.S);
    uint32_t j = lane;
    for (; j + 96 < nvec; j += 128) {  // 4 independent loads in flight per lane
      const uint4 a = __ldcs(g + j), b = __ldcs(g + j + 32), d = __ldcs(g + j + 64), e = __ldcs(g + j + 96);
      slice[j] = a;
      slice[j + 32] = b;
      slice[j + 64] = d;
      slice[j + 96] = e;
    }
    for (; j < nvec; j += 32) slice[j] = __ldcs(g + j);
    __syncwarp();
    const uint8_t* sb = reinterpret_cast<const uint8_t*>(slice);
    for (uint32_t r = lane; r < recs; r += 32) {
      uint8_t* rec = const_cast<uint8_t*>(sb) + (size_t)r * p.S;
      float x[3], v[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        x[k] = *reinterpret_cast<const float*>(rec + p.fpos[k]);
        v[k] = *reinterpret_cast<const float*>(rec + p.fvel[k]);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) *reinterpret_cast<float*>(rec + p.fpos[k]) = move1(x[k], v[k], p.dt);
    }
    __syncwarp();
    for (j = lane; j < nvec; j += 32) __stcs(g + j, slice[j]);
    __syncwarp();
  }
}

// TMA variant (the default for AoS): tiles of T whole records move in and out
// of an NS-stage shared-memory ring with cp.async.bulk; the 8 consumer warps
// update Pos in place, the producer warp (one lane) stores the tile from the
// same stage and refills the stage once the store has read it out.
//   full[s]  the tile's bytes landed in stage s   (TMA -> consumers)
//   done[s]  consumers updated stage s            (consumers -> producer)
constexpr int kMoveConsumers = 256;

__global__ void __launch_bounds__(kMoveConsumers + 32, 1) k_move_aos_tma(const __grid_constant__ MoveParams p) {
  extern __shared__ __align__(128) uint8_t smem_tma[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_tma);
  uint64_t* done = full + 8;
  uint8_t* ring = smem_tma + 128;
  const uint32_t T = p.tile, NS = p.ns;
  const uint32_t tile_bytes = T * p.S;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (uint32_t s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&done[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint64_t n_tiles = p.N / T;  // whole tiles; the rest goes to the generic kernel
  const uint64_t first = blockIdx.x, stride = gridDim.x;
  const uint32_t n_my = first < n_tiles ? (uint32_t)((n_tiles - first + stride - 1) / stride) : 0;
  uint8_t* g0 = p.blobs[p.blob] + p.base;

  if (warp == kMoveConsumers / 32) {  // ------------------------------ producer
    if (lane == 0) {
      auto load = [&](uint32_t i, uint32_t s) {
        const uint64_t tile = first + (uint64_t)i * stride;
        mbar_arrive_expect_tx(&full[s], tile_bytes);
        bulk_g2s(ring + (size_t)s * tile_bytes, g0 + tile * tile_bytes, tile_bytes, &full[s]);
      };
      for (uint32_t i = 0; i < NS && i < n_my; ++i) load(i, i);
      uint32_t s = 0, ph = 0, sprev = NS - 1;
      for (uint32_t i = 0; i < n_my; ++i) {
        const uint64_t tile = first + (uint64_t)i * stride;
        mbar_wait(&done[s], ph);
        bulk_s2g(g0 + tile * tile_bytes, ring + (size_t)s * tile_bytes, tile_bytes);
        bulk_commit();
        // keep this store in flight; the previous tile's stage is free once
        // its store has been read out: refill it
        if (i > 0 && i - 1 + NS < n_my) {
          bulk_wait_read<1>();
          load(i - 1 + NS, sprev);
        }
        sprev = s;
        if (++s == NS) { s = 0; ph ^= 1; }
      }
      bulk_wait_all();
    }
    return;
  }
  // ------------------------------------------------------------- consumers
  uint32_t s = 0, ph = 0;
  for (uint32_t i = 0; i < n_my; ++i) {
    if (tid == 0) mbar_wait(&full[s], ph);
    asm volatile("bar.sync 1, %0;" ::"n"(kMoveConsumers) : "memory");
    uint8_t* img = ring + (size_t)s * tile_bytes;
    for (uint32_t r = tid; r < T; r += kMoveConsumers) {  // record stride S: conflict-free for odd S/4
      uint8_t* rec = img + (size_t)r * p.S;
      float x[3], v[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        x[k] = *reinterpret_cast<const float*>(rec + p.fpos[k]);
        v[k] = *reinterpret_cast<const float*>(rec + p.fvel[k]);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) *reinterpret_cast<float*>(rec + p.fpos[k]) = move1(x[k], v[k], p.dt);
    }
    fence_proxy_async_smem();  // generic-proxy writes -> the TMA store's reads
    asm volatile("bar.sync 1, %0;" ::"n"(kMoveConsumers) : "memory");
    if (tid == 0) mbar_arrive(&done[s]);
    if (++s == NS) { s = 0; ph ^= 1; }
  }
}

int launch_move_aos_tma(const MoveParams& p, void* stream) {
  const uint64_t n_tiles = p.N / p.tile;
  if (n_tiles) {
    const int smem = 128 + (int)(p.ns * p.tile * p.S);
    static LaunchCache cache[64];
    int dev = 0, per_sm = 1;
    cudaGetDevice(&dev);
    int e = prepare_kernel(k_move_aos_tma, kMoveConsumers + 32, smem, &cache[dev & 63], &per_sm);
    if (e) return e;
    int sms = 148;
    current_device_sms(&sms);
    uint64_t grid = (uint64_t)sms * per_sm;
    if (grid > n_tiles) grid = n_tiles;
    k_move_aos_tma<<<(unsigned)grid, kMoveConsumers + 32, smem, (cudaStream_t)stream>>>(p);
    count_launch();
    e = (int)cudaGetLastError();
    if (e) return e;
  }
  return launch_move_generic_range(p, n_tiles * p.tile, stream);  // the partial last tile
}

int launch_move_aos(const MoveParams& p, void* stream) {
  if (p.tile) return launch_move_aos_tma(p, stream);
  if (p.N == 0) return 0;
  const uint64_t recs = 32ull * p.g;
  const uint64_t n_chunks = p.N / recs;
  if (n_chunks) {
    const int smem = (kThreads / 32) * 2 * (int)p.g * (int)p.S * 16;
    static LaunchCache cache[64];
    int dev = 0, per_sm = 1;
    cudaGetDevice(&dev);
    int e = prepare_kernel(k_move_aos, kThreads, smem, &cache[dev & 63], &per_sm);
    if (e) return e;
    int sms = 148;
    current_device_sms(&sms);
    uint64_t grid = (uint64_t)sms * per_sm;
    const uint64_t need = (n_chunks + kThreads / 32 - 1) / (kThreads / 32);
    if (grid > need) grid = need;
    k_move_aos<<<(unsigned)grid, kThreads, smem, (cudaStream_t)stream>>>(p);
    count_launch();
    e = (int)cudaGetLastError();
    if (e) return e;
  }
  return launch_move_generic_range(p, n_chunks * recs, stream);  // the partial last chunk
}

}  // namespace llb
