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
  static std::atomic<int> cache[64];  // zero-initialised (static storage)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  if (dev >= 0 && dev < 64) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c > 0) { *sms = c; return 0; }
  }
  int v = 0;
  e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return (int)e;
  if (dev >= 0 && dev < 64) cache[dev].store(v, std::memory_order_relaxed);
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

// -------------------------------------------------------------- transpose
// 2-d views of different linearisations (row / column-major / Morton, P:140-
// 142): a CTA moves 32x32-record tiles, reading them in the source's storage
// order (consecutive threads = consecutive source positions) into a
// leaf-major shared tile (32 x 32, XOR-swizzled against bank conflicts, see
// tile_slot), then writing them in the destination's storage order.
__device__ __forceinline__ void tile_order(uint32_t kind, uint32_t q, uint32_t& dy, uint32_t& dx) {
  if (kind == LLAMA_COL_MAJOR) {
    dy = q & 31;
    dx = q >> 5;
  } else if (kind == LLAMA_MORTON) {  // the last index supplies bit 0 (reading #26)
    dx = (q & 1) | ((q >> 1) & 2) | ((q >> 2) & 4) | ((q >> 3) & 8) | ((q >> 4) & 16);
    dy = ((q >> 1) & 1) | ((q >> 2) & 2) | ((q >> 3) & 4) | ((q >> 4) & 8) | ((q >> 5) & 16);
  } else {
    dy = q >> 5;
    dx = q & 31;
  }
}

// Slot of tile element (dy, dx): rows of 32 with an XOR swizzle chosen so that
// 32 lanes walking a row, a column, or a 4 x 8 Morton block hit 32 distinct
// banks (4-byte elements): bank = dx ^ f(dy), f(4a + b) = 8b + a.
__device__ __forceinline__ uint32_t tile_slot(uint32_t dy, uint32_t dx) {
  return dy * 32 + (dx ^ (((dy & 3) << 3) | (dy >> 2)));
}

// One element of `size` bytes; kAligned: every element of both sides is
// naturally aligned (planner), so a typed access without runtime checks.
template <bool kAligned>
__device__ __forceinline__ void move_elem(uint8_t* d, const uint8_t* s, uint32_t size) {
  if (!kAligned) {
    copy_elem(d, s, size);
    return;
  }
  switch (size) {
    case 8: *reinterpret_cast<uint64_t*>(d) = *reinterpret_cast<const uint64_t*>(s); break;
    case 4: *reinterpret_cast<uint32_t*>(d) = *reinterpret_cast<const uint32_t*>(s); break;
    case 2: *reinterpret_cast<uint16_t*>(d) = *reinterpret_cast<const uint16_t*>(s); break;
    default: *d = *s; break;
  }
}

// Each thread owns the tile positions q = tid + 256*j (j < 4) of a side's
// storage order; leaves in the outer loop so the four records' accesses of
// one leaf are independent.  kUniform: every leaf of a side shares L and B
// (not a split), so a record's block / lane are computed once, not per leaf.
template <bool kUniform>
__device__ __forceinline__ uint64_t tile_leaf_offset(uint64_t f, uint64_t q, uint64_t r, const DevLeaf& l) {
  if (!kUniform) return leaf_offset(f, l);
  return l.base + q * l.B + l.F + r * l.size;
}

// Per-CTA table of a linear side's leaves (built once per CTA in shared
// memory: one 16-byte load per leaf instead of the descriptor's fields from
// parameter space): element of record f at g + f * m, tile at tbz & 0xFFFFFF,
// leaf size tbz >> 24.
struct __align__(16) LinEnt {
  uint8_t* g;
  uint32_t m;
  uint32_t tbz;
};

// kLinear sides (every leaf either L = 1 or one block holding all records,
// fewer than 2^32 records): leaf element of record f at g + f * m (m = B for
// L = 1, the leaf size for one block); one 32-bit multiply-add into a 64-bit
// address instead of the block / lane split (a 64-bit division for SoA, L = N).
template <typename T, bool kLoad>
__device__ __forceinline__ void lin_leaf_t(uint8_t* t, uint8_t* g, uint32_t m, const uint32_t (&f)[4],
                                           const uint32_t (&e)[4], const bool (&ok)[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (ok[j]) {
      T* ge = reinterpret_cast<T*>(g + (uint64_t)f[j] * m);
      T* te = reinterpret_cast<T*>(t) + e[j];
      if (kLoad)
        *te = *ge;
      else
        *ge = *te;
    }
}

template <bool kAligned, bool kLoad>
__device__ __forceinline__ void lin_leaf(uint8_t* t, uint8_t* g, uint32_t m, uint32_t size, const uint32_t (&f)[4],
                                         const uint32_t (&e)[4], const bool (&ok)[4]) {
  if (kAligned) {
    switch (size) {
      case 4: lin_leaf_t<uint32_t, kLoad>(t, g, m, f, e, ok); return;
      case 8: lin_leaf_t<uint64_t, kLoad>(t, g, m, f, e, ok); return;
      case 2: lin_leaf_t<uint16_t, kLoad>(t, g, m, f, e, ok); return;
      case 1: lin_leaf_t<uint8_t, kLoad>(t, g, m, f, e, ok); return;
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (ok[j]) {
      uint8_t* ge = g + (uint64_t)f[j] * m;
      uint8_t* te = t + e[j] * size;
      if (kLoad)
        move_elem<kAligned>(te, ge, size);
      else
        move_elem<kAligned>(ge, te, size);
    }
}

// Element-wise source with linear sides whose leaves all have one naturally
// aligned size T: two leaves x four records per pass, so eight loads of a
// thread are in flight before the first is consumed (one leaf per pass: the
// shared store waits on its load before the next leaf's loads issue).
template <typename T, typename Get>
__device__ __forceinline__ void lin_load_fixed(uint8_t* tsm, const Get& get, int K, const uint32_t (&f)[4],
                                               const uint32_t (&e)[4], const bool (&ok)[4]) {
  constexpr int U = 2;
  for (int k0 = 0; k0 < K; k0 += U) {
    T v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k0 + u < K) {
        const LinEnt l = get(k0 + u);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (ok[j]) v[u][j] = *reinterpret_cast<const T*>(l.g + (uint64_t)f[j] * l.m);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k0 + u < K) {
        T* t = reinterpret_cast<T*>(tsm + (get(k0 + u).tbz & 0xFFFFFFu));
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (ok[j]) t[e[j]] = v[u][j];
      }
  }
}

// Raw AoS side of a full tile: its 1024 records in the side's storage order
// are 32 contiguous segments of 32 records (rows or columns) or, for Morton,
// one segment of 1024; moved as 16-byte vectors between global memory and a
// record-major shared buffer (record q of the storage order at q * S).
__device__ __forceinline__ void raw_tile(uint8_t* g0, uint8_t* raw, const DevLin& lin, uint64_t y0, uint64_t x0,
                                         uint32_t S, bool load) {
  const uint32_t nseg = lin.kind == LLAMA_MORTON ? 1 : 32;
  const uint32_t seg_vecs = (1024 / nseg) * S / 16;
  // segment j starts at the tile corner's position + j rows (row-major) or
  // + j columns (column-major); one Morton segment
  const uint64_t f0 = lin_storage2d(y0, x0, lin);
  const uint64_t fstep = lin.kind == LLAMA_ROW_MAJOR ? lin.ext[1] : lin.ext[0];
  for (uint32_t v = threadIdx.x; v < nseg * seg_vecs; v += kThreads) {
    const uint32_t j = v / seg_vecs, o = v - j * seg_vecs;
    uint4* g = reinterpret_cast<uint4*>(g0 + (f0 + j * fstep) * S) + o;
    uint4* r = reinterpret_cast<uint4*>(raw) + v;
    if (load)
      *r = __ldcs(g);
    else
      __stcs(g, *r);
  }
}

// kRaw: a raw AoS side exists (separate instantiation: the raw code costs
// registers, and element-only tiles are latency-bound, so occupancy matters)
template <bool kAligned, bool kUniform, bool kRaw, int kLin>
__global__ void __launch_bounds__(kThreads) k_transpose2d(const __grid_constant__ NaiveParams p) {
  extern __shared__ __align__(16) uint8_t tsm[];
  const uint64_t tiles_x = (p.W + 31) / 32, n_tiles = tiles_x * ((p.H + 31) / 32);
  uint8_t* raw = tsm + p.rawoff;
  // kLin: the leaf table, [0, K) source, [K, 2K) destination; in shared
  // memory when p.linoff != 0 (not with a raw side: its 56 KB of tile + raw
  // buffer for Particle7 fill a quarter SM exactly), else from parameters
  LinEnt* lt = reinterpret_cast<LinEnt*>(tsm + p.linoff);
  auto ent = [&](int i) -> LinEnt {
    const int k = i < p.K ? i : i - p.K;
    const DevLeaf& l = i < p.K ? p.sl[k] : p.dl[k];
    uint8_t* b = i < p.K ? const_cast<uint8_t*>(p.sb[l.blob]) : p.db[l.blob];
    return LinEnt{b + l.base + l.F, l.L == 1 ? (uint32_t)l.B : l.size, p.tbase[k] | (l.size << 24)};
  };
  if (kLin && p.linoff) {
    for (int i = threadIdx.x; i < 2 * p.K; i += kThreads) lt[i] = ent(i);
    __syncthreads();
  }
  for (uint64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t y0 = (t / tiles_x) * 32, x0 = (t % tiles_x) * 32;
    const bool full = y0 + 32 <= p.H && x0 + 32 <= p.W;
    // storage positions of the tile corner (the rest follow without divisions
    // or bit loops: a full aligned 32x32 block is 1024 consecutive Morton codes)

    uint64_t f[4], qb[4], rl[4];
    uint32_t e[4];
    bool ok[4];
    if (kRaw && p.sraw && full) {  // coalesced vectors in, then records -> the leaf-major tile
      raw_tile(const_cast<uint8_t*>(p.sb[p.sl[0].blob]) + p.sl[0].base, raw, p.slin, y0, x0, p.sS, true);
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t q = threadIdx.x + kThreads * j;
        uint32_t dy, dx;
        tile_order(p.slin.kind, q, dy, dx);
        e[j] = tile_slot(dy, dx);
        f[j] = (uint64_t)q * p.sS;
      }
      if (kAligned && kLin && p.tlinear == 4 && p.raw_typed) {  // one 4-byte size: typed, 32-bit offsets
        uint32_t fr[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) fr[j] = (uint32_t)f[j];
        for (int k = 0; k < p.K; ++k) {
          const uint32_t F = (uint32_t)p.sl[k].F;
          uint32_t* tk = reinterpret_cast<uint32_t*>(tsm + p.tbase[k]);
#pragma unroll
          for (int j = 0; j < 4; ++j) tk[e[j]] = *reinterpret_cast<const uint32_t*>(raw + fr[j] + F);
        }
      } else
      for (int k = 0; k < p.K; ++k) {
        const uint32_t size = p.sl[k].size, F = (uint32_t)p.sl[k].F;
        uint8_t* tk = tsm + p.tbase[k];
#pragma unroll
        for (int j = 0; j < 4; ++j) move_elem<kAligned>(tk + e[j] * size, raw + f[j] + F, size);
      }
      __syncthreads();
      goto store_phase;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t dy, dx;
      tile_order(p.slin.kind, threadIdx.x + kThreads * j, dy, dx);
      ok[j] = y0 + dy < p.H && x0 + dx < p.W;
      f[j] = ok[j] ? lin_storage2d(y0 + dy, x0 + dx, p.slin) : 0;
      e[j] = tile_slot(dy, dx);
      if (!kLin) {
        const DevLeaf& l0 = p.sl[0];
        qb[j] = l0.lshift != kNoShift ? (f[j] >> l0.lshift) : f[j] / l0.L;
        rl[j] = f[j] - qb[j] * l0.L;
      }
    }
    if (kLin == 4 || kLin == 8) {
      uint32_t fl[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) fl[j] = (uint32_t)f[j];
      auto get = [&](int k) { return p.linoff ? lt[k] : ent(k); };
      if (kLin == 4)
        lin_load_fixed<uint32_t>(tsm, get, p.K, fl, e, ok);
      else
        lin_load_fixed<uint64_t>(tsm, get, p.K, fl, e, ok);
    } else if (kLin) {
      uint32_t fl[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) fl[j] = (uint32_t)f[j];
      for (int k = 0; k < p.K; ++k) {
        const LinEnt l = p.linoff ? lt[k] : ent(k);
        lin_leaf<kAligned, true>(tsm + (l.tbz & 0xFFFFFFu), l.g, l.m, l.tbz >> 24, fl, e, ok);
      }
    } else
    for (int k = 0; k < p.K; ++k) {
      const DevLeaf l = p.sl[k];
      const uint8_t* sb = p.sb[l.blob];
      uint8_t* t = tsm + p.tbase[k];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (ok[j]) move_elem<kAligned>(t + e[j] * l.size, sb + tile_leaf_offset<kUniform>(f[j], qb[j], rl[j], l), l.size);
    }
    __syncthreads();
  store_phase:
    if (kRaw && p.draw && full) {  // the leaf-major tile -> records, then coalesced vectors out
      if (p.dpad) {  // destination padding goes out as 0 (reading #12)
        for (uint32_t o = 16 * threadIdx.x; o < 1024 * p.dS; o += 16 * kThreads)
          *reinterpret_cast<uint4*>(raw + o) = make_uint4(0, 0, 0, 0);
        __syncthreads();
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t q = threadIdx.x + kThreads * j;
        uint32_t dy, dx;
        tile_order(p.dlin.kind, q, dy, dx);
        e[j] = tile_slot(dy, dx);
        f[j] = (uint64_t)q * p.dS;
      }
      if (kAligned && kLin && p.tlinear == 4 && p.raw_typed) {
        uint32_t fr[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) fr[j] = (uint32_t)f[j];
        for (int k = 0; k < p.K; ++k) {
          const uint32_t F = (uint32_t)p.dl[k].F;
          const uint32_t* tk = reinterpret_cast<const uint32_t*>(tsm + p.tbase[k]);
#pragma unroll
          for (int j = 0; j < 4; ++j) *reinterpret_cast<uint32_t*>(raw + fr[j] + F) = tk[e[j]];
        }
      } else
      for (int k = 0; k < p.K; ++k) {
        const uint32_t size = p.dl[k].size, F = (uint32_t)p.dl[k].F;
        const uint8_t* tk = tsm + p.tbase[k];
#pragma unroll
        for (int j = 0; j < 4; ++j) move_elem<kAligned>(raw + f[j] + F, tk + e[j] * size, size);
      }
      __syncthreads();
      raw_tile(p.db[p.dl[0].blob] + p.dl[0].base, raw, p.dlin, y0, x0, p.dS, false);
      __syncthreads();
      continue;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t dy, dx;
      tile_order(p.dlin.kind, threadIdx.x + kThreads * j, dy, dx);
      ok[j] = y0 + dy < p.H && x0 + dx < p.W;
      f[j] = ok[j] ? lin_storage2d(y0 + dy, x0 + dx, p.dlin) : 0;
      e[j] = tile_slot(dy, dx);
      if (!kLin) {
        const DevLeaf& l0 = p.dl[0];
        qb[j] = l0.lshift != kNoShift ? (f[j] >> l0.lshift) : f[j] / l0.L;
        rl[j] = f[j] - qb[j] * l0.L;
      }
    }
    if (kLin) {  // (stores do not stall: the one-leaf pass; the two-leaf pass measured -3% here)
      uint32_t fl[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) fl[j] = (uint32_t)f[j];
      for (int k = 0; k < p.K; ++k) {
        const LinEnt l = p.linoff ? lt[p.K + k] : ent(p.K + k);
        lin_leaf<kAligned, false>(tsm + (l.tbz & 0xFFFFFFu), l.g, l.m, l.tbz >> 24, fl, e, ok);
      }
    } else
    for (int k = 0; k < p.K; ++k) {
      const DevLeaf l = p.dl[k];
      uint8_t* db = p.db[l.blob];
      const uint8_t* t = tsm + p.tbase[k];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (ok[j]) move_elem<kAligned>(db + tile_leaf_offset<kUniform>(f[j], qb[j], rl[j], l), t + e[j] * l.size, l.size);
    }
    __syncthreads();
  }
}

int launch_transpose2d(const NaiveParams& p, void* stream) {
  const uint64_t n_tiles = ((p.W + 31) / 32) * ((p.H + 31) / 32);
  if (n_tiles == 0) return 0;
  static LaunchCache cache[24][64];
  int dev = 0, per_sm = 1, sms = 148;
  cudaGetDevice(&dev);
  // index: aligned + 2 uniform + 4 raw (+ 8 linear, mixed leaf sizes; 16 / 20:
  // linear with one aligned 4- / 8-byte leaf size; linear sides are uniform)
  void (*const kerns[24])(NaiveParams) = {
      k_transpose2d<false, false, false, 0>, k_transpose2d<true, false, false, 0>,
      k_transpose2d<false, true, false, 0>,  k_transpose2d<true, true, false, 0>,
      k_transpose2d<false, false, true, 0>,  k_transpose2d<true, false, true, 0>,
      k_transpose2d<false, true, true, 0>,   k_transpose2d<true, true, true, 0>,
      nullptr, nullptr, k_transpose2d<false, true, false, 1>, k_transpose2d<true, true, false, 1>,
      nullptr, nullptr, k_transpose2d<false, true, true, 1>,  k_transpose2d<true, true, true, 1>,
      nullptr, k_transpose2d<true, true, false, 4>, nullptr, k_transpose2d<true, true, true, 4>,
      nullptr, k_transpose2d<true, true, false, 8>, nullptr, k_transpose2d<true, true, true, 8>};
  int v = (p.taligned ? 1 : 0) + (p.tuniform ? 2 : 0) + ((p.sraw || p.draw) ? 4 : 0);
  if (p.tuniform && p.tlinear) {
    // (only for an element-wise source: with a raw source the loads are
    // vectors and the variant's registers only cost occupancy, -5%)
    const int fixed = p.taligned && (p.tlinear == 4 || p.tlinear == 8) && !p.sraw;
    v = fixed ? (p.tlinear == 4 ? 16 : 20) + 1 + ((p.sraw || p.draw) ? 2 : 0) : v + 8;
  }
  auto kern = kerns[v];
  int e = prepare_kernel(kern, kThreads, (int)p.tsmem, &cache[v][dev & 63], &per_sm);
  if (e) return e;
  current_device_sms(&sms);
  uint64_t grid = (uint64_t)sms * per_sm;
  if (grid > n_tiles) grid = n_tiles;
  kern<<<(unsigned)grid, kThreads, p.tsmem, (cudaStream_t)stream>>>(p);
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
