// k_permute_direct.cu -- AoS <-> SoA for records with many leaves (HEP100,
// P:775): the tile permute's SoA side would be K TMA ops of T * s_k bytes per
// tile (100 ops of 64-512 B for HEP), so here only the AoS side goes through
// shared memory (one TMA op per tile, an ns-stage ring) and the SoA side is
// read / written element by element by the consumer warps: a warp takes one
// leaf of 32 consecutive records, so every global access is a contiguous
// 32 * s_k-byte run.  Warp-specialised like k_permute_ws:
//   AoS -> SoA: full[s]  source tile landed  (TMA -> consumers)
//               empty[s] consumers done      (consumers -> producer: refill)
//   SoA -> AoS: dfull[s] destination tile written (consumers -> producer: store)
//               dempty[s] its store read it out    (producer -> consumers)
#include "device.cuh"
#include "launch.hpp"

namespace llb {

namespace {
constexpr int kCons = 256;  // consumer threads
constexpr int kBars = 128;  // 2 rings x <= 8 stages x 8 B
}  // namespace

// Per-CTA leaf table in class order (after the ring and its 16-byte slack):
// one 16-byte shared load per leaf visit instead of a dependent chain of
// parameter-space loads (order[i], then the descriptor's fields).
struct __align__(16) DTab {
  uint8_t* gptr;
  uint32_t F;
  uint32_t a_img;  // bits 0-7; bits 8-31: staging offset (DirectLeaf::stg)
};
extern __shared__ __align__(128) uint8_t dsmem[];
__device__ __forceinline__ const DTab* dtab(const DirectParams& p) {
  return reinterpret_cast<const DTab*>(dsmem + kBars + (size_t)p.ns * p.stage + 16);
}

// An element of `s` bytes at a shared-memory address aligned to `a`.
__device__ __forceinline__ uint64_t sm_gather(const uint8_t* p, uint32_t s, uint32_t a) {
  if (a >= s) {
    switch (s) {
      case 8: return *reinterpret_cast<const uint64_t*>(p);
      case 4: return *reinterpret_cast<const uint32_t*>(p);
      case 2: return *reinterpret_cast<const uint16_t*>(p);
      default: return *p;
    }
  }
  if (a == 4)  // s == 8
    return (uint64_t)*reinterpret_cast<const uint32_t*>(p) | ((uint64_t)*reinterpret_cast<const uint32_t*>(p + 4) << 32);
  if (s == 1) return *p;
  // misaligned: the aligned 32-bit words covering the element, funnel-shifted
  // (pointer arithmetic on p keeps the shared address space: LDS, not LD)
  const uint32_t lo2 = (uint32_t)(reinterpret_cast<uintptr_t>(p) & 3);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(p - lo2);
  const uint32_t sh = 8 * lo2;
  const uint32_t w0 = w[0], w1 = w[1];
  const uint32_t lo = __funnelshift_r(w0, w1, sh);
  if (s <= 4) return s == 4 ? lo : (s == 2 ? (lo & 0xFFFFu) : lo);
  const uint32_t hi = __funnelshift_r(w1, w[2], sh);
  return (uint64_t)lo | ((uint64_t)hi << 32);
}

// The same for an element whose address is 4-byte aligned minus LO2 bytes
// at every record (record stride a multiple of 4: the word phase is a
// per-leaf constant), shifts fixed at compile time.
template <uint32_t SZ, uint32_t LO2>
__device__ __forceinline__ uint64_t sm_gather_ph(const uint8_t* p) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(p - LO2);
  if (SZ == 8) {
    if (LO2 == 0) return (uint64_t)w[0] | ((uint64_t)w[1] << 32);
    const uint32_t w1 = w[1];
    return (uint64_t)__funnelshift_r(w[0], w1, 8 * LO2) | ((uint64_t)__funnelshift_r(w1, w[2], 8 * LO2) << 32);
  }
  if (SZ == 4) return LO2 == 0 ? w[0] : __funnelshift_r(w[0], w[1], 8 * LO2);
  if (SZ == 2) return LO2 < 3 ? (w[0] >> (8 * LO2)) & 0xFFFFu : __funnelshift_r(w[0], w[1], 24) & 0xFFFFu;
  return (w[0] >> (8 * LO2)) & 0xFFu;
}

// Store an element whose first byte sits LO2 bytes past a 4-byte boundary
// (fixed per leaf when the record stride is a multiple of 4): the widest
// naturally aligned pieces, chosen at compile time (never touching the
// neighbouring leaves' bytes).
template <uint32_t SZ, uint32_t LO2, uint32_t OFF>
struct ScatterPh {
  static __device__ __forceinline__ void run(uint8_t* p, uint64_t v) {
    constexpr uint32_t a = LO2 + OFF, rem = SZ - OFF;
    constexpr uint32_t w = (a % 4 == 0 && rem >= 4) ? 4 : ((a % 2 == 0 && rem >= 2) ? 2 : 1);
    if (w == 4)
      *reinterpret_cast<uint32_t*>(p + OFF) = (uint32_t)(v >> (8 * OFF));
    else if (w == 2)
      *reinterpret_cast<uint16_t*>(p + OFF) = (uint16_t)(v >> (8 * OFF));
    else
      p[OFF] = (uint8_t)(v >> (8 * OFF));
    ScatterPh<SZ, LO2, OFF + w>::run(p, v);
  }
};
template <uint32_t SZ, uint32_t LO2>
struct ScatterPh<SZ, LO2, SZ> {
  static __device__ __forceinline__ void run(uint8_t*, uint64_t) {}
};

__device__ __forceinline__ void sm_scatter(uint8_t* p, uint64_t v, uint32_t s, uint32_t a) {
  if (a >= s) {
    switch (s) {
      case 8: *reinterpret_cast<uint64_t*>(p) = v; return;
      case 4: *reinterpret_cast<uint32_t*>(p) = (uint32_t)v; return;
      case 2: *reinterpret_cast<uint16_t*>(p) = (uint16_t)v; return;
      default: *p = (uint8_t)v; return;
    }
  }
  if (a == 4) {
    *reinterpret_cast<uint32_t*>(p) = (uint32_t)v;
    *reinterpret_cast<uint32_t*>(p + 4) = (uint32_t)(v >> 32);
  } else if (a == 2) {
    for (uint32_t j = 0; j < s; j += 2) *reinterpret_cast<uint16_t*>(p + j) = (uint16_t)(v >> (8 * j));
  } else {
    for (uint32_t j = 0; j < s; ++j) p[j] = (uint8_t)(v >> (8 * j));
  }
}

__device__ __forceinline__ uint64_t gl_load(const uint8_t* p, uint32_t s, uint32_t a) {
  if (a < s) {
    uint64_t v = 0;
    for (uint32_t j = 0; j < s; ++j) v |= (uint64_t)__ldcs(p + j) << (8 * j);
    return v;
  }
  switch (s) {
    case 8: return __ldcs(reinterpret_cast<const unsigned long long*>(p));
    case 4: return __ldcs(reinterpret_cast<const unsigned int*>(p));
    case 2: return __ldcs(reinterpret_cast<const unsigned short*>(p));
    default: return __ldcs(p);
  }
}

__device__ __forceinline__ void gl_store(uint8_t* p, uint64_t v, uint32_t s, uint32_t a) {
  if (a < s) {
    for (uint32_t j = 0; j < s; ++j) __stcs(p + j, (uint8_t)(v >> (8 * j)));
    return;
  }
  switch (s) {
    case 8: __stcs(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v); return;
    case 4: __stcs(reinterpret_cast<unsigned int*>(p), (unsigned int)v); return;
    case 2: __stcs(reinterpret_cast<unsigned short*>(p), (unsigned short)v); return;
    default: __stcs(p, (uint8_t)v); return;
  }
}

__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory"); }

template <uint32_t SZ> struct UT;
template <> struct UT<1> { typedef uint8_t T; };
template <> struct UT<2> { typedef uint16_t T; };
template <> struct UT<4> { typedef uint32_t T; };
template <> struct UT<8> { typedef unsigned long long T; };

// One class of leaves (equal size, alignment classes) for the tile's records
// lane and lane + 32: warps take the class's leaves in turn, kU at a time, so
// each lane has 2 * kU independent accesses in flight.
template <bool kA2S, uint32_t SZ, bool kImgA, bool kGlobA, bool kFull, int kPh = -1>
__device__ __forceinline__ void direct_class(const DirectParams& p, const DirectClass& c, uint8_t* img,
                                             uint64_t t0, uint32_t nrec, int warp, int lane) {
  typedef typename UT<SZ>::T U;
  constexpr int kU = kA2S ? 4 : (SZ == 8 ? 4 : 8);
  const bool ok0r = kFull || (uint32_t)lane < nrec, ok1r = kFull || (uint32_t)lane + 32 < nrec;
  const uint32_t r0 = (uint32_t)lane * p.S, r1 = ((uint32_t)lane + 32) * p.S;
  for (uint32_t i0 = c.k0 + warp; i0 < c.k1; i0 += kU * (kCons / 32)) {
    U v[kU][2];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t i = i0 + u * (kCons / 32);
      const bool has = i < c.k1;
      const DTab l = dtab(p)[has ? i : c.k0];
      const bool ok0 = has && ok0r, ok1 = has && ok1r;
      if (kA2S) {
        if (kImgA) {
          v[u][0] = ok0 ? *reinterpret_cast<const U*>(img + r0 + l.F) : U(0);
          v[u][1] = ok1 ? *reinterpret_cast<const U*>(img + r1 + l.F) : U(0);
        } else if (kPh >= 0) {
          v[u][0] = ok0 ? (U)sm_gather_ph<SZ, (kPh < 0 ? 0u : (uint32_t)kPh)>(img + r0 + l.F) : U(0);
          v[u][1] = ok1 ? (U)sm_gather_ph<SZ, (kPh < 0 ? 0u : (uint32_t)kPh)>(img + r1 + l.F) : U(0);
        } else {
          v[u][0] = ok0 ? (U)sm_gather(img + r0 + l.F, SZ, l.a_img & 0xFFu) : U(0);
          v[u][1] = ok1 ? (U)sm_gather(img + r1 + l.F, SZ, l.a_img & 0xFFu) : U(0);
        }
      } else {
        const U* g = reinterpret_cast<const U*>(l.gptr) + t0;
        if (kGlobA) {
          v[u][0] = ok0 ? __ldcs(g + lane) : U(0);
          v[u][1] = ok1 ? __ldcs(g + lane + 32) : U(0);
        } else {
          v[u][0] = ok0 ? (U)gl_load(reinterpret_cast<const uint8_t*>(g + lane), SZ, 1) : U(0);
          v[u][1] = ok1 ? (U)gl_load(reinterpret_cast<const uint8_t*>(g + lane + 32), SZ, 1) : U(0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t i = i0 + u * (kCons / 32);
      const bool has = i < c.k1;
      const DTab l = dtab(p)[has ? i : c.k0];
      const bool ok0 = has && ok0r, ok1 = has && ok1r;
      if (kA2S) {
        U* g = reinterpret_cast<U*>(l.gptr) + t0;
        if (kGlobA) {
          if (ok0) __stcs(g + lane, v[u][0]);
          if (ok1) __stcs(g + lane + 32, v[u][1]);
        } else {
          if (ok0) gl_store(reinterpret_cast<uint8_t*>(g + lane), v[u][0], SZ, 1);
          if (ok1) gl_store(reinterpret_cast<uint8_t*>(g + lane + 32), v[u][1], SZ, 1);
        }
      } else {
        if (kImgA) {
          if (ok0) *reinterpret_cast<U*>(img + r0 + l.F) = v[u][0];
          if (ok1) *reinterpret_cast<U*>(img + r1 + l.F) = v[u][1];
        } else if (kPh >= 0) {
          constexpr uint32_t ph = kPh < 0 ? 0u : (uint32_t)kPh;
          if (ok0) ScatterPh<SZ, ph, 0>::run(img + r0 + l.F, v[u][0]);
          if (ok1) ScatterPh<SZ, ph, 0>::run(img + r1 + l.F, v[u][1]);
        } else {
          if (ok0) sm_scatter(img + r0 + l.F, v[u][0], SZ, l.a_img & 0xFFu);
          if (ok1) sm_scatter(img + r1 + l.F, v[u][1], SZ, l.a_img & 0xFFu);
        }
      }
    }
  }
}

// The same for naturally aligned images whose record stride is an even
// number of words (HEP aligned: 480 B = 120 words): 32 lanes on one leaf of 32
// records would hit 4 banks (8-way conflicts), so a warp access covers 4
// leaves x 8 consecutive records (lane = 8 * leaf + record): at most 2-way
// conflicts, and each leaf still writes / reads a contiguous 8 * SZ-byte run.
template <bool kA2S, uint32_t SZ, bool kGlobA, bool kFull>
__device__ __forceinline__ void direct_class_mix(const DirectParams& p, const DirectClass& c, uint8_t* img,
                                                 uint64_t t0, uint32_t nrec, int warp, int lane) {
  typedef typename UT<SZ>::T U;
  const uint32_t sub = (uint32_t)lane >> 3, rl = (uint32_t)lane & 7;
  for (uint32_t g0 = c.k0 + 4 * warp; g0 < c.k1; g0 += 4 * (kCons / 32)) {
    const uint32_t i = g0 + sub;
    const bool has = i < c.k1;
    const DirectLeaf& l = p.leaf[p.order[has ? i : c.k0]];
    const uint32_t F = l.F;
    U* g = reinterpret_cast<U*>(l.gptr) + t0;
    U v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t r = 8 * q + rl;
      const bool ok = has && (kFull || r < nrec);
      if (kA2S) {
        v[q] = ok ? *reinterpret_cast<const U*>(img + r * p.S + F) : U(0);
      } else if (kGlobA) {
        v[q] = ok ? __ldcs(g + r) : U(0);
      } else {
        v[q] = ok ? (U)gl_load(reinterpret_cast<const uint8_t*>(g + r), SZ, 1) : U(0);
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t r = 8 * q + rl;
      if (!(has && (kFull || r < nrec))) continue;
      if (!kA2S) {
        *reinterpret_cast<U*>(img + r * p.S + F) = v[q];
      } else if (kGlobA) {
        __stcs(g + r, v[q]);
      } else {
        gl_store(reinterpret_cast<uint8_t*>(g + r), v[q], SZ, 1);
      }
    }
  }
}

// SoA -> AoS, a class of 4- / 8-byte leaves aligned in both the image and
// global memory: each element goes global -> shared by cp.async (LDGSTS), so
// a lane has every element of its share of the class in flight without
// holding registers (the register path waits on its loads every 8 leaves).
// Lane mapping as in direct_class_mix (p.mix) or direct_class.
template <uint32_t SZ, bool kFull>
__device__ __forceinline__ void direct_class_async(const DirectParams& p, const DirectClass& c, uint8_t* img,
                                                   uint64_t t0, uint32_t nrec, int warp, int lane) {
  typedef typename UT<SZ>::T U;
  const uint32_t base = smem_u32(img);
  if (p.mix) {
    const uint32_t sub = (uint32_t)lane >> 3, rl = (uint32_t)lane & 7;
    for (uint32_t g0 = c.k0 + 4 * warp; g0 < c.k1; g0 += 4 * (kCons / 32)) {
      const uint32_t i = g0 + sub;
      if (i >= c.k1) continue;
      const DTab l = dtab(p)[i];
      const U* g = reinterpret_cast<const U*>(l.gptr) + t0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t r = 8 * q + rl;
        if (kFull || r < nrec)
          asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(base + r * p.S + l.F), "l"(g + r),
                       "n"(SZ)
                       : "memory");
      }
    }
    return;
  }
  for (uint32_t i = c.k0 + warp; i < c.k1; i += kCons / 32) {
    const DTab l = dtab(p)[i];
    const U* g = reinterpret_cast<const U*>(l.gptr) + t0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t r = (uint32_t)lane + 32 * h;
      if (kFull || r < nrec)
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(base + r * p.S + l.F), "l"(g + r), "n"(SZ)
                     : "memory");
    }
  }
}


// SoA -> AoS, a misaligned 4- / 8-byte class of a fixed word phase: its
// elements land by cp.async in an aligned staging area (T per leaf, after
// the leaf table), and after the tile's wait they are scattered from there
// into the image in compile-time pieces -- no register round trip through
// global latency for them.

__device__ __forceinline__ uint8_t* dstage(const DirectParams& p) {
  return dsmem + kBars + (size_t)p.ns * p.stage + 16 + 16 * (size_t)p.K;
}

template <uint32_t SZ, bool kFull>
__device__ __forceinline__ void direct_stage_in(const DirectParams& p, const DirectClass& c, uint64_t t0,
                                                uint32_t nrec, int warp, int lane) {
  typedef typename UT<SZ>::T U;
  const uint32_t base = smem_u32(dstage(p));
  for (uint32_t i = c.k0 + warp; i < c.k1; i += kCons / 32) {
    const DTab l = dtab(p)[i];
    const U* g = reinterpret_cast<const U*>(l.gptr) + t0;
    const uint32_t st = base + (l.a_img >> 8);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t r = (uint32_t)lane + 32 * h;
      if (kFull || r < nrec)
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(st + r * SZ), "l"(g + r), "n"(SZ) : "memory");
    }
  }
}

template <uint32_t SZ, uint32_t PH, bool kFull>
__device__ __forceinline__ void direct_stage_out(const DirectParams& p, const DirectClass& c, uint8_t* img,
                                                 uint32_t nrec, int warp, int lane) {
  typedef typename UT<SZ>::T U;
  const uint8_t* stg = dstage(p);
  for (uint32_t i = c.k0 + warp; i < c.k1; i += kCons / 32) {
    const DTab l = dtab(p)[i];
    const U* st = reinterpret_cast<const U*>(stg + (l.a_img >> 8));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t r = (uint32_t)lane + 32 * h;
      if (kFull || r < nrec) ScatterPh<SZ, PH, 0>::run(img + r * p.S + l.F, st[r]);
    }
  }
}

// SoA -> AoS, an image-aligned class of 1- / 2-byte leaves whose SoA runs
// start 16-byte aligned (full tiles): each leaf's T * SZ-byte run lands in the
// staging area as 16-byte cp.async chunks ((leaf, chunk) pairs spread over
// all consumer threads), then moves into the image element by element.

template <uint32_t SZ>
__device__ __forceinline__ void direct_chunk_in(const DirectParams& p, const DirectClass& c, uint64_t t0, int tid) {
  constexpr uint32_t kCh = 64 * SZ / 16;  // chunks per leaf (T = 64)
  const uint32_t base = smem_u32(dstage(p));
  for (uint32_t x = tid; x < (c.k1 - c.k0) * kCh; x += kCons) {
    const uint32_t i = c.k0 + x / kCh, ch = x % kCh;
    const DTab l = dtab(p)[i];
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + (l.a_img >> 8) + 16 * ch),
                 "l"(l.gptr + t0 * SZ + 16 * ch)
                 : "memory");
  }
}

template <uint32_t SZ>
__device__ __forceinline__ void direct_chunk_out(const DirectParams& p, const DirectClass& c, uint8_t* img, int warp,
                                                 int lane) {
  typedef typename UT<SZ>::T U;
  const uint8_t* stg = dstage(p);
  for (uint32_t i = c.k0 + warp; i < c.k1; i += kCons / 32) {
    const DTab l = dtab(p)[i];
    const U* st = reinterpret_cast<const U*>(stg + (l.a_img >> 8));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t r = (uint32_t)lane + 32 * h;
      *reinterpret_cast<U*>(img + r * p.S + l.F) = st[r];
    }
  }
}

template <uint32_t SZ, bool kFull>
__device__ __forceinline__ void direct_stage_out_c(const DirectParams& p, const DirectClass& c, uint8_t* img,
                                                   uint32_t nrec, int warp, int lane) {
  switch ((c.kind >> 7) & 3) {
    case 0: direct_stage_out<SZ, 0, kFull>(p, c, img, nrec, warp, lane); break;
    case 1: direct_stage_out<SZ, 1, kFull>(p, c, img, nrec, warp, lane); break;
    case 2: direct_stage_out<SZ, 2, kFull>(p, c, img, nrec, warp, lane); break;
    default: direct_stage_out<SZ, 3, kFull>(p, c, img, nrec, warp, lane); break;
  }
}

template <bool kA2S, uint32_t SZ, bool kFull>
__device__ __forceinline__ void direct_class_a(const DirectParams& p, const DirectClass& c, uint8_t* img, uint64_t t0,
                                               uint32_t nrec, int warp, int lane) {
  if (p.mix && (c.kind & 16)) {
    if (c.kind & 32)
      direct_class_mix<kA2S, SZ, true, kFull>(p, c, img, t0, nrec, warp, lane);
    else
      direct_class_mix<kA2S, SZ, false, kFull>(p, c, img, t0, nrec, warp, lane);
    return;
  }
  if ((c.kind & 64) && (c.kind & 32)) {  // misaligned image leaf of a fixed word phase
    switch ((c.kind >> 7) & 3) {
      case 0: direct_class<kA2S, SZ, false, true, kFull, 0>(p, c, img, t0, nrec, warp, lane); return;
      case 1: direct_class<kA2S, SZ, false, true, kFull, 1>(p, c, img, t0, nrec, warp, lane); return;
      case 2: direct_class<kA2S, SZ, false, true, kFull, 2>(p, c, img, t0, nrec, warp, lane); return;
      default: direct_class<kA2S, SZ, false, true, kFull, 3>(p, c, img, t0, nrec, warp, lane); return;
    }
  }
  switch (c.kind & 48) {
    case 48: direct_class<kA2S, SZ, true, true, kFull>(p, c, img, t0, nrec, warp, lane); break;
    case 16: direct_class<kA2S, SZ, true, false, kFull>(p, c, img, t0, nrec, warp, lane); break;
    case 32: direct_class<kA2S, SZ, false, true, kFull>(p, c, img, t0, nrec, warp, lane); break;
    default: direct_class<kA2S, SZ, false, false, kFull>(p, c, img, t0, nrec, warp, lane); break;
  }
}

// one class through registers (the size-specialised loops above)
template <bool kA2S, bool kFull>
__device__ __forceinline__ void direct_class_regs(const DirectParams& p, const DirectClass& c, uint8_t* img,
                                                  uint64_t t0, uint32_t nrec, int warp, int lane) {
  switch (c.kind & 15) {
    case 8: direct_class_a<kA2S, 8, kFull>(p, c, img, t0, nrec, warp, lane); break;
    case 4: direct_class_a<kA2S, 4, kFull>(p, c, img, t0, nrec, warp, lane); break;
    case 2: direct_class_a<kA2S, 2, kFull>(p, c, img, t0, nrec, warp, lane); break;
    default: direct_class_a<kA2S, 1, kFull>(p, c, img, t0, nrec, warp, lane); break;
  }
}

// full tiles (every record present) and the partial last tile.  SoA -> AoS
// with cp.async: the planner orders the classes [0, e0) chunk-staged, [e0, e1)
// staged, [e1, e2) cp.async into the image, [e2, n) registers (partial tiles
// move the chunk-staged classes through registers: their runs would overrun).
template <bool kA2S, bool kFull>
__device__ __forceinline__ void direct_tile(const DirectParams& p, uint8_t* img, uint64_t t0, uint32_t nrec, int warp,
                                            int lane) {
  const bool as = !kA2S && p.async;
  const uint32_t e0 = as ? p.cat_end[0] : 0, e1 = as ? p.cat_end[1] : 0, e2 = as ? p.cat_end[2] : 0;
  if (as) {  // the cp.async classes first, then the register classes overlap them
    if (kFull)
      for (uint32_t ci = 0; ci < e0; ++ci) {
        const DirectClass c = p.cls[ci];
        if ((c.kind & 15) == 2)
          direct_chunk_in<2>(p, c, t0, warp * 32 + lane);
        else
          direct_chunk_in<1>(p, c, t0, warp * 32 + lane);
      }
    for (uint32_t ci = e0; ci < e1; ++ci) {
      const DirectClass c = p.cls[ci];
      if ((c.kind & 15) == 8)
        direct_stage_in<8, kFull>(p, c, t0, nrec, warp, lane);
      else
        direct_stage_in<4, kFull>(p, c, t0, nrec, warp, lane);
    }
    for (uint32_t ci = e1; ci < e2; ++ci) {
      const DirectClass c = p.cls[ci];
      if ((c.kind & 15) == 8)
        direct_class_async<8, kFull>(p, c, img, t0, nrec, warp, lane);
      else
        direct_class_async<4, kFull>(p, c, img, t0, nrec, warp, lane);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (!kFull)
      for (uint32_t ci = 0; ci < e0; ++ci) {
        const DirectClass c = p.cls[ci];  // (a copy: its fields stay in registers)
        direct_class_regs<kA2S, kFull>(p, c, img, t0, nrec, warp, lane);
      }
  }
  for (uint32_t ci = e2; ci < p.n_cls; ++ci) {
    const DirectClass c = p.cls[ci];
    direct_class_regs<kA2S, kFull>(p, c, img, t0, nrec, warp, lane);
  }
  if (as && e1 > 0) {  // the staged classes: wait for the tile's cp.asyncs, then copy out
    asm volatile("cp.async.wait_all;" ::: "memory");
    cons_sync();
    if (kFull)
      for (uint32_t ci = 0; ci < e0; ++ci) {
        const DirectClass c = p.cls[ci];
        if ((c.kind & 15) == 2)
          direct_chunk_out<2>(p, c, img, warp, lane);
        else
          direct_chunk_out<1>(p, c, img, warp, lane);
      }
    for (uint32_t ci = e0; ci < e1; ++ci) {
      const DirectClass c = p.cls[ci];
      if ((c.kind & 15) == 8)
        direct_stage_out_c<8, kFull>(p, c, img, nrec, warp, lane);
      else
        direct_stage_out_c<4, kFull>(p, c, img, nrec, warp, lane);
    }
  }
}

template <bool kA2S>
__global__ void __launch_bounds__(kCons + 32, 3) k_permute_direct(const __grid_constant__ DirectParams p) {
  uint8_t* smem = dsmem;
  uint64_t* ready = reinterpret_cast<uint64_t*>(smem);  // A2S: full; S2A: dfull
  uint64_t* freed = ready + 8;                         // A2S: empty; S2A: dempty
  uint8_t* ring = smem + kBars;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (!kA2S)  // destination padding bytes are never written: zero the ring once
    for (uint32_t o = 16 * tid; o < p.ns * p.stage; o += 16 * (kCons + 32))
      *reinterpret_cast<uint4*>(ring + o) = make_uint4(0, 0, 0, 0);
  for (uint32_t i = tid; i < p.K; i += kCons + 32) {
    const DirectLeaf& l = p.leaf[p.order[i]];
    const_cast<DTab*>(dtab(p))[i] = DTab{l.gptr, l.F, l.a_img | (l.stg << 8)};
  }
  if (tid == 0) {
    for (uint32_t s = 0; s < p.ns; ++s) {
      mbar_init(&ready[s], 1);
      mbar_init(&freed[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (kA2S && blockIdx.x == 0 && warp < kCons / 32)
    for (uint32_t g = 0; g < p.n_gaps; ++g)
      for (uint32_t o = tid; o < p.gap_len[g]; o += kCons) p.blobs[1][p.gap_blob[g]][p.gap_off[g] + o] = 0;

  const uint64_t first = blockIdx.x, stride = gridDim.x;
  const uint32_t n_my = first < p.n_tiles ? (uint32_t)((p.n_tiles - first + stride - 1) / stride) : 0;
  const int X = kA2S ? 0 : 1;  // the AoS side
  uint8_t* ag = p.blobs[X][p.ablob] + p.abase;
  auto tile_rec = [&](uint32_t i) -> uint32_t {
    const uint64_t t0 = (first + (uint64_t)i * stride) * p.T;
    return (uint32_t)(p.N - t0 < p.T ? p.N - t0 : p.T);
  };

  if (warp == kCons / 32) {  // --------------------------------- producer
    if (lane == 0) {
      if (kA2S) {
        auto load = [&](uint32_t i, uint32_t s) {
          const uint64_t t0 = (first + (uint64_t)i * stride) * p.T;
          const uint32_t body = (tile_rec(i) * p.S) & ~15u;
          mbar_arrive_expect_tx(&ready[s], body);
          if (body) bulk_g2s(ring + (size_t)s * p.stage, ag + t0 * p.S, body, &ready[s]);
        };
        for (uint32_t i = 0; i < p.ns && i < n_my; ++i) load(i, i);
        uint32_t s = 0, ph = 0;
        for (uint32_t i = 0; i + p.ns < n_my; ++i) {
          mbar_wait_sleep(&freed[s], ph);
          load(i + p.ns, s);
          if (++s == p.ns) { s = 0; ph ^= 1; }
        }
      } else {
        uint32_t s = 0, ph = 0;
        for (uint32_t i = 0; i < n_my; ++i) {
          const uint64_t t0 = (first + (uint64_t)i * stride) * p.T;
          const uint32_t body = (tile_rec(i) * p.S) & ~15u;
          mbar_wait_sleep(&ready[s], ph);
          if (body) bulk_s2g(ag + t0 * p.S, ring + (size_t)s * p.stage, body);
          bulk_commit();
          bulk_wait_read<0>();
          mbar_arrive(&freed[s]);
          if (++s == p.ns) { s = 0; ph ^= 1; }
        }
        bulk_wait_all();
      }
    }
    return;
  }
  // ------------------------------------------------------------ consumers
  uint32_t s = 0, ph = 0;
  for (uint32_t i = 0; i < n_my; ++i) {
    const uint64_t t0 = (first + (uint64_t)i * stride) * p.T;
    const uint32_t nrec = tile_rec(i);
    const uint32_t bytes = nrec * p.S, body = bytes & ~15u;
    uint8_t* img = ring + (size_t)s * p.stage;
    if (tid == 0) mbar_wait(kA2S ? &ready[s] : &freed[s], kA2S ? ph : ph ^ 1);
    cons_sync();
    if (kA2S && body < bytes) {  // sub-16-byte tail of the last tile
      for (uint32_t o = body + tid; o < bytes; o += kCons) img[o] = ag[t0 * p.S + o];
      cons_sync();
    }
    // classes of equal-size leaves, each a specialised loop (warp w takes a
    // class's leaves w, w+8, ...; records lane and lane + 32; T = 64)
    if (nrec == p.T)
      direct_tile<kA2S, true>(p, img, t0, nrec, warp, lane);
    else
      direct_tile<kA2S, false>(p, img, t0, nrec, warp, lane);
    if (!kA2S) {
      if (p.async) asm volatile("cp.async.wait_all;" ::: "memory");
      if (body < bytes) {  // the last tile's sub-16-byte tail goes out directly
        cons_sync();
        for (uint32_t o = body + tid; o < bytes; o += kCons) ag[t0 * p.S + o] = img[o];
      }
      fence_proxy_async_smem();  // generic-proxy image writes -> the TMA store's reads
    }
    cons_sync();
    if (tid == 0) mbar_arrive(kA2S ? &freed[s] : &ready[s]);
    if (++s == p.ns) { s = 0; ph ^= 1; }
  }
}

int launch_permute_direct(const DirectParams& p, void* stream) {
  if (p.n_tiles == 0) return 0;
  static LaunchCache cache[2][64];
  int dev = 0, per_sm = 1, sms = 148;
  cudaGetDevice(&dev);
  // + slack (funnel reads of the last element) + the leaf table + staging
  const int smem = kBars + (int)(p.ns * p.stage) + 16 + 16 * (int)p.K + (int)p.stg_bytes;
  auto kern = p.a2s ? k_permute_direct<true> : k_permute_direct<false>;
  int e = prepare_kernel(kern, kCons + 32, smem, &cache[p.a2s ? 1 : 0][dev & 63], &per_sm);
  if (e) return e;
  current_device_sms(&sms);
  uint64_t grid = (uint64_t)sms * per_sm;
  if (grid > p.n_tiles) grid = p.n_tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kCons + 32);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t le = cudaLaunchKernelEx(&cfg, kern, p);
  count_launch();
  return le != cudaSuccess ? (int)le : (int)cudaGetLastError();
}

}  // namespace llb
