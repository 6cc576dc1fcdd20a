// k_transpose_wide.cu -- transposing copy of wide records (SURVEY §8(f) f4:
// rank-2 views of different storage orders; reading #26).
//
// The JIT transpose (jit_kernel2d.cuh) stages TY x 32-record tiles of every
// side; a 100-leaf HEP100 record (380 / 480 B) does not fit that.  Here a tile
// is 2^lty x 2^ltx records shaped per pair (WideParams): an AoS side ("A") is
// staged whole-record as a shared-memory image of the tile's storage runs
// (cp.async 16-/8-/4-byte chunks: contiguous global reads whatever the other
// side's order), an SoA / AoSoA side ("E") is read or written element by
// element with the warp's lanes along that side's own storage order, so every
// global access is coalesced.  E -> E pairs transpose each leaf through a
// shared-memory element buffer (32 x 32 elements, one pad element per 32).
#include "device.cuh"
#include "launch.hpp"

namespace llb {
namespace {

constexpr int kWT = 256;

__device__ __forceinline__ uint32_t part1by1(uint32_t x) {  // low 16 bits -> even bits
  x &= 0xFFFFu;
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

__device__ __forceinline__ uint32_t compact1by1(uint32_t x) {  // even bits -> low 16 bits
  x &= 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0F0F0F0Fu;
  x = (x | (x >> 4)) & 0x00FF00FFu;
  x = (x | (x >> 8)) & 0x0000FFFFu;
  return x;
}

__device__ __forceinline__ uint64_t spread64(uint64_t x) {  // low 32 bits -> even bits
  x &= 0xFFFFFFFFull;
  x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
  x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
  x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}

// Tile-local index t along a side's storage order -> (row r, column c).
// A Morton tile is 2^a x 2^a or 2^a x 2^(a+1) records at a multiple of its
// size, i.e. one contiguous run of codes (reading #26: x on the even bits).
__device__ __forceinline__ void t_rc(uint32_t lin, uint32_t t, uint32_t lty, uint32_t ltx, uint32_t& r,
                                     uint32_t& c) {
  if (lin == LLAMA_ROW_MAJOR) {
    r = t >> ltx;
    c = t & ((1u << ltx) - 1);
  } else if (lin == LLAMA_COL_MAJOR) {
    c = t >> lty;
    r = t & ((1u << lty) - 1);
  } else {
    c = compact1by1(t);
    r = compact1by1(t >> 1);
  }
}

__device__ __forceinline__ uint32_t rc_t(uint32_t lin, uint32_t r, uint32_t c, uint32_t lty, uint32_t ltx) {
  if (lin == LLAMA_ROW_MAJOR) return (r << ltx) | c;
  if (lin == LLAMA_COL_MAJOR) return (c << lty) | r;
  return part1by1(c) | (part1by1(r) << 1);
}

// storage position of array index (y, x)
__device__ __forceinline__ uint64_t storage2(uint32_t lin, uint64_t y, uint64_t x, uint64_t H, uint64_t W) {
  if (lin == LLAMA_ROW_MAJOR) return y * W + x;
  if (lin == LLAMA_COL_MAJOR) return x * H + y;
  return spread64(x) | (spread64(y) << 1);
}

// image offset of the block of the record at index t along the A side's own
// order (runs hold whole AoSoA-L blocks; plain AoS: L = 1), and its lane:
// leaf k of the record sits at img_off + F_k + lane * s_k
__device__ __forceinline__ uint32_t img_off(const WideSide& s, uint32_t t) {
  return (t >> s.lrun) * s.pitch + ((t & ((1u << s.lrun) - 1)) >> s.lL) * (uint32_t)s.B;
}
__device__ __forceinline__ uint32_t img_lane(const WideSide& s, uint32_t t) { return t & ((1u << s.lL) - 1); }

// hoisted block split of a uniform E side: off = leaf ptr + qB + rem * s_k
__device__ __forceinline__ void esplit(const WideSide& s, uint64_t p, uint64_t& qB, uint64_t& rem) {
  uint64_t q;
  if (s.lshift != kNoShift) {
    q = p >> s.lshift;
  } else {  // round-up multiplier (Granlund-Montgomery): exact for every 64-bit p, no division call
    const uint64_t t = __umul64hi(p, s.magic);
    q = (t + ((p - t) >> 1)) >> (s.mshift - 1);
  }
  qB = q * s.B;
  rem = p - q * s.L;
}

template <int U>
__device__ __forceinline__ uint64_t ld_unit(const uint8_t* s) {
  if constexpr (U == 8) return *reinterpret_cast<const uint64_t*>(s);
  if constexpr (U == 4) return *reinterpret_cast<const uint32_t*>(s);
  if constexpr (U == 2) return *reinterpret_cast<const uint16_t*>(s);
  return *s;
}

template <int U>
__device__ __forceinline__ void st_unit(uint8_t* d, uint64_t v) {
  if constexpr (U == 8) *reinterpret_cast<uint64_t*>(d) = v;
  if constexpr (U == 4) *reinterpret_cast<uint32_t*>(d) = (uint32_t)v;
  if constexpr (U == 2) *reinterpret_cast<uint16_t*>(d) = (uint16_t)v;
  if constexpr (U == 1) *d = (uint8_t)v;
}

// an SZ-byte element through accesses of U bytes (little endian)
template <int SZ, int U>
__device__ __forceinline__ uint64_t ld(const uint8_t* s) {
  uint64_t v = 0;
#pragma unroll
  for (int j = 0; j < SZ / U; ++j) v |= ld_unit<U>(s + j * U) << (8 * U * j);
  return v;
}

template <int SZ, int U>
__device__ __forceinline__ void st(uint8_t* d, uint64_t v) {
#pragma unroll
  for (int j = 0; j < SZ / U; ++j) st_unit<U>(d + j * U, v >> (8 * U * j));
}

// The per-record move loops issue the loads of KG leaves before their
// stores (KG = 2 where the loads are global or shared-memory reads whose
// latency would otherwise be exposed per element; 1 where only the stores
// are global, which do not block).

// (size, unit) -> one of the ten instantiations, f(integral_constant...) style
template <typename F>
__device__ __forceinline__ void dispatch(uint32_t size, uint32_t unit, F&& f) {
  switch (size * 16 + unit) {
    case 1 * 16 + 1: f.template run<1, 1>(); break;
    case 2 * 16 + 2: f.template run<2, 2>(); break;
    case 2 * 16 + 1: f.template run<2, 1>(); break;
    case 4 * 16 + 4: f.template run<4, 4>(); break;
    case 4 * 16 + 2: f.template run<4, 2>(); break;
    case 4 * 16 + 1: f.template run<4, 1>(); break;
    case 8 * 16 + 8: f.template run<8, 8>(); break;
    case 8 * 16 + 4: f.template run<8, 4>(); break;
    case 8 * 16 + 2: f.template run<8, 2>(); break;
    default: f.template run<8, 1>(); break;
  }
}

__device__ __forceinline__ void cp_async(uint8_t* s, const uint8_t* g, uint32_t n) {
  if (n == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
  else if (n == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(s)), "l"(g) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Tensor-map TMA (SASS UTMALDG / UTMASTG): the tile's runs of an A side as one box.
__device__ __forceinline__ void tma_load(uint8_t* sdst, const CUtensorMap* m, uint32_t rank, uint32_t c0, uint32_t c1,
                                         uint32_t c2, uint64_t* bar) {
  if (rank == 2)
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(smem_u32(sdst)), "l"(m), "r"(c0), "r"(c1), "r"(smem_u32(bar))
                 : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(sdst)), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_store(const CUtensorMap* m, uint32_t rank, uint32_t c0, uint32_t c1, uint32_t c2,
                                          const uint8_t* ssrc) {
  if (rank == 2)
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(m), "r"(c0),
                 "r"(c1), "r"(smem_u32(ssrc))
                 : "memory");
  else
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(m), "r"(c0),
                 "r"(c1), "r"(c2), "r"(smem_u32(ssrc))
                 : "memory");
}

struct Tile {
  uint64_t y0, x0;
  uint32_t h, w;  // valid rows / columns (ragged edge tiles)
};

// runs of an A side inside a tile: (count, records per valid run)
__device__ __forceinline__ void runs_of(const WideSide& s, const Tile& tl, uint32_t& nruns, uint32_t& len) {
  if (s.lin == LLAMA_ROW_MAJOR) nruns = tl.h, len = tl.w;
  else if (s.lin == LLAMA_COL_MAJOR) nruns = tl.w, len = tl.h;
  else nruns = 1, len = tl.h * tl.w;  // Morton tiles are always full
}

// global byte offset of run j's first record
__device__ __forceinline__ uint64_t run_start(const WideParams& p, const WideSide& s, const Tile& tl, uint32_t j) {
  uint32_t r, c;
  t_rc(s.lin, j << s.lrun, p.lty, p.ltx, r, c);
  return s.base + storage2(s.lin, tl.y0 + r, tl.x0 + c, p.H, p.W) * s.S;
}

// A source: the tile's runs -> image (cp.async; chunk-sized body, 4-byte tail)
__device__ __forceinline__ void load_image(const WideParams& p, const WideSide& s, const Tile& tl, uint8_t* img) {
  uint32_t nruns, len;
  runs_of(s, tl, nruns, len);
  const uint8_t* blob = p.sb[s.blob];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ch = s.chunk;
  const uint32_t bytes = len * s.S, body = bytes / ch * ch;
  if (nruns >= kWT / 32) {  // a warp per run
    for (uint32_t j = warp; j < nruns; j += kWT / 32) {
      const uint8_t* g = blob + run_start(p, s, tl, j);
      uint8_t* d = img + j * s.pitch;
      for (uint32_t u = lane * ch; u < body; u += 32 * ch) cp_async(d + u, g + u, ch);
      for (uint32_t u = body + lane * 4; u < bytes; u += 128) cp_async(d + u, g + u, 4);
    }
  } else {  // few long runs (a Morton tile is one): the whole CTA per run
    for (uint32_t j = 0; j < nruns; ++j) {
      const uint8_t* g = blob + run_start(p, s, tl, j);
      uint8_t* d = img + j * s.pitch;
      for (uint32_t u = threadIdx.x * ch; u < body; u += kWT * ch) cp_async(d + u, g + u, ch);
      for (uint32_t u = body + threadIdx.x * 4; u < bytes; u += kWT * 4) cp_async(d + u, g + u, 4);
    }
  }
}

template <int U, int STRIDE = 32>
__device__ __forceinline__ void copy_run(uint8_t* g, const uint8_t* s, uint32_t bytes, uint32_t lane) {
  for (uint32_t u = lane * U; u + U <= bytes; u += STRIDE * U) {
    if constexpr (U == 16) *reinterpret_cast<uint4*>(g + u) = *reinterpret_cast<const uint4*>(s + u);
    if constexpr (U == 8) *reinterpret_cast<uint2*>(g + u) = *reinterpret_cast<const uint2*>(s + u);
    if constexpr (U == 4) *reinterpret_cast<uint32_t*>(g + u) = *reinterpret_cast<const uint32_t*>(s + u);
  }
}

// A destination: image -> the tile's runs (vector stores; chunk-sized body, 4-byte tail)
__device__ __forceinline__ void flush_image(const WideParams& p, const WideSide& s, const Tile& tl,
                                            const uint8_t* img) {
  uint32_t nruns, len;
  runs_of(s, tl, nruns, len);
  uint8_t* blob = p.db[s.blob];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t bytes = len * s.S, body = bytes / s.chunk * s.chunk;
  if (nruns >= kWT / 32) {  // a warp per run
    for (uint32_t j = warp; j < nruns; j += kWT / 32) {
      uint8_t* g = blob + run_start(p, s, tl, j);
      const uint8_t* d = img + j * s.pitch;
      if (s.chunk == 16) copy_run<16>(g, d, body, lane);
      else if (s.chunk == 8) copy_run<8>(g, d, body, lane);
      else copy_run<4>(g, d, body, lane);
      copy_run<4>(g + body, d + body, bytes - body, lane);
    }
  } else {  // the whole CTA per run
    for (uint32_t j = 0; j < nruns; ++j) {
      uint8_t* g = blob + run_start(p, s, tl, j);
      const uint8_t* d = img + j * s.pitch;
      if (s.chunk == 16) copy_run<16, kWT>(g, d, body, threadIdx.x);
      else if (s.chunk == 8) copy_run<8, kWT>(g, d, body, threadIdx.x);
      else copy_run<4, kWT>(g, d, body, threadIdx.x);
      copy_run<4, kWT>(g + body, d + body, bytes - body, threadIdx.x);
    }
  }
}

__device__ __forceinline__ Tile tile_of(const WideParams& p, uint32_t tile) {
  Tile tl;
  uint32_t ty, tx;  // (32-bit: no division call)
  if (p.yfast) {
    const uint32_t nty = (uint32_t)p.nty;
    tx = tile / nty;
    ty = tile - tx * nty;
  } else {
    const uint32_t ntx = (uint32_t)p.ntx;
    ty = tile / ntx;
    tx = tile - ty * ntx;
  }
  tl.y0 = ty << p.lty;
  tl.x0 = tx << p.ltx;
  const uint64_t hh = p.H - tl.y0, ww = p.W - tl.x0;
  tl.h = (uint32_t)(hh < (1ull << p.lty) ? hh : (1ull << p.lty));
  tl.w = (uint32_t)(ww < (1ull << p.ltx) ? ww : (1ull << p.ltx));
  return tl;
}

// box coordinates of a tile on an A side (row-major: {x0 * S / e, y0};
// column-major: {0, y0 / g, x0})
__device__ __forceinline__ void box_coords(const WideSide& s, const Tile& tl, uint32_t& c0, uint32_t& c1,
                                           uint32_t& c2) {
  if (s.tma == 2) {
    c0 = (uint32_t)(tl.x0 * s.S / s.elsz);
    c1 = (uint32_t)tl.y0;
    c2 = 0;
  } else {
    c0 = 0;
    c1 = (uint32_t)(tl.y0 / s.g);
    c2 = (uint32_t)tl.x0;
  }
}

// A source image: one TMA box (thread 0 issues, every thread waits on the
// mbarrier's phase) or the cp.async run copies
__device__ __forceinline__ void load_src(const WideParams& p, const Tile& tl, uint8_t* smem, uint32_t& phase) {
  const WideSide& s = p.side[0];
  if (s.tma) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + p.bar);
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(bar, s.box_bytes);
      if (s.tma == 1) {  // a Morton tile: one contiguous run, one bulk copy (UBLKCP)
        bulk_g2s(smem + s.img, p.sb[s.blob] + run_start(p, s, tl, 0), s.box_bytes, bar);
      } else {
        uint32_t c0, c1, c2;
        box_coords(s, tl, c0, c1, c2);
        tma_load(smem + s.img, &p.tmap[0], s.tma, c0, c1, c2, bar);
      }
    }
    mbar_wait(bar, phase);
    phase ^= 1;
  } else {
    load_image(p, s, tl, smem + s.img);
    cp_async_wait_all();
  }
}

// A destination image -> global: one TMA box store (thread 0; the image is
// reused only after its read-out, hence wait_group.read before the barrier
// that ends the tile), or vector run stores.  The writers fenced their
// generic-proxy shared-memory writes before the preceding barrier.
__device__ __forceinline__ void flush_dst(const WideParams& p, const Tile& tl, uint8_t* smem) {
  const WideSide& s = p.side[1];
  if (s.tma) {
    if (threadIdx.x == 0) {
      if (s.tma == 1) {
        bulk_s2g(p.db[s.blob] + run_start(p, s, tl, 0), smem + s.img, s.box_bytes);
      } else {
        uint32_t c0, c1, c2;
        box_coords(s, tl, c0, c1, c2);
        tma_store(&p.tmap[1], s.tma, c0, c1, c2, smem + s.img);
      }
      bulk_commit();
      bulk_wait_read<0>();
    }
  } else {
    flush_image(p, s, tl, smem + s.img);
  }
}

// ---------------------------------------------------------------- moves
// A -> E: thread = (record t along the destination's order, leaf lane kl);
// a warp holds 32 consecutive destination records of one leaf: one coalesced
// store per leaf.
template <bool UNI>
struct MovesAE {
  const WideParams& p;
  const uint8_t* src;  // src image + block offset
  uint64_t qB, rem, pos;
  uint32_t j0, j1, kl, nl, ln;  // ln: the record's lane in its block
  template <int SZ, int U>
  __device__ __forceinline__ void run() {
    constexpr int KG = 1;
#pragma unroll 1
    for (uint32_t j = j0 + kl; j < j1; j += nl * KG) {
      uint64_t v[KG];
#pragma unroll
      for (int g = 0; g < KG; ++g)
        if (j + g * nl < j1) v[g] = ld<SZ, U>(src + p.leaf[j + g * nl].soff + ln * SZ);
#pragma unroll
      for (int g = 0; g < KG; ++g) {
        const uint32_t jj = j + g * nl;
        if (jj >= j1) break;
        uint8_t* d = UNI ? p.leaf[jj].dp + qB + rem * SZ : p.db[p.dl[jj].blob] + leaf_offset(pos, p.dl[jj]);
        st<SZ, U>(d, v[g]);
      }
    }
  }
};

// E -> A: thread = (record t along the source's order, leaf lane): coalesced loads
template <bool UNI>
struct MovesEA {
  const WideParams& p;
  uint8_t* dst;  // dst image + block offset
  uint64_t qB, rem, pos;
  uint32_t j0, j1, kl, nl, ln;
  template <int SZ, int U>
  __device__ __forceinline__ void run() {
    constexpr int KG = 2;
#pragma unroll 1
    for (uint32_t j = j0 + kl; j < j1; j += nl * KG) {
      uint64_t v[KG];
#pragma unroll
      for (int g = 0; g < KG; ++g) {
        const uint32_t jj = j + g * nl;
        if (jj >= j1) break;
        const uint8_t* s =
            UNI ? p.leaf[jj].sp + qB + rem * SZ : p.sb[p.sl[jj].blob] + leaf_offset(pos, p.sl[jj]);
        v[g] = ld<SZ, U>(s);
      }
#pragma unroll
      for (int g = 0; g < KG; ++g)
        if (j + g * nl < j1) st<SZ, U>(dst + p.leaf[j + g * nl].doff + ln * SZ, v[g]);
    }
  }
};

// A -> A with different record layouts: image -> image leaf moves
struct MovesAA {
  const WideParams& p;
  const uint8_t* src;
  uint8_t* dst;
  uint32_t j0, j1, kl, nl, sln, dln;
  template <int SZ, int U>
  __device__ __forceinline__ void run() {
    constexpr int KG = 2;
#pragma unroll 1
    for (uint32_t j = j0 + kl; j < j1; j += nl * KG) {
      uint64_t v[KG];
#pragma unroll
      for (int g = 0; g < KG; ++g)
        if (j + g * nl < j1) v[g] = ld<SZ, U>(src + p.leaf[j + g * nl].soff + sln * SZ);
#pragma unroll
      for (int g = 0; g < KG; ++g)
        if (j + g * nl < j1) st<SZ, U>(dst + p.leaf[j + g * nl].doff + dln * SZ, v[g]);
    }
  }
};

// ------------------------------------------------- 4-record groups (grp)
// A thread moves 4 consecutive records along the E side's storage order:
// one vector of 4 * s_k bytes on the E side (a leaf class whose group
// addresses are all 16-byte / 4 * s_k aligned, VEC) and 4 scalar accesses to
// the image.  4 elements of SZ bytes are packed into SZ 32-bit words.
// 4 elements of SZ bytes packed little endian into 4 * SZ bytes (two uint4 at most);
// the element index is a template argument, so the pack never leaves registers
struct Pk {
  uint4 a, b;
};

template <int I>
struct Ix {
  static constexpr int v = I;
};

template <typename F>
__device__ __forceinline__ void each4(F&& f) {
  f(Ix<0>{});
  f(Ix<1>{});
  f(Ix<2>{});
  f(Ix<3>{});
}

template <int W>
__device__ __forceinline__ uint32_t& word(Pk& k) {
  if constexpr (W == 0) return k.a.x;
  if constexpr (W == 1) return k.a.y;
  if constexpr (W == 2) return k.a.z;
  if constexpr (W == 3) return k.a.w;
  if constexpr (W == 4) return k.b.x;
  if constexpr (W == 5) return k.b.y;
  if constexpr (W == 6) return k.b.z;
  return k.b.w;
}

template <int SZ, int I>
__device__ __forceinline__ void pk_set(Pk& k, uint64_t v) {
  if constexpr (SZ == 1) word<0>(k) = I == 0 ? (uint32_t)v : (word<0>(k) | ((uint32_t)v << (8 * I)));
  if constexpr (SZ == 2) word<I / 2>(k) = (I & 1) ? (word<I / 2>(k) | ((uint32_t)v << 16)) : (uint32_t)v;
  if constexpr (SZ == 4) word<I>(k) = (uint32_t)v;
  if constexpr (SZ == 8) word<2 * I>(k) = (uint32_t)v, word<2 * I + 1>(k) = (uint32_t)(v >> 32);
}

template <int SZ, int I>
__device__ __forceinline__ uint64_t pk_get(Pk& k) {
  if constexpr (SZ == 1) return (word<0>(k) >> (8 * I)) & 0xFFu;
  if constexpr (SZ == 2) return (word<I / 2>(k) >> (16 * (I & 1))) & 0xFFFFu;
  if constexpr (SZ == 4) return word<I>(k);
  return (uint64_t)word<2 * I>(k) | ((uint64_t)word<2 * I + 1>(k) << 32);
}

template <int SZ>
__device__ __forceinline__ void vst(uint8_t* d, const Pk& k) {
  if constexpr (SZ == 1) *reinterpret_cast<uint32_t*>(d) = k.a.x;
  if constexpr (SZ == 2) *reinterpret_cast<uint2*>(d) = make_uint2(k.a.x, k.a.y);
  if constexpr (SZ == 4) *reinterpret_cast<uint4*>(d) = k.a;
  if constexpr (SZ == 8) reinterpret_cast<uint4*>(d)[0] = k.a, reinterpret_cast<uint4*>(d)[1] = k.b;
}

template <int SZ>
__device__ __forceinline__ void vld(const uint8_t* s, Pk& k) {
  if constexpr (SZ == 1) k.a.x = *reinterpret_cast<const uint32_t*>(s);
  if constexpr (SZ == 2) {
    const uint2 v = *reinterpret_cast<const uint2*>(s);
    k.a.x = v.x, k.a.y = v.y;
  }
  if constexpr (SZ == 4) k.a = *reinterpret_cast<const uint4*>(s);
  if constexpr (SZ == 8) k.a = reinterpret_cast<const uint4*>(s)[0], k.b = reinterpret_cast<const uint4*>(s)[1];
}

template <typename F>
__device__ __forceinline__ void dispatch_vec(uint32_t size, uint32_t unit, bool vec, F&& f) {
  switch (size * 32 + unit * 2 + (vec ? 1 : 0)) {
    case 1 * 32 + 1 * 2 + 1: f.template run<1, 1, true>(); break;
    case 1 * 32 + 1 * 2: f.template run<1, 1, false>(); break;
    case 2 * 32 + 2 * 2 + 1: f.template run<2, 2, true>(); break;
    case 2 * 32 + 2 * 2: f.template run<2, 2, false>(); break;
    case 2 * 32 + 1 * 2 + 1: f.template run<2, 1, true>(); break;
    case 2 * 32 + 1 * 2: f.template run<2, 1, false>(); break;
    case 4 * 32 + 4 * 2 + 1: f.template run<4, 4, true>(); break;
    case 4 * 32 + 4 * 2: f.template run<4, 4, false>(); break;
    case 4 * 32 + 2 * 2 + 1: f.template run<4, 2, true>(); break;
    case 4 * 32 + 2 * 2: f.template run<4, 2, false>(); break;
    case 4 * 32 + 1 * 2 + 1: f.template run<4, 1, true>(); break;
    case 4 * 32 + 1 * 2: f.template run<4, 1, false>(); break;
    case 8 * 32 + 8 * 2 + 1: f.template run<8, 8, true>(); break;
    case 8 * 32 + 8 * 2: f.template run<8, 8, false>(); break;
    case 8 * 32 + 4 * 2 + 1: f.template run<8, 4, true>(); break;
    case 8 * 32 + 4 * 2: f.template run<8, 4, false>(); break;
    case 8 * 32 + 2 * 2 + 1: f.template run<8, 2, true>(); break;
    case 8 * 32 + 2 * 2: f.template run<8, 2, false>(); break;
    case 8 * 32 + 1 * 2 + 1: f.template run<8, 1, true>(); break;
    default: f.template run<8, 1, false>(); break;
  }
}

// A -> E: image scalars -> one E vector per leaf (nv = valid records of the group)
struct GroupAE {
  const WideParams& p;
  const uint8_t* img;
  uint32_t ro0, ro1, ro2, ro3, ln0, ln1, ln2, ln3;
  uint64_t qB, rem;
  uint32_t nv, j0, j1, kl, nl;
  template <int SZ, int U, bool VEC>
  __device__ __forceinline__ void run() {
    const uint32_t ro[4] = {ro0 + ln0 * SZ, ro1 + ln1 * SZ, ro2 + ln2 * SZ, ro3 + ln3 * SZ};  // (+ lanes)
#pragma unroll 1
    for (uint32_t j = j0 + kl; j < j1; j += nl) {
      const uint32_t so = p.leaf[j].soff;
      Pk k{};
      each4([&](auto I) {
        if (I.v < (int)nv) pk_set<SZ, I.v>(k, ld<SZ, U>(img + ro[I.v] + so));
      });
      uint8_t* d = p.leaf[j].dp + qB + rem * SZ;
      if (VEC && nv == 4) {
        vst<SZ>(d, k);
      } else {
        each4([&](auto I) {
          if (I.v < (int)nv) st<SZ, U>(d + I.v * SZ, pk_get<SZ, I.v>(k));
        });
      }
    }
  }
};

// E -> A staged (stage): phase 1 moves every leaf's groups of the tile by
// cp.async into a staging area (leaf j: the tile's elements in E order at
// stg + buf_j), so all of a thread's loads are in flight at once; phase 2
// scatters them from shared memory into the image.
struct StageEA {
  const WideParams& p;
  uint8_t* stg;
  uint64_t qB, rem;
  uint32_t gi, nv, j0, j1, kl, nl;
  template <int SZ, int U, bool VEC>
  __device__ __forceinline__ void run() {
#pragma unroll 1
    for (uint32_t j = j0 + kl; j < j1; j += nl) {
      const WideLeaf& l = p.leaf[j];
      const uint8_t* s = l.sp + qB + rem * SZ;
      uint8_t* d = stg + l.buf + gi * 4 * SZ;
      if (VEC && nv == 4) {
        if constexpr (SZ == 8) {
          cp_async(d, s, 16);
          cp_async(d + 16, s + 16, 16);
        } else {
          cp_async(d, s, 4 * SZ);
        }
      } else {
        each4([&](auto I) {
          if (I.v < (int)nv) st<SZ, SZ>(d + I.v * SZ, ld<SZ, U>(s + I.v * SZ));
        });
      }
    }
  }
};

struct ScatterEA {
  const WideParams& p;
  const uint8_t* stg;
  uint8_t* img;
  uint32_t ro0, ro1, ro2, ro3, ln0, ln1, ln2, ln3;
  uint32_t gi, nv, j0, j1, kl, nl;
  template <int SZ, int U, bool VEC>
  __device__ __forceinline__ void run() {
    const uint32_t ro[4] = {ro0 + ln0 * SZ, ro1 + ln1 * SZ, ro2 + ln2 * SZ, ro3 + ln3 * SZ};  // (+ lanes)
#pragma unroll 1
    for (uint32_t j = j0 + kl; j < j1; j += nl) {
      const WideLeaf& l = p.leaf[j];
      Pk k{};
      vld<SZ>(stg + l.buf + gi * 4 * SZ, k);  // (the staging group is 4 * s_k-aligned)
      each4([&](auto I) {
        if (I.v < (int)nv) st<SZ, U>(img + ro[I.v] + l.doff, pk_get<SZ, I.v>(k));
      });
    }
  }
};

// E -> A: one E vector per leaf -> image scalars (two leaves' loads in flight)
struct GroupEA {
  const WideParams& p;
  uint8_t* img;
  uint32_t ro0, ro1, ro2, ro3, ln0, ln1, ln2, ln3;
  uint64_t qB, rem;
  uint32_t nv, j0, j1, kl, nl;
  template <int SZ, int U, bool VEC>
  __device__ __forceinline__ void ld_group(uint32_t j, Pk& k) {
    const uint8_t* s = p.leaf[j].sp + qB + rem * SZ;
    if (VEC && nv == 4) {
      vld<SZ>(s, k);
    } else {
      each4([&](auto I) {
        if (I.v < (int)nv) pk_set<SZ, I.v>(k, ld<SZ, U>(s + I.v * SZ));
      });
    }
  }
  template <int SZ, int U>
  __device__ __forceinline__ void st_group(uint32_t j, Pk& k, const uint32_t* ro) {
    const uint32_t doff = p.leaf[j].doff;
    each4([&](auto I) {
      if (I.v < (int)nv) st<SZ, U>(img + ro[I.v] + doff, pk_get<SZ, I.v>(k));
    });
  }
  template <int SZ, int U, bool VEC>
  __device__ __forceinline__ void run() {
    const uint32_t ro[4] = {ro0 + ln0 * SZ, ro1 + ln1 * SZ, ro2 + ln2 * SZ, ro3 + ln3 * SZ};  // (+ lanes)
    if constexpr (SZ >= 4 && U == SZ) {
      if (p.async) {  // (knob wide_async) 4- / 8-byte elements aligned on both sides: cp.async element copies
#pragma unroll 1
        for (uint32_t j = j0 + kl; j < j1; j += nl) {
          const uint8_t* s = p.leaf[j].sp + qB + rem * SZ;
          const uint32_t doff = p.leaf[j].doff;
          each4([&](auto I) {
            if (I.v < (int)nv) cp_async(img + ro[I.v] + doff, s + I.v * SZ, SZ);
          });
        }
        return;
      }
    }
    // LG leaves' loads in flight before their stores (4 while a pack is <= 16 bytes)
    constexpr int LG = SZ == 8 ? 2 : 4;
#pragma unroll 1
    for (uint32_t j = j0 + kl; j < j1; j += LG * nl) {
      Pk k[LG];
#pragma unroll
      for (int g = 0; g < LG; ++g) {
        k[g] = Pk{};
        if (j + g * nl < j1) ld_group<SZ, U, VEC>(j + g * nl, k[g]);
      }
#pragma unroll
      for (int g = 0; g < LG; ++g)
        if (j + g * nl < j1) st_group<SZ, U>(j + g * nl, k[g], ro);
    }
  }
};

// E -> E in 4-element groups (grp): the leaf's 32 x 32 tile sits in a
// shared-memory buffer in source order, 16-byte chunks of a 32-element run
// XOR-swizzled by (run / 4) % 8 (conflict-free transposed reads for 4-byte
// elements); a group is one cp.async of 4 * s_k bytes in, and 4 shared reads
// + one vector store out.
__device__ __forceinline__ uint32_t ee_off(uint32_t t) {  // element index of source-order t in the buffer
  const uint32_t run = t >> 5, q = (t >> 2) & 7;
  return (run << 5) + ((q ^ ((run >> 2) & 7)) << 2) + (t & 3);
}

struct LoadEEg {
  const WideParams& p;
  uint8_t* buf;
  uint64_t qB, rem;
  uint32_t off0, nv, j;
  template <int SZ, int U>
  __device__ __forceinline__ void run() {
    const WideLeaf& l = p.leaf[j];
    const uint8_t* s = l.sp + qB + rem * SZ;
    uint8_t* d = buf + l.buf + off0 * SZ;
    if (nv == 4 && (l.vec & 1)) {
      if constexpr (SZ == 8) {
        cp_async(d, s, 16);
        cp_async(d + 16, s + 16, 16);
      } else {
        cp_async(d, s, 4 * SZ);
      }
    } else {
      each4([&](auto I) {
        if (I.v < (int)nv) st<SZ, SZ>(d + I.v * SZ, ld<SZ, U>(s + I.v * SZ));
      });
    }
  }
};

struct StoreEEg {
  const WideParams& p;
  const uint8_t* buf;
  uint64_t qB, rem;
  uint32_t o0, o1, o2, o3, nv, j;
  template <int SZ, int U>
  __device__ __forceinline__ void run() {
    const WideLeaf& l = p.leaf[j];
    const uint8_t* b = buf + l.buf;
    const uint32_t o[4] = {o0, o1, o2, o3};
    Pk k{};
    each4([&](auto I) {
      if (I.v < (int)nv) pk_set<SZ, I.v>(k, ld<SZ, SZ>(b + o[I.v] * SZ));
    });
    uint8_t* d = l.dp + qB + rem * SZ;
    if (nv == 4 && (l.vec & 2)) {
      vst<SZ>(d, k);
    } else {
      each4([&](auto I) {
        if (I.v < (int)nv) st<SZ, U>(d + I.v * SZ, pk_get<SZ, I.v>(k));
      });
    }
  }
};

// E -> E, one leaf of a batch: 4 records per thread (1024-record tiles)
template <bool UNI>
struct LoadEE {
  const WideParams& p;
  uint8_t* buf;
  const uint64_t* qB;
  const uint64_t* rem;
  const uint64_t* pos;
  const uint32_t* idx;
  uint32_t valid, j;
  template <int SZ, int U>
  __device__ __forceinline__ void run() {
    const WideLeaf& l = p.leaf[j];
    uint64_t v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (valid >> i & 1) {
        const uint8_t* s = UNI ? l.sp + qB[i] + rem[i] * SZ : p.sb[p.sl[j].blob] + leaf_offset(pos[i], p.sl[j]);
        v[i] = ld<SZ, U>(s);
      }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (valid >> i & 1) st<SZ, SZ>(buf + l.buf + idx[i] * SZ, v[i]);
  }
};

template <bool UNI>
struct StoreEE {
  const WideParams& p;
  const uint8_t* buf;
  const uint64_t* qB;
  const uint64_t* rem;
  const uint64_t* pos;
  const uint32_t* idx;
  uint32_t valid, j;
  template <int SZ, int U>
  __device__ __forceinline__ void run() {
    const WideLeaf& l = p.leaf[j];
    uint64_t v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (valid >> i & 1) v[i] = ld<SZ, SZ>(buf + l.buf + idx[i] * SZ);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (valid >> i & 1) {
        uint8_t* d = UNI ? l.dp + qB[i] + rem[i] * SZ : p.db[p.dl[j].blob] + leaf_offset(pos[i], p.dl[j]);
        st<SZ, U>(d, v[i]);
      }
  }
};

template <int MODE, bool UNI, bool GRP, int MINB>
__global__ void __launch_bounds__(kWT, MINB) k_transpose_wide(const __grid_constant__ WideParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const WideSide& S0 = p.side[0];
  const WideSide& S1 = p.side[1];
  const uint32_t tid = threadIdx.x, lt = p.lty + p.ltx, n = 1u << lt;
  uint32_t phase = 0;  // of the TMA mbarrier (source box loads)
  if (S0.tma) {
    if (tid == 0) {
      mbar_init(reinterpret_cast<uint64_t*>(smem + p.bar), 1);
      fence_mbar_init();
    }
    __syncthreads();
  }
  if ((MODE == 1 || MODE == 2) && p.dzero) {  // padding bytes of the destination image stay 0
    for (uint32_t u = tid * 16; u < S1.img_bytes; u += kWT * 16)
      *reinterpret_cast<uint4*>(smem + S1.img + u) = make_uint4(0, 0, 0, 0);
    __syncthreads();
  }
  // thread -> (record t, leaf lane kl of nl) for tiles of <= 256 records
  const uint32_t nl = n >= kWT ? 1 : kWT >> lt, kl = n >= kWT ? 0 : tid >> lt, t0 = tid & (n - 1);
  for (uint32_t item = blockIdx.x; item < (uint32_t)p.n_items; item += gridDim.x) {
    if constexpr (MODE == 4 && GRP) {
      const uint32_t tile = item / p.nbatch;
      const uint32_t b = item - tile * p.nbatch;
      const Tile tl = tile_of(p, tile);
      uint8_t* buf = smem + p.buf;
      const uint32_t t0 = 4 * tid;  // this thread's group: source order (load), destination order (store)
      uint32_t nv = 0, r0 = 0, c0 = 0;
      each4([&](auto I) {
        uint32_t r, c;
        t_rc(S0.lin, t0 + I.v, p.lty, p.ltx, r, c);
        if (I.v == 0) r0 = r, c0 = c;
        if (r < tl.h && c < tl.w && nv == (uint32_t)I.v) ++nv;
      });
      uint64_t qB = 0, rem = 0;
      if (nv) esplit(S0, storage2(S0.lin, tl.y0 + r0, tl.x0 + c0, p.H, p.W), qB, rem);
      if (nv) {
#pragma unroll 1
        for (uint32_t j = p.bstart[b]; j < p.bstart[b + 1]; ++j)
          dispatch(p.leaf[j].size, p.leaf[j].unit, LoadEEg{p, buf, qB, rem, ee_off(t0), nv, j});
      }
      cp_async_wait_all();
      __syncthreads();
      uint32_t o[4];
      nv = 0;
      each4([&](auto I) {
        uint32_t r, c;
        t_rc(S1.lin, t0 + I.v, p.lty, p.ltx, r, c);
        if (I.v == 0) r0 = r, c0 = c;
        o[I.v] = ee_off(rc_t(S0.lin, r, c, p.lty, p.ltx));
        if (r < tl.h && c < tl.w && nv == (uint32_t)I.v) ++nv;
      });
      if (nv) {
        esplit(S1, storage2(S1.lin, tl.y0 + r0, tl.x0 + c0, p.H, p.W), qB, rem);
#pragma unroll 1
        for (uint32_t j = p.bstart[b]; j < p.bstart[b + 1]; ++j)
          dispatch(p.leaf[j].size, p.leaf[j].unit, StoreEEg{p, buf, qB, rem, o[0], o[1], o[2], o[3], nv, j});
      }
      __syncthreads();
    } else if constexpr (MODE == 4) {
      const uint32_t tile = item / p.nbatch;
      const uint32_t b = item - tile * p.nbatch;
      const Tile tl = tile_of(p, tile);
      uint8_t* buf = smem + p.buf;
      uint64_t qB[4], rem[4], pos[4];
      uint32_t idx[4], valid = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // source order
        uint32_t r, c;
        const uint32_t t = tid + i * kWT;
        t_rc(S0.lin, t, p.lty, p.ltx, r, c);
        qB[i] = rem[i] = 0;
        idx[i] = t + (t >> 5);
        pos[i] = 0;
        if (r < tl.h && c < tl.w) {
          valid |= 1u << i;
          pos[i] = storage2(S0.lin, tl.y0 + r, tl.x0 + c, p.H, p.W);
          if (UNI) esplit(S0, pos[i], qB[i], rem[i]);
        }
      }
#pragma unroll 1
      for (uint32_t j = p.bstart[b]; j < p.bstart[b + 1]; ++j)
        dispatch(p.leaf[j].size, p.leaf[j].unit, LoadEE<UNI>{p, buf, qB, rem, pos, idx, valid, j});
      __syncthreads();
      valid = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {  // destination order
        uint32_t r, c;
        const uint32_t t = tid + i * kWT;
        t_rc(S1.lin, t, p.lty, p.ltx, r, c);
        const uint32_t ts = rc_t(S0.lin, r, c, p.lty, p.ltx);
        idx[i] = ts + (ts >> 5);
        qB[i] = rem[i] = 0;
        pos[i] = 0;
        if (r < tl.h && c < tl.w) {
          valid |= 1u << i;
          pos[i] = storage2(S1.lin, tl.y0 + r, tl.x0 + c, p.H, p.W);
          if (UNI) esplit(S1, pos[i], qB[i], rem[i]);
        }
      }
#pragma unroll 1
      for (uint32_t j = p.bstart[b]; j < p.bstart[b + 1]; ++j)
        dispatch(p.leaf[j].size, p.leaf[j].unit, StoreEE<UNI>{p, buf, qB, rem, pos, idx, valid, j});
      __syncthreads();
    } else {
      const Tile tl = tile_of(p, item);
      if constexpr (MODE == 0 || MODE == 2 || MODE == 3) {
        load_src(p, tl, smem, phase);
        __syncthreads();
      }
      if constexpr (MODE == 3) {  // same record layout: flush the destination runs from the source image
        uint32_t nruns, len;
        runs_of(S1, tl, nruns, len);
        const uint32_t warp = tid >> 5, lane = tid & 31, u = p.u3;
        const bool wpr = nruns >= kWT / 32;  // a warp per run, else the warps share each run's records
        for (uint32_t j = wpr ? warp : 0; j < nruns; j += wpr ? kWT / 32 : 1) {
          uint8_t* g = p.db[S1.blob] + run_start(p, S1, tl, j);
          for (uint32_t q = wpr ? 0 : warp; q < len; q += wpr ? 1 : kWT / 32) {
            uint32_t r, c;
            t_rc(S1.lin, (j << S1.lrun) + q, p.lty, p.ltx, r, c);
            const uint8_t* s = smem + S0.img + img_off(S0, rc_t(S0.lin, r, c, p.lty, p.ltx));
            uint8_t* d = g + (uint64_t)q * S1.S;
            if (u == 16) copy_run<16>(d, s, S1.S, lane);
            else if (u == 8) copy_run<8>(d, s, S1.S, lane);
            else copy_run<4>(d, s, S1.S, lane);
          }
        }
        __syncthreads();
        continue;
      }
      if constexpr (GRP) {
        {  // 4-record groups along the E side's order
          const WideSide& E = MODE == 0 ? S1 : S0;
          const WideSide& A = MODE == 0 ? S0 : S1;
          const uint32_t ng = n >> 2, gl = ng >= kWT ? 1 : kWT / ng;
          for (uint32_t gi = tid % ng; gi < ng; gi += kWT) {
            uint32_t ro[4], ln[4], nv = 0, r0 = 0, c0 = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              uint32_t r, c;
              t_rc(E.lin, 4 * gi + i, p.lty, p.ltx, r, c);
              if (i == 0) r0 = r, c0 = c;
              const uint32_t ta = rc_t(A.lin, r, c, p.lty, p.ltx);
              ro[i] = img_off(A, ta);
              ln[i] = img_lane(A, ta);
              if (r < tl.h && c < tl.w && nv == (uint32_t)i) ++nv;
            }
            if (!nv) continue;
            uint64_t qB, rem;
            esplit(E, storage2(E.lin, tl.y0 + r0, tl.x0 + c0, p.H, p.W), qB, rem);
            const uint32_t kl2 = tid / ng < gl ? tid / ng : 0;
            if (MODE == 1 && p.stage) {  // phase 1: cp.async into the staging area
#pragma unroll 1
              for (uint32_t q = 0; q < p.n_cls; ++q) {
                const WideClass& cl = p.cls[q];
                StageEA m{p, smem + p.buf, qB, rem, gi, nv, cl.j0, cl.j1, kl2, gl};
                dispatch_vec(cl.size, cl.unit & 0xFF, cl.unit >> 8, m);
              }
              continue;
            }
#pragma unroll 1
            for (uint32_t q = 0; q < p.n_cls; ++q) {
              const WideClass& cl = p.cls[q];
              if constexpr (MODE == 0) {
                GroupAE m{p, smem + A.img, ro[0], ro[1], ro[2], ro[3], ln[0], ln[1], ln[2], ln[3], qB, rem, nv, cl.j0, cl.j1,
                          kl2, gl};
                dispatch_vec(cl.size, cl.unit & 0xFF, cl.unit >> 8, m);
              } else {
                GroupEA m{p, smem + A.img, ro[0], ro[1], ro[2], ro[3], ln[0], ln[1], ln[2], ln[3], qB, rem, nv, cl.j0, cl.j1,
                          kl2, gl};
                dispatch_vec(cl.size, cl.unit & 0xFF, cl.unit >> 8, m);
              }
            }
          }
          if (MODE == 1 && p.stage) {  // phase 2: staging -> image
            cp_async_wait_all();
            __syncthreads();
            for (uint32_t gi = tid % ng; gi < ng; gi += kWT) {
              uint32_t ro[4], ln[4], nv = 0;
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                uint32_t r, c;
                t_rc(E.lin, 4 * gi + i, p.lty, p.ltx, r, c);
                const uint32_t ta = rc_t(A.lin, r, c, p.lty, p.ltx);
                ro[i] = img_off(A, ta);
                ln[i] = img_lane(A, ta);
                if (r < tl.h && c < tl.w && nv == (uint32_t)i) ++nv;
              }
              if (!nv) continue;
              const uint32_t kl2 = tid / ng < gl ? tid / ng : 0;
#pragma unroll 1
              for (uint32_t q = 0; q < p.n_cls; ++q) {
                const WideClass& cl = p.cls[q];
                ScatterEA m{p, smem + p.buf, smem + A.img, ro[0], ro[1], ro[2], ro[3], ln[0], ln[1], ln[2], ln[3], gi, nv,
                            cl.j0, cl.j1, kl2, gl};
                dispatch_vec(cl.size, cl.unit & 0xFF, cl.unit >> 8, m);
              }
            }
          }
          if constexpr (MODE == 1) {
            if (p.async) cp_async_wait_all();  // (the cp.async element copies into the image)
            fence_proxy_async_smem();          // image writes -> the TMA store
          }
          __syncthreads();
          if constexpr (MODE == 1) {
            flush_dst(p, tl, smem);
            __syncthreads();
          }
          continue;
        }
      }
      if constexpr (!GRP) for (uint32_t t = t0; t < n; t += kWT) {
        uint32_t r, c;
        const uint32_t ord = MODE == 1 ? S0.lin : S1.lin;  // lanes along the E side (A -> A: the destination)
        t_rc(ord, t, p.lty, p.ltx, r, c);
        if (r >= tl.h || c >= tl.w) continue;
        if constexpr (MODE == 0) {
          const uint32_t ts = rc_t(S0.lin, r, c, p.lty, p.ltx);
          MovesAE<UNI> m{p, smem + S0.img + img_off(S0, ts), 0, 0, 0, 0, 0, kl, nl, img_lane(S0, ts)};
          m.pos = storage2(S1.lin, tl.y0 + r, tl.x0 + c, p.H, p.W);
          if (UNI) esplit(S1, m.pos, m.qB, m.rem);
#pragma unroll 1
          for (uint32_t q = 0; q < p.n_cls; ++q) {
            m.j0 = p.cls[q].j0;
            m.j1 = p.cls[q].j1;
            dispatch(p.cls[q].size, p.cls[q].unit & 0xFF, m);
          }
        } else if constexpr (MODE == 1) {
          const uint32_t td = rc_t(S1.lin, r, c, p.lty, p.ltx);
          MovesEA<UNI> m{p, smem + S1.img + img_off(S1, td), 0, 0, 0, 0, 0, kl, nl, img_lane(S1, td)};
          m.pos = storage2(S0.lin, tl.y0 + r, tl.x0 + c, p.H, p.W);
          if (UNI) esplit(S0, m.pos, m.qB, m.rem);
#pragma unroll 1
          for (uint32_t q = 0; q < p.n_cls; ++q) {
            m.j0 = p.cls[q].j0;
            m.j1 = p.cls[q].j1;
            dispatch(p.cls[q].size, p.cls[q].unit & 0xFF, m);
          }
        } else {
          const uint32_t ts = rc_t(S0.lin, r, c, p.lty, p.ltx);
          MovesAA m{p, smem + S0.img + img_off(S0, ts), smem + S1.img + img_off(S1, t), 0, 0, kl, nl,
                    img_lane(S0, ts), img_lane(S1, t)};
#pragma unroll 1
          for (uint32_t q = 0; q < p.n_cls; ++q) {
            m.j0 = p.cls[q].j0;
            m.j1 = p.cls[q].j1;
            dispatch(p.cls[q].size, p.cls[q].unit & 0xFF, m);
          }
        }
      }
      if constexpr (MODE == 1 || MODE == 2) fence_proxy_async_smem();
      __syncthreads();
      if constexpr (MODE == 1 || MODE == 2) {
        flush_dst(p, tl, smem);
        __syncthreads();
      }
    }
  }
}

}  // namespace

namespace {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = []() -> EncodeFn {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<EncodeFn>(f);
  }();  // (a function-local static: initialised once, thread-safe)
  return fn;
}

// the box of side X over its blob: row-major [H][W * S] or column-major
// [W][H / g][g * S] in elsz-byte elements (WideSide)
int encode_side(WideParams& q, int X, uint8_t* blob) {
  const WideSide& s = q.side[X];
  EncodeFn fn = encode_fn();
  if (!fn) return (int)cudaErrorNotSupported;
  const CUtensorMapDataType dt = s.elsz == 8   ? CU_TENSOR_MAP_DATA_TYPE_UINT64
                                 : s.elsz == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32
                                 : s.elsz == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                               : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  const uint64_t S = s.S, H = q.H, W = q.W, TY = 1ull << q.lty, TX = 1ull << q.ltx;
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3], estr[3] = {1, 1, 1};
  cuuint32_t rank;
  if (s.tma == 2) {
    rank = 2;
    dims[0] = W * S / s.elsz, dims[1] = H;
    strides[0] = W * S;
    box[0] = (cuuint32_t)(TX * S / s.elsz), box[1] = (cuuint32_t)TY;
  } else {
    rank = 3;
    dims[0] = s.g * S / s.elsz, dims[1] = H / s.g, dims[2] = W;
    strides[0] = s.g * S, strides[1] = H * S;
    box[0] = (cuuint32_t)(s.g * S / s.elsz), box[1] = (cuuint32_t)(TY / s.g), box[2] = (cuuint32_t)TX;
  }
  const CUresult r = fn(&q.tmap[X], dt, rank, blob + s.base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

}  // namespace

int launch_transpose_wide(const WideParams& p0, void* stream) {
  if (p0.n_items == 0) return 0;
  const WideParams* pp = &p0;
  WideParams q;
  if (p0.side[0].tma >= 2 || p0.side[1].tma >= 2) {  // the blob addresses are part of the tensor maps
    q = p0;
    for (int X = 0; X < 2; ++X)
      if (q.side[X].tma >= 2) {  // (tma == 1: plain bulk copies, no map)
        uint8_t* blob = X == 0 ? const_cast<uint8_t*>(q.sb[q.side[0].blob]) : q.db[q.side[1].blob];
        if (int e = encode_side(q, X, blob)) return e;
      }
    pp = &q;
  }
  const WideParams& p = *pp;
  static LaunchCache cache[13][64];
  // index: mode + 5 * (every E side uniform: block split hoisted, no per-leaf
  // division); 10 / 11 / 12: modes 0 / 1 / 4 in 4-record groups.  Minimum CTAs per SM
  // from the shared memory a HEP100 tile takes (48-61 KB: 3-4), so the
  // register budget never costs occupancy.
  void (*const kerns[13])(WideParams) = {
      k_transpose_wide<0, false, false, 3>, k_transpose_wide<1, false, false, 3>,
      k_transpose_wide<2, false, false, 3>, k_transpose_wide<3, false, false, 4>,
      k_transpose_wide<4, false, false, 2>, k_transpose_wide<0, true, false, 3>,
      k_transpose_wide<1, true, false, 3>,  k_transpose_wide<2, true, false, 3>,
      k_transpose_wide<3, true, false, 4>,  k_transpose_wide<4, true, false, 2>,
      k_transpose_wide<0, true, true, 4>,   k_transpose_wide<1, true, true, 4>,
      k_transpose_wide<4, true, true, 4>};
  if (p.mode > 4) return (int)cudaErrorInvalidValue;
  const bool uni = (p.side[0].A || p.side[0].uni) && (p.side[1].A || p.side[1].uni);
  const int v = p.grp && uni && (p.mode <= 1 || p.mode == 4) ? (p.mode == 4 ? 12 : 10 + (int)p.mode)
                                                               : (int)p.mode + (uni ? 5 : 0);
  int dev = 0, per_sm = 1, sms = 148;
  cudaGetDevice(&dev);
  auto kern = kerns[v];
  int e = prepare_kernel(kern, kWT, (int)p.smem, &cache[v][dev & 63], &per_sm);
  if (e) return e;
  current_device_sms(&sms);
  uint64_t grid = (uint64_t)sms * per_sm;
  if (grid > p.n_items) grid = p.n_items;
  kern<<<(unsigned)grid, kWT, p.smem, (cudaStream_t)stream>>>(p);
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace llb
