// jit_kernel2d.cuh -- device skeleton of the plan-time specialised
// TRANSPOSING copy: 2-d views whose
// linearisations differ (row-major / column-major / Morton), so the
// copy is also a transpose / Morton reorder.  NOT compiled by nvcc: embedded
// by _build.py, compiled by NVRTC with the code jit.cpp generates.
//
// A tile is LLB_TY x 32 records (ty, tx), LLB_TY = 32 or 16 (16 keeps two
// CTAs per SM for small records).  On each side the tile is a set of
// contiguous storage segments: LLB_TY rows of 32 (row-major), 32 columns of
// LLB_TY (column-major) or one run of 32 * LLB_TY codes (Morton).  Every segment of an AoS part moves by
// one TMA bulk copy (loads issued by consumer threads 0..31, stores by the
// store warp's 32 lanes); every segment of a SoA source leaf moves as 16-byte
// cp.async chunks spread over the consumers; SoA destination leaves are
// stored straight to global memory by llb_permute2d.  In shared memory the
// segments of a part / leaf sit at a padded pitch (odd multiple of 16 B), so
// records of one warp that lie in 32 different segments spread over the banks.
//
// Generated before the marker: LLB_NS, LLB_ND, LLB_SSTAGE, LLB_DSTAGE,
// LLB_NCHUNK, LLB_SRC_TMA, LLB_MINB, LLB_NTX (tiles along x), LLB_NTILES,
// LLB_H, LLB_W (extents), LLB_SLIN / LLB_DLIN (0 row, 1 col, 2 Morton); at the
// marker: llb_ctab[] (chunk: smem offset | log2 s_k << 18 | leaf << 20, and
// segment index | chunk index in the segment << 16 in a second word; the smem
// offset may be swizzled), llb_src_tma2d(),
// llb_dst_tma2d(), llb_permute2d().

#ifndef LLB_CONS
#define LLB_CONS 256  // consumer threads (generated)
#endif

extern __shared__ __align__(128) uint8_t llb_smem[];

__device__ __forceinline__ uint32_t llb_sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void llb_mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(llb_sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void llb_mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\nLLBW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra LLBW_%=;\n}" ::"r"(
          llb_sa(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void llb_mbar_wait_sleep(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n\t.reg .pred p;\nLLBS_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t@!p bra LLBS_%=;\n}" ::"r"(
          llb_sa(b)),
      "r"(ph), "r"(20000)
      : "memory");
}
__device__ __forceinline__ void llb_mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(llb_sa(b)) : "memory");
}
__device__ __forceinline__ void llb_mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(llb_sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void llb_g2s(void* s, const void* g, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(llb_sa(s)),
               "l"(g), "r"(bytes), "r"(llb_sa(b))
               : "memory");
}
__device__ __forceinline__ void llb_s2g(void* g, const void* s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(llb_sa(s)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void llb_cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(llb_sa(s)), "l"(g));
}
__device__ __forceinline__ void llb_cp_arrive_noinc(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(llb_sa(b)) : "memory");
}
__device__ __forceinline__ void llb_cons_sync() { asm volatile("bar.sync 1, %0;" ::"n"(LLB_CONS) : "memory"); }
__device__ __forceinline__ void llb_stg(uint8_t* p, uint8_t v) { asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(p), "h"((unsigned short)v) : "memory"); }
__device__ __forceinline__ void llb_stg(uint8_t* p, uint16_t v) { asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p), "h"(v) : "memory"); }
__device__ __forceinline__ void llb_stg(uint8_t* p, uint32_t v) { asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__device__ __forceinline__ void llb_stg(uint8_t* p, uint64_t v) { asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ void llb_stg(uint8_t* p, uint2 v) {
  asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ void llb_stg(uint8_t* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// bits of a 5-bit index spread to the even positions (Morton, #26:
// the last index supplies bit 0)
__device__ __forceinline__ uint32_t llb_spread(uint32_t v) {
  v = (v | (v << 8)) & 0x00FF00FFu;
  v = (v | (v << 4)) & 0x0F0F0F0Fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}
__device__ __forceinline__ uint32_t llb_unspread(uint32_t v) {  // the even bits of v, packed
  v &= 0x55555555u;
  v = (v | (v >> 1)) & 0x33333333u;
  v = (v | (v >> 2)) & 0x0F0F0F0Fu;
  v = (v | (v >> 4)) & 0x00FF00FFu;
  v = (v | (v >> 8)) & 0x0000FFFFu;
  return v;
}
__device__ __forceinline__ uint64_t llb_morton(uint32_t y, uint32_t x) {
  return ((uint64_t)llb_spread(y) << 1) | (uint64_t)llb_spread(x);
}
// the storage position of tile (ty, tx)'s first record and the distance between
// its segments, for a linearisation
__device__ __forceinline__ void llb_tile_pos(uint32_t lin, uint32_t ty, uint32_t tx, uint64_t* pos0, uint64_t* pitch) {
  if (lin == 0) { *pos0 = (uint64_t)(ty * LLB_TY) * LLB_W + tx * 32; *pitch = LLB_W; }
  else if (lin == 1) { *pos0 = (uint64_t)(tx * 32) * LLB_H + ty * LLB_TY; *pitch = LLB_H; }
  else { *pos0 = llb_morton(ty * LLB_TY, tx * 32); *pitch = 0; }  // the tile's codes are one aligned run
}

// ==== LLB_GENERATED ====

// block mode: block b of the tile -> (by, bx) in units of 4 x 4 records
// (LLB_BMAP: 0 x fastest, 1 y fastest, 2 / 3 their diagonals, 4 Morton)
__device__ __forceinline__ void llb_bmap(uint32_t b, uint32_t* by, uint32_t* bx) {
  constexpr uint32_t nby = LLB_TY / 4;
  if (LLB_BMAP == 0) { *bx = b % 8u; *by = b / 8u; }
  else if (LLB_BMAP == 1) { *by = b % nby; *bx = b / nby; }
  else if (LLB_BMAP == 2) { *bx = b % 8u; *by = (b / 8u + *bx) % nby; }
  else if (LLB_BMAP == 3) { *by = b % nby; *bx = (b / nby + *by) % 8u; }
  else {  // Morton over the 8 columns and the first 8 rows of blocks, then further rows (64-row tiles)
    *by = llb_unspread((b >> 1) & 0x15u) | ((b >> 6) << 3);
    *bx = llb_unspread(b & 0x15u);
  }
}

extern "C" __global__ void __launch_bounds__(LLB_CONS + 32, LLB_MINB) llb_jit_transpose(const __grid_constant__ LlbJitParams p) {
  uint64_t* full = reinterpret_cast<uint64_t*>(llb_smem);
  uint64_t* dfull = full + 16;
  uint64_t* dempty = full + 24;
  uint8_t* sring = llb_smem + 256;
  uint8_t* dring = sring + LLB_NS * LLB_SSTAGE;
  const uint8_t** sgs = reinterpret_cast<const uint8_t**>(dring + LLB_ND * LLB_DSTAGE);
  uint32_t* ctab = reinterpret_cast<uint32_t*>(sgs + 2 * LLB_JIT_MAX_LEAVES);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < LLB_NS; ++s) llb_mbar_init(&full[s], LLB_CONS);
    for (int d = 0; d < (LLB_ND > 0 ? LLB_ND : 1); ++d) {
      llb_mbar_init(&dfull[d], 1);
      llb_mbar_init(&dempty[d], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (uint32_t o = 16 * tid; o < LLB_ND * LLB_DSTAGE; o += 16 * (LLB_CONS + 32))
    *reinterpret_cast<uint4*>(dring + o) = make_uint4(0, 0, 0, 0);
  for (uint32_t c = tid; c < 2 * LLB_NCHUNK; c += LLB_CONS + 32) ctab[c] = llb_ctab[c];
  for (uint32_t k = tid; k < p.K; k += LLB_CONS + 32) sgs[k] = p.sg[k];
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (blockIdx.x == 0 && warp < LLB_CONS / 32)
    for (uint32_t g = 0; g < p.n_gaps; ++g)
      for (uint32_t o = tid; o < p.gap_len[g]; o += LLB_CONS) p.blobs[1][p.gap_blob[g]][p.gap_off[g] + o] = 0;

  const uint64_t first = blockIdx.x, stride = gridDim.x;
  const uint32_t n_my = first < LLB_NTILES ? (uint32_t)((LLB_NTILES - first + stride - 1) / stride) : 0;
  auto tile_of = [&](uint32_t i, uint32_t* ty, uint32_t* tx) {
    const uint32_t t = (uint32_t)(first + (uint64_t)i * stride);
    if (LLB_TORDER == 1) {
      *ty = t % LLB_NTY;
      *tx = t / LLB_NTY;
    } else if (LLB_TORDER == 2) {  // Morton order inside groups of 8 x 8 tiles, groups x fastest
      const uint32_t g = t / 64u, w = t % 64u;
      *ty = (g / (LLB_NTX / 8u)) * 8u + llb_unspread(w >> 1);
      *tx = (g % (LLB_NTX / 8u)) * 8u + llb_unspread(w);
    } else {
      *ty = t / LLB_NTX;
      *tx = t % LLB_NTX;
    }
  };

  if (warp == LLB_CONS / 32) {  // ------------------------------ store warp
    if (LLB_ND > 0) {
      uint32_t d = 0, dph = 0;
      for (uint32_t i = 0; i < n_my; ++i) {
        uint32_t ty, tx;
        tile_of(i, &ty, &tx);
        llb_mbar_wait_sleep(&dfull[d], dph);
        llb_dst_tma2d(p, dring + d * LLB_DSTAGE, ty, tx, lane);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(LLB_ND > 0 ? LLB_ND - 1 : 0) : "memory");
        __syncwarp();
        if (lane == 0 && i >= (uint32_t)(LLB_ND > 0 ? LLB_ND - 1 : 0))
          llb_mbar_arrive(&dempty[(d + 1) % (LLB_ND > 0 ? LLB_ND : 1)]);
        if (++d == (LLB_ND > 0 ? LLB_ND : 1)) { d = 0; dph ^= 1; }
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    return;
  }
  // ------------------------------------------------------------- consumers
  auto issue = [&](uint32_t i, uint32_t s) {
    uint32_t ty, tx;
    tile_of(i, &ty, &tx);
    uint8_t* stage = sring + s * LLB_SSTAGE;
    if (LLB_SRC_TMA > 0 && tid == 0) llb_mbar_expect_tx(&full[s], LLB_SRC_TMA);
    llb_src_tma2d(p, stage, ty, tx, (uint32_t)tid, &full[s]);  // TMA segment ops (tid < 32) / cp.async chunks
    uint64_t pos0, pitch;
    llb_tile_pos(LLB_SLIN, ty, tx, &pos0, &pitch);
#pragma unroll 4
    for (uint32_t c = tid; c < LLB_NCHUNK; c += LLB_CONS) {
      const uint32_t e = ctab[2 * c], w = ctab[2 * c + 1], so = e & 0x3FFFFu, lg = (e >> 18) & 3u, k = e >> 20;
      llb_cp16(stage + so, sgs[k] + ((pos0 + (uint64_t)(w & 0xFFFFu) * pitch) << lg) + 16u * (w >> 16));
    }
    llb_cp_arrive_noinc(&full[s]);
  };
  for (uint32_t i = 0; i < LLB_NS && i < n_my; ++i) issue(i, i);
  // thread -> record of the tile: warp w, lane l -> (yy, xx) = (w + 8 * j, l), j = 0..3
  uint32_t s = 0, sph = 0, d = 0, dph = 0;
  for (uint32_t i = 0; i < n_my; ++i) {
    uint32_t ty, tx;
    tile_of(i, &ty, &tx);
    if (tid == 0) {
      llb_mbar_wait(&full[s], sph);
      if (LLB_ND > 0 && i >= (uint32_t)LLB_ND) llb_mbar_wait(&dempty[d], dph ^ 1);
    }
    llb_cons_sync();
    const uint8_t* sim = sring + s * LLB_SSTAGE;
    uint8_t* dim = dring + d * LLB_DSTAGE;
#if LLB_BLOCK
    // a thread = one 4 x 4 block and program part (warp % LLB_P)
    {
      const uint32_t part = (uint32_t)warp % LLB_P, grp = (uint32_t)warp / LLB_P;
#pragma unroll 1
      for (uint32_t b = grp * 32u + (uint32_t)lane; b < (LLB_TY / 4) * 8u; b += LLB_CONS / LLB_P) {
        uint32_t by, bx;
        llb_bmap(b, &by, &bx);
        if (!LLB_ABLATE) llb_block2d(p, sim, dim, ty, tx, by, bx, part);
      }
    }
#else
    // lanes run along the destination's storage order when it is stored
    // straight to global memory (SoA leaves): row (xx), column (yy), Morton
    // (the low 5 bits of the tile's Morton code) -- coalesced element stores
    // the thread's 4 records unrolled: independent load -> store chains overlap
#pragma unroll
    for (uint32_t q = (uint32_t)warp; q < LLB_TY; q += LLB_CONS / 32) {
      uint32_t yy, xx;
      if (LLB_LANES == 1) { yy = (uint32_t)lane; xx = q; }
      else if (LLB_LANES == 3) {  // 4 rows x 8 columns per warp access: both a row- and a column-major
        // image see 4 / 8 segments and 8 / 4 consecutive records (no 4-way bank conflicts)
        yy = (q / 4) * 4 + ((uint32_t)lane >> 3);
        xx = (q % 4) * 8 + ((uint32_t)lane & 7u);
      }
      else if (LLB_LANES == 2) {
        const uint32_t code = q * 32 + (uint32_t)lane;  // Morton code within the tile: bit 0 from x
        yy = llb_unspread(code >> 1);
        xx = llb_unspread(code);
      } else { yy = q; xx = (uint32_t)lane; }
      if (!LLB_ABLATE) llb_permute2d(p, sim, dim, ty, tx, yy, xx);
    }
#endif
    if (LLB_ND > 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    llb_cons_sync();
    if (LLB_ND > 0 && tid == 0) llb_mbar_arrive(&dfull[d]);
    if (i + LLB_NS < n_my) issue(i + LLB_NS, s);
    llb_dst_lsu2d(p, dim, ty, tx, (uint32_t)tid);  // AoS destination segments as 16-byte chunks (knob jit_dst_lsu)
    if (++s == LLB_NS) { s = 0; sph ^= 1; }
    if (LLB_ND > 0 && ++d == (LLB_ND > 0 ? LLB_ND : 1)) { d = 0; dph ^= 1; }
  }
}
