// jit_kernel.cuh -- device skeleton of the plan-time specialised permute
// (DESIGN.md "k_jit_permute").  NOT compiled by nvcc: _build.py embeds this
// file (and jit_params.h) as strings into the library, and jit.cpp compiles
// them with NVRTC for sm_100a together with the code it generates for one
// mapping pair: the tile geometry as macros, the TMA segment list of the
// AoS-like parts, the cp.async chunk table of the SoA source leaves, and the
// per-record move program llb_permute (straight-line loads / byte permutes /
// stores with compile-time offsets -- the paper's compile-time specialised
// copies, specialised at plan time instead).
//
// Generated: the macros LLB_T, LLB_NS, LLB_ND, LLB_SSTAGE, LLB_DSTAGE,
// LLB_NCHUNK, LLB_NDCHUNK, LLB_SRC_TMA, LLB_MINB, LLB_P, LLB_G, LLB_CW, LLB_DCW,
// LLB_NSLOT, LLB_NMUL (before this file) and, at the LLB_GENERATED marker,
// llb_ctab[] / llb_dctab[] (source / destination 16-byte chunks: one word
// smem offset | log2 s_k << 18 | leaf << 20 per SoA leaf chunk, or, with
// padded AoS part images (LLB_CW / LLB_DCW == 2), two words: smem offset |
// slot << 18 and the offset in the tile's run, the global address being
// gs[slot] + t0 * mul[slot] + offset), llb_fill_slots(), llb_src_tma(),
// llb_dst_tma(), llb_permute().
//
// Roles:
//   8 consumer warps  wait for source stage s, run llb_permute for their
//                  records (lane = record group) and program part (warp % P);
//                  SoA destination leaves are stored straight to global memory
//                  by llb_permute (coalesced: lane = record); then, the stage
//                  free, they issue source tile i+NS into it: TMA bulk loads of
//                  the AoS-like parts (thread 0, expect_tx) and 16-byte
//                  cp.async chunks of every SoA leaf's T * s_k run (all
//                  threads; completion counted on the stage's mbarrier with
//                  cp.async.mbarrier.arrive.noinc).
//   store warp     TMA bulk stores of the AoS-like destination parts of each
//                  tile, up to ND - 1 in flight.
// The last partial tile (and AoSoA tail lanes) is moved element-wise through
// the normal form by the consumers of the last CTA.

#define LLB_CONS 256

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
// (no "memory" clobber: the producer's chunk loop must be free to hoist the
// next chunks' table loads above this one; the cp.async.mbarrier.arrive after
// the loop orders the copies against the consumers)
__device__ __forceinline__ void llb_cp16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(llb_sa(s)), "l"(g));
}
__device__ __forceinline__ void llb_cp_arrive_noinc(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(llb_sa(b)) : "memory");
}
__device__ __forceinline__ void llb_cons_sync() { asm volatile("bar.sync 1, %0;" ::"n"(LLB_CONS) : "memory"); }

// streaming global stores of the SoA destination elements (written once)
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

__device__ __forceinline__ uint64_t llb_nf(const LlbJitLeaf& l, uint64_t i) {
  const uint64_t q = i / l.L;
  return l.base + q * l.B + l.F + (i - q * l.L) * l.size;
}

// ==== LLB_GENERATED ====

extern "C" __global__ void __launch_bounds__(LLB_CONS + 32, LLB_MINB) llb_jit_permute(const __grid_constant__ LlbJitParams p) {
  uint64_t* full = reinterpret_cast<uint64_t*>(llb_smem);
  uint64_t* dfull = full + 16;
  uint64_t* dempty = full + 24;
  uint8_t* sring = llb_smem + 256;
  uint8_t* dring = sring + LLB_NS * LLB_SSTAGE;
  // per slot: the SoA source element-0 pointer minus the leaf's segment offset
  // in the stage, so a 1-word chunk's global address is sgs[k] + soff + (t0 <<
  // lg); 2-word chunks: sgs[slot] + t0 * smul[slot] + offset
  const uint8_t** sgs = reinterpret_cast<const uint8_t**>(dring + LLB_ND * LLB_DSTAGE);
  uint8_t** dgs = reinterpret_cast<uint8_t**>(dring + LLB_ND * LLB_DSTAGE + 8 * LLB_NSLOT);  // SoA dst pointers minus segment offsets
  uint32_t* smul = reinterpret_cast<uint32_t*>(dgs + LLB_NSLOT);
  uint32_t* dmul = smul + LLB_NMUL;
  uint32_t* ctab = dmul + LLB_NMUL;
  uint32_t* dctab = ctab + ((LLB_NCHUNK * LLB_CW + 1u) & ~1u);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < LLB_NS; ++s) llb_mbar_init(&full[s], LLB_CONS);  // every consumer's cp.async arrival (+ TMA bytes)
    for (int d = 0; d < (LLB_ND > 0 ? LLB_ND : 1); ++d) {
      llb_mbar_init(&dfull[d], 1);
      llb_mbar_init(&dempty[d], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // destination images: padding bytes are never written by the program, so
  // they stay 0 (reading #12)
  for (uint32_t o = 16 * tid; o < LLB_ND * LLB_DSTAGE; o += 16 * (LLB_CONS + 32))
    *reinterpret_cast<uint4*>(dring + o) = make_uint4(0, 0, 0, 0);
  for (uint32_t c = tid; c < LLB_NCHUNK * LLB_CW; c += LLB_CONS + 32) ctab[c] = llb_ctab[c];
  for (uint32_t c = tid; c < LLB_NDCHUNK * LLB_DCW; c += LLB_CONS + 32) dctab[c] = llb_dctab[c];
  for (uint32_t k = tid; k < p.K; k += LLB_CONS + 32) {
    sgs[k] = p.sg[k] - llb_seg[k];
    dgs[k] = p.dg[k] - llb_dseg[k];
  }
  if (tid == LLB_CONS) llb_fill_slots(p, sgs, smul, dgs, dmul);
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (blockIdx.x == 0 && warp < LLB_CONS / 32)
    for (uint32_t g = 0; g < p.n_gaps; ++g)
      for (uint32_t o = tid; o < p.gap_len[g]; o += LLB_CONS) p.blobs[1][p.gap_blob[g]][p.gap_off[g] + o] = 0;

  const uint64_t first = blockIdx.x, stride = gridDim.x;
  const uint32_t n_my = first < p.n_full ? (uint32_t)((p.n_full - first + stride - 1) / stride) : 0;

  if (warp == LLB_CONS / 32) {  // ------------------------------ store warp
    if (LLB_ND > 0) {
      uint32_t d = 0, dph = 0;
      for (uint32_t i = 0; i < n_my; ++i) {
        // store tile i (its TMA ops spread over the 32 lanes), keep up to
        // ND - 1 stores in flight: hand back the buffer of tile i - (ND - 1)
        // once its stores have read it out
        const uint64_t t0 = (first + (uint64_t)i * stride) * LLB_T;
        llb_mbar_wait_sleep(&dfull[d], dph);
        llb_dst_tma(p, dring + d * LLB_DSTAGE, t0, (uint32_t)lane);
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
  // Source tile i+NS goes into stage s as soon as every consumer has finished
  // tile i there: TMA bulk loads of the AoS-like parts (thread 0, expect_tx)
  // and the SoA leaves' 16-byte cp.async chunks spread over all 256 consumer
  // threads (measured: one issuing warp per CTA capped a CTA at ~15 GB/s);
  // each thread's cp.async.mbarrier.arrive.noinc counts on full[s].
  auto issue = [&](uint32_t i, uint32_t s) {
    const uint64_t t0 = (first + (uint64_t)i * stride) * LLB_T;
    uint8_t* stage = sring + s * LLB_SSTAGE;
    if (LLB_SRC_TMA > 0 && tid == 0) {
      llb_mbar_expect_tx(&full[s], LLB_SRC_TMA);
      llb_src_tma(p, stage, t0, &full[s]);
    }
#if LLB_CW == 2
#pragma unroll 4
    for (uint32_t c = tid; c < LLB_NCHUNK; c += LLB_CONS) {
      const uint2 e = reinterpret_cast<const uint2*>(ctab)[c];
      const uint32_t sl = e.x >> 18;
      llb_cp16(stage + (e.x & 0x3FFFFu), sgs[sl] + t0 * smul[sl] + e.y);
    }
#else
#pragma unroll 4
    for (uint32_t c = tid; c < LLB_NCHUNK; c += LLB_CONS) {
      const uint32_t e = ctab[c], so = e & 0x3FFFFu;
      llb_cp16(stage + so, sgs[e >> 20] + so + (t0 << ((e >> 18) & 3u)));
    }
#endif
    llb_cp_arrive_noinc(&full[s]);
  };
  for (uint32_t i = 0; i < LLB_NS && i < n_my; ++i) issue(i, i);
  const uint32_t part = (uint32_t)warp % LLB_P, grp = (uint32_t)warp / LLB_P;
  uint32_t s = 0, sph = 0, d = 0, dph = 0;
  for (uint32_t i = 0; i < n_my; ++i) {
    const uint64_t t0 = (first + (uint64_t)i * stride) * LLB_T;
    if (tid == 0) {
      llb_mbar_wait(&full[s], sph);
      if (LLB_ND > 0 && i >= (uint32_t)LLB_ND) llb_mbar_wait(&dempty[d], dph ^ 1);
    }
    llb_cons_sync();
    const uint8_t* sim = sring + s * LLB_SSTAGE;
    uint8_t* dim = dring + d * LLB_DSTAGE;
    // r = a group of LLB_G consecutive records (lane = group)
    for (uint32_t r = grp * 32 + lane; r < LLB_T / LLB_G; r += (LLB_CONS / LLB_P))
      if (!LLB_ABLATE) llb_permute(p, sim, dim, t0, part, r);
    if (LLB_ND > 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    llb_cons_sync();  // every consumer is done with stage s (and destination buffer d)
    if (LLB_ND > 0 && tid == 0) llb_mbar_arrive(&dfull[d]);
    if (i + LLB_NS < n_my) issue(i + LLB_NS, s);
    // image-staged SoA destination leaves and padded AoS parts: 16-byte
    // chunks out by every consumer
#if LLB_DCW == 2
#pragma unroll 4
    for (uint32_t c = tid; c < LLB_NDCHUNK; c += LLB_CONS) {
      const uint2 e = reinterpret_cast<const uint2*>(dctab)[c];
      const uint32_t sl = e.x >> 18;
      llb_stg(dgs[sl] + t0 * dmul[sl] + e.y, *reinterpret_cast<const uint4*>(dim + (e.x & 0x3FFFFu)));
    }
#else
#pragma unroll 4
    for (uint32_t c = tid; c < LLB_NDCHUNK; c += LLB_CONS) {
      const uint32_t e = dctab[c], so = e & 0x3FFFFu;
      llb_stg(dgs[e >> 20] + so + (t0 << ((e >> 18) & 3u)), *reinterpret_cast<const uint4*>(dim + so));
    }
#endif
    if (++s == LLB_NS) { s = 0; sph ^= 1; }
    if (LLB_ND > 0 && ++d == (LLB_ND > 0 ? LLB_ND : 1)) { d = 0; dph ^= 1; }
  }
  // --------------------------------------- the last partial tile (element-wise)
  const uint64_t t_tail = p.n_full * LLB_T;
  if (blockIdx.x == gridDim.x - 1 && t_tail < p.N) {
    for (uint32_t z = 0; z < p.n_zero; ++z)
      for (uint64_t o = tid; o < p.zero_len[z]; o += LLB_CONS) p.blobs[1][p.zero_blob[z]][p.zero_off[z] + o] = 0;
    llb_cons_sync();
    const uint64_t n = (p.N - t_tail) * p.K;
    for (uint64_t x = tid; x < n; x += LLB_CONS) {
      const uint64_t i = t_tail + x / p.K;
      const uint32_t k = (uint32_t)(x % p.K);
      const LlbJitLeaf& a = p.leaf[0][k];
      const LlbJitLeaf& b = p.leaf[1][k];
      const uint8_t* sp = p.blobs[0][a.blob] + llb_nf(a, i);
      uint8_t* dp = p.blobs[1][b.blob] + llb_nf(b, i);
      for (uint32_t j = 0; j < a.size; ++j) dp[j] = sp[j];
    }
  }
}
