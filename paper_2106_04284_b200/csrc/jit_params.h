// jit_params.h -- the runtime parameter block of the plan-time specialised
// ("JIT") permute kernel.  Shared verbatim by the host (jit.cpp) and the
// NVRTC-compiled device code (embedded into the generated source), so it uses
// only fixed-width built-in types and no includes.  Everything that is the
// same for every launch of a plan (tile geometry, leaf offsets, the move
// program) is compiled into the kernel as constants; this block carries what
// changes per call (blob pointers) and the generic descriptors of the tail
// path (the last partial tile, moved element-wise through the normal form).
#ifndef LLB_JIT_PARAMS_H
#define LLB_JIT_PARAMS_H

#define LLB_JIT_MAX_LEAVES 128
#define LLB_JIT_MAX_BLOBS 128
#define LLB_JIT_MAX_ZERO 16

// One leaf's normal form: off(i) = base + (i / L) * B + F + (i % L) * size.
struct LlbJitLeaf {
  unsigned long long base, F, L, B;
  unsigned int blob, size, pad0, pad1;
};

struct LlbJitParams {
  unsigned long long N;       // records
  unsigned long long n_full;  // full tiles (records [0, n_full * T) go through the tile pipeline)
  unsigned int K;             // leaves
  unsigned int n_gaps;        // destination padding outside every tile (aligned SoA single-blob gaps)
  unsigned int n_zero;        // destination byte ranges the tail path zeroes before its element copies
  unsigned int pad_;
  unsigned char* blobs[2][LLB_JIT_MAX_BLOBS];      // [0] src, [1] dst (per call)
  const unsigned char* sg[LLB_JIT_MAX_LEAVES];     // src SoA leaves: element 0 (per call)
  unsigned char* dg[LLB_JIT_MAX_LEAVES];           // dst SoA leaves: element 0 (per call)
  LlbJitLeaf leaf[2][LLB_JIT_MAX_LEAVES];          // tail path: both sides' normal forms
  unsigned int gap_blob[LLB_JIT_MAX_LEAVES];
  unsigned int gap_len[LLB_JIT_MAX_LEAVES];
  unsigned long long gap_off[LLB_JIT_MAX_LEAVES];
  unsigned int zero_blob[LLB_JIT_MAX_ZERO];
  unsigned long long zero_off[LLB_JIT_MAX_ZERO];
  unsigned long long zero_len[LLB_JIT_MAX_ZERO];
};

#endif
