// jit.hpp -- the plan-time specialised permute:
// for one mapping pair the planner generates the kernel's move program with
// compile-time offsets and compiles it with NVRTC for sm_100a (the paper
// specialises its copies at compile time through C++ templates, P:555-562,
// P:759-761; a runtime descriptor specialises at plan time instead).
#pragma once
#include <memory>
#include <string>

#include "jit_params.h"
#include "mapping.hpp"

namespace llb {

struct Knobs;
struct JitModule;  // compiled cubin + per-device loaded kernels (jit.cpp)

struct JitPlan {
  std::shared_ptr<JitModule> mod;
  std::string source;           // the generated CUDA source (for tests / inspection)
  LlbJitParams params;          // everything but the per-call pointers
  std::string kernel = "llb_jit_permute";  // or "llb_jit_transpose" (2-d tiles, different linearisations)
  uint64_t n_tiles = 0;         // tiles of the tile pipeline (the grid is bounded by it)
  uint32_t threads = 256 + 32;  // CTA size (consumers + the store warp)
  uint32_t T = 0, ns = 0, nd = 0, parts = 0, minb = 1;
  uint32_t smem = 0;            // dynamic shared memory per CTA
  uint32_t src_soa[LLB_JIT_MAX_LEAVES] = {};  // 1: src leaf k is a SoA leaf (sg pointer patched per call)
  uint32_t dst_soa[LLB_JIT_MAX_LEAVES] = {};  // 1: dst leaf k is stored to global memory (dg pointer)
};

// Builds and compiles the specialised kernel for the pair; false with *why
// when the pair is not eligible (or NVRTC is unavailable / fails).
bool plan_jit(const Mapping& s, const Mapping& d, int tile_records, const Knobs& kn, JitPlan* out, std::string* why);

// The transposing variant: rank-2 views of different linearisations (row /
// column / Morton) in 32 x 32-record tiles (jit_kernel2d.cuh).
bool plan_jit2d(const Mapping& s, const Mapping& d, const Knobs& kn, JitPlan* out, std::string* why);

// Enqueues the copy (patches the blob pointers into a copy of the params).
int launch_jit(const JitPlan& jp, const Mapping& s, void* const* src_blobs, const Mapping& d, void* const* dst_blobs,
               bool pdl, void* stream);

}  // namespace llb
