// plan.hpp -- the copy planner (specialised copies for related
// mappings, "run time analysis of the two views to find contiguous memory
// chunks").  A plan is computed once per (src mapping, dst mapping, options)
// and cached; per call only the blob pointers are patched in.
#pragma once
#include <memory>
#include <string>

#include "jit.hpp"
#include "mapping.hpp"
#include "params.hpp"

namespace llb {

// Explicit tuning overrides (llama_copy_options.knobs); -1 = the measured default.
struct Knobs {
  int64_t v[LLAMA_KNOB_COUNT];
  Knobs() {
    for (auto& x : v) x = -1;
  }
  explicit Knobs(const int64_t* in) : Knobs() {
    if (in)
      for (int k = 0; k < LLAMA_KNOB_COUNT; ++k) v[k] = in[k] < 0 ? -1 : in[k];
  }
  bool given(llama_knob k) const { return v[k] >= 0; }
  uint64_t get(llama_knob k, uint64_t def) const { return v[k] >= 0 ? (uint64_t)v[k] : def; }
};

struct Plan {
  llama_path path = LLAMA_PATH_NAIVE;
  bool empty = false;         // nothing to do (no destination bytes)
  bool naive_zero_fill = false;
  bool pdl = true;            // PERMUTE: programmatic dependent launch
  bool permute_v1 = false;    // PERMUTE: the barrier-synchronised kernel instead of the warp-specialised one
  int smem_bytes = 0;
  uint64_t src_bytes = 0, dst_bytes = 0;
  std::unique_ptr<NaiveParams> naive;
  std::unique_ptr<FillParams> fill;
  std::unique_ptr<BlobCopyParams> blobcopy;
  std::unique_ptr<BulkCopyParams> bulkcopy;  // TMA variant of the blob copy
  std::unique_ptr<RunParams> run;
  std::unique_ptr<PermParams> perm;
  std::unique_ptr<DirectParams> direct;  // PERMUTE path, direct variant (AoS <-> SoA, many leaves)
  std::unique_ptr<JitPlan> jit;          // PERMUTE path, plan-time specialised kernel (wide records, splits)
  std::unique_ptr<WideParams> wide;      // TRANSPOSE path, wide records (k_transpose_wide)
};

// Checks S:484-486 (same leaf types, same extents).
llama_status check_compatible(const Mapping& s, const Mapping& d, std::string* err);

// Builds a plan for `path` (LLAMA_PATH_AUTO = the planner's choice).
// UNSUPPORTED if a forced path does not apply to the pair.
llama_status make_plan(const Mapping& s, const Mapping& d, llama_path path, int tile_records, const Knobs& kn,
                       Plan* out, std::string* err);

// Path-specific builders; return false (with *why) when not applicable.
bool plan_blobcopy(const Mapping& s, const Mapping& d, const Knobs& kn, Plan* p, std::string* why);
bool plan_transpose(const Mapping& s, const Mapping& d, const Knobs& kn, Plan* p, std::string* why);
bool plan_wide(const Mapping& s, const Mapping& d, const Knobs& kn, Plan* p, std::string* why);
bool plan_run(const Mapping& s, const Mapping& d, Plan* p, std::string* why);
bool plan_permute(const Mapping& s, const Mapping& d, int tile_records, const Knobs& kn, Plan* p, std::string* why);
bool plan_direct(const Mapping& s, const Mapping& d, int tile_records, const Knobs& kn, Plan* p, std::string* why);
void plan_naive(const Mapping& s, const Mapping& d, Plan* p);

FillParams make_fill(const Mapping& m, uint8_t value);

}  // namespace llb
