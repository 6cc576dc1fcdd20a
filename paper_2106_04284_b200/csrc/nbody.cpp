// nbody.cpp -- C ABI of the n-body move (Listing P:643-645)
// and its path planner.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>

#include "capi_internal.hpp"
#include "launch.hpp"

namespace {

// A leaf's records are laid out in 16-byte aligned runs of >= 4 (SoA, or
// AoSoA / split parts with L % 4 == 0): particles 4q..4q+3 are one vector.
bool leaf_runs4(const llb::Mapping& m, int k) {
  const bool one_block = m.Bk[k] == 0 && m.Lk[k] >= m.N;
  if (!one_block && (m.Lk[k] % 4 != 0 || m.Bk[k] % 16 != 0)) return false;
  return (m.base[k] + m.F[k]) % 16 == 0;
}

bool leaf_aligned4(const llb::Mapping& m, int k) {
  const bool one_block = m.Bk[k] == 0 && m.Lk[k] >= m.N;
  return (m.base[k] + m.F[k]) % 4 == 0 && (one_block || m.Bk[k] % 4 == 0);
}

}  // namespace

extern "C" {

llama_status llama_nbody_move_ex(const llama_mapping* mh, void* const* blobs, const int32_t* pos_leaves,
                                 const int32_t* vel_leaves, float dt, llama_move_path path,
                                 llama_move_path* path_used, void* stream) {
  if (!mh || !blobs || !pos_leaves || !vel_leaves)
    return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  try {
    const llb::Mapping& m = mh->m;
    int leaves[6];
    for (int c = 0; c < 3; ++c) {
      leaves[c] = pos_leaves[c];
      leaves[3 + c] = vel_leaves[c];
    }
    for (int j = 0; j < 6; ++j) {
      if (leaves[j] < 0 || leaves[j] >= m.K()) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "leaf index out of range");
      if (m.sizes[leaves[j]] != 4) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "Pos / Vel leaves must be 4-byte (f32)");
      for (int q = 0; q < j; ++q)
        if (leaves[q] == leaves[j]) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "a leaf is listed twice");
    }
    for (int c = 0; c < 3; ++c) {
      const int k = leaves[c];
      if (m.Bk[k] == 0 && m.Lk[k] < m.N && m.N > 1)
        return llb::set_error(LLAMA_ERR_UNSUPPORTED, "Pos maps several particles onto one place (One)");
    }
    for (int b = 0; b < m.nblobs(); ++b) {
      if (m.blob_sizes[b] == 0) continue;
      if (!blobs[b]) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "NULL blob");
      if (reinterpret_cast<uintptr_t>(blobs[b]) % 16) return llb::set_error(LLAMA_ERR_ALIGNMENT, "blob not 16-byte aligned");
    }

    llb::MoveParams p;
    std::memset(&p, 0, sizeof(p));
    p.N = m.N;
    p.dt = dt;
    p.aligned = 1;
    for (int c = 0; c < 3; ++c) {
      p.pos[c] = m.dev_leaf(leaves[c]);
      p.vel[c] = m.dev_leaf(leaves[3 + c]);
    }
    for (int j = 0; j < 6; ++j) p.aligned &= leaf_aligned4(m, leaves[j]) ? 1u : 0u;
    for (int c = 0; c < 3; ++c) {
      p.lpos[c] = (uint32_t)leaves[c];
      p.lvel[c] = (uint32_t)leaves[3 + c];
    }
    if (m.trace) {  // Trace / Heatmap: the element-wise kernel counts its resolutions
      p.traced = 1;
      p.tr = llb::dev_trace(m);
      if (path != LLAMA_MOVE_AUTO && path != LLAMA_MOVE_GENERIC)
        return llb::set_error(LLAMA_ERR_UNSUPPORTED, "a traced view moves through the GENERIC path");
      path = LLAMA_MOVE_GENERIC;
    }
    for (int b = 0; b < m.nblobs(); ++b) p.blobs[b] = static_cast<uint8_t*>(blobs[b]);

    // RUNS: every Pos / Vel leaf in 16-byte aligned runs of >= 4 particles
    bool runs = true;
    for (int j = 0; j < 6; ++j) runs = runs && leaf_runs4(m, leaves[j]);
    // AOS: all six leaves in one AoS part (L = 1) with a record stride and
    // leaf offsets that are multiples of 4, whole chunks 16-byte aligned
    bool aos = false;
    for (const llb::Part& q : m.parts) {
      if (q.kind != LLAMA_AOS || q.L != 1) continue;
      bool all = true;
      for (int j = 0; j < 6; ++j)
        all = all && std::find(q.leaves.begin(), q.leaves.end(), leaves[j]) != q.leaves.end();
      if (!all) continue;
      const uint64_t S = q.B, base = m.base[leaves[0]];
      bool ok = S % 4 == 0 && base % 16 == 0 && S > 0;
      for (int j = 0; j < 6; ++j) ok = ok && m.F[leaves[j]] % 4 == 0;
      const uint64_t g = ok ? 16 / std::gcd<uint64_t>(S, 16) : 0;
      if (ok && 8 * 32 * g * S <= 200 * 1024) {  // 8 warps' slices of 32*g records
        aos = true;
        p.S = (uint32_t)S;
        p.g = (uint32_t)g;
        p.base = base;
        p.blob = m.blob[leaves[0]];
        for (int c = 0; c < 3; ++c) {
          p.fpos[c] = (uint32_t)m.F[leaves[c]];
          p.fvel[c] = (uint32_t)m.F[leaves[3 + c]];
        }
        // TMA ring: tiles of T records (a multiple of 256, ~32 KB, T*S a
        // 16-byte multiple since S % 4 == 0 and T % 4 == 0), up to 8 stages
        // in ~200 KB of shared memory; the AOS_LSU path selects the
        // warp-staged LSU kernel instead (measured slower: 5.2 vs 6.3 TB/s)
        const uint64_t T = std::max<uint64_t>(256, (32768 / S) / 256 * 256);
        const uint64_t ns = std::min<uint64_t>(8, (200 * 1024) / (T * S));
        if (path != LLAMA_MOVE_AOS_LSU && ns >= 2 && T * S <= 64 * 1024) {
          p.tile = (uint32_t)T;
          p.ns = (uint32_t)ns;
        }
      }
      break;
    }
    llama_move_path use = path;
    if (use == LLAMA_MOVE_AUTO) use = runs ? LLAMA_MOVE_RUNS : aos ? LLAMA_MOVE_AOS : LLAMA_MOVE_GENERIC;
    if (use == LLAMA_MOVE_RUNS && !runs)
      return llb::set_error(LLAMA_ERR_UNSUPPORTED, "RUNS needs 16-byte aligned runs of >= 4 particles per leaf");
    if ((use == LLAMA_MOVE_AOS || use == LLAMA_MOVE_AOS_LSU) && !aos)
      return llb::set_error(LLAMA_ERR_UNSUPPORTED, "AOS needs Pos / Vel in one AoS part with 4-byte aligned fields");
    if (use < LLAMA_MOVE_AUTO || use > LLAMA_MOVE_AOS_LSU) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "bad path");
    if (path_used) *path_used = use;
    if (m.N == 0) return LLAMA_OK;
    int e = use == LLAMA_MOVE_RUNS ? llb::launch_move_runs(p, stream)
            : (use == LLAMA_MOVE_AOS || use == LLAMA_MOVE_AOS_LSU) ? llb::launch_move_aos(p, stream)
                                    : llb::launch_move_generic(p, stream);
    if (e) return llb::set_error(LLAMA_ERR_CUDA, std::string("move launch: ") + llb::cuda_error_string(e));
    return LLAMA_OK;
  } catch (...) {
    return llb::set_error(LLAMA_ERR_OOM, "out of host memory");
  }
}

llama_status llama_nbody_move(const llama_mapping* m, void* const* blobs, const int32_t* pos_leaves,
                              const int32_t* vel_leaves, float dt, void* stream) {
  return llama_nbody_move_ex(m, blobs, pos_leaves, vel_leaves, dt, LLAMA_MOVE_AUTO, nullptr, stream);
}

}  // extern "C"
