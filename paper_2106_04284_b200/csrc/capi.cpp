// capi.cpp -- the C ABI (include/llama_b200.h): validation, plan cache,
// launches.  No C++ exception crosses this boundary.
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <tuple>
#include <vector>

#include "capi_internal.hpp"
#include "launch.hpp"
#include "plan.hpp"

namespace {

thread_local std::string g_err;

llama_status fail(llama_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

using PlanKey = std::tuple<uint64_t, uint64_t, int, int, std::vector<int64_t>>;
std::mutex g_mu;
std::map<PlanKey, std::shared_ptr<llb::Plan>> g_plans;

llama_status get_plan(const llb::Mapping& s, const llb::Mapping& d, const llama_copy_options* options,
                      std::shared_ptr<llb::Plan>* out) {
  const llama_path path = options ? options->path : LLAMA_PATH_AUTO;
  const int tile = options ? options->tile_records : 0;
  const llb::Knobs kn(options ? options->knobs : nullptr);
  PlanKey key{s.id, d.id, (int)path, tile, std::vector<int64_t>(kn.v, kn.v + LLAMA_KNOB_COUNT)};
  {
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) { *out = it->second; return LLAMA_OK; }
  }
  auto plan = std::make_shared<llb::Plan>();
  std::string err;
  llama_status st = llb::make_plan(s, d, path, tile, kn, plan.get(), &err);
  if (st != LLAMA_OK) return fail(st, err);
  std::lock_guard<std::mutex> g(g_mu);
  g_plans[key] = plan;
  *out = plan;
  return LLAMA_OK;
}

llama_status cuda_fail(int e, const char* what) {
  return fail(LLAMA_ERR_CUDA, std::string(what) + ": " + llb::cuda_error_string(e));
}

// Blob pointer checks shared by copy and generate.
llama_status check_blobs(const llb::Mapping& m, void* const* blobs, const char* name) {
  if (!blobs) return fail(LLAMA_ERR_INVALID_ARGUMENT, std::string(name) + " is NULL");
  for (int b = 0; b < m.nblobs(); ++b) {
    if (m.blob_sizes[b] == 0) continue;
    if (!blobs[b]) return fail(LLAMA_ERR_INVALID_ARGUMENT, std::string(name) + "[" + std::to_string(b) + "] is NULL");
    if (reinterpret_cast<uintptr_t>(blobs[b]) % 16)
      return fail(LLAMA_ERR_ALIGNMENT, std::string(name) + "[" + std::to_string(b) + "] is not 16-byte aligned");
  }
  return LLAMA_OK;
}

}  // namespace

namespace llb {
llama_status set_error(llama_status s, const std::string& msg) { return fail(s, msg); }
}  // namespace llb

extern "C" {

llama_status llama_mapping_create(const llama_mapping_desc* desc, llama_mapping** out) {
  if (!desc || !out) return fail(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  try {
    auto* m = new llama_mapping;
    std::string err;
    llama_status st = llb::build_mapping(*desc, &m->m, &err);
    if (st != LLAMA_OK) {
      delete m;
      return fail(st, err);
    }
    *out = m;
    return LLAMA_OK;
  } catch (const std::bad_alloc&) {
    return fail(LLAMA_ERR_OOM, "out of host memory");
  } catch (...) {
    return fail(LLAMA_ERR_INVALID_ARGUMENT, "unexpected error");
  }
}

llama_status llama_mapping_create_from_schema(const char* schema, const int64_t* extents, int32_t rank,
                                              llama_kind kind, int64_t lanes, int32_t aligned,
                                              llama_mapping** out) {
  if (!schema) return fail(LLAMA_ERR_INVALID_ARGUMENT, "NULL schema");
  try {
    std::vector<llama_scalar> leaves;
    std::string err;
    if (!llb::parse_schema(schema, &leaves, &err)) return fail(LLAMA_ERR_INVALID_ARGUMENT, err);
    if (leaves.size() > (size_t)LLAMA_MAX_LEAVES) return fail(LLAMA_ERR_UNSUPPORTED, "more than LLAMA_MAX_LEAVES leaves");
    llama_mapping_desc d{leaves.data(), (int32_t)leaves.size(), extents, rank, kind, lanes, aligned};
    return llama_mapping_create(&d, out);
  } catch (const std::bad_alloc&) {
    return fail(LLAMA_ERR_OOM, "out of host memory");
  } catch (...) {
    return fail(LLAMA_ERR_INVALID_ARGUMENT, "unexpected error");
  }
}

llama_status llama_mapping_create_split(const llama_mapping* a, const llama_mapping* b, const int32_t* leaves_a,
                                        int32_t n_a, llama_mapping** out) {
  if (!a || !b || !out || (n_a > 0 && !leaves_a)) return fail(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  try {
    auto* m = new llama_mapping;
    std::string err;
    llama_status st = llb::build_split(a->m, b->m, leaves_a, n_a, &m->m, &err);
    if (st != LLAMA_OK) {
      delete m;
      return fail(st, err);
    }
    *out = m;
    return LLAMA_OK;
  } catch (const std::bad_alloc&) {
    return fail(LLAMA_ERR_OOM, "out of host memory");
  } catch (...) {
    return fail(LLAMA_ERR_INVALID_ARGUMENT, "unexpected error");
  }
}

llama_status llama_mapping_with_linearizer(const llama_mapping* m, llama_linearizer lin, llama_mapping** out) {
  if (!m || !out) return fail(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  try {
    auto* c = new llama_mapping(*m);
    std::string err;
    llama_status st = llb::set_linearizer(&c->m, lin, &err);
    if (st != LLAMA_OK) {
      delete c;
      return fail(st, err);
    }
    *out = c;
    return LLAMA_OK;
  } catch (...) {
    return fail(LLAMA_ERR_OOM, "out of host memory");
  }
}

void llama_mapping_destroy(llama_mapping* m) {
  if (!m) return;
  {
    std::lock_guard<std::mutex> g(g_mu);
    for (auto it = g_plans.begin(); it != g_plans.end();) {
      if (std::get<0>(it->first) == m->m.id || std::get<1>(it->first) == m->m.id) it = g_plans.erase(it);
      else ++it;
    }
  }
  delete m;
}

int32_t llama_blob_count(const llama_mapping* m) { return m ? m->m.nblobs() : -1; }

llama_status llama_blob_sizes(const llama_mapping* m, uint64_t* sizes, int32_t capacity) {
  if (!m || !sizes) return fail(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  if (capacity < m->m.nblobs()) return fail(LLAMA_ERR_INVALID_ARGUMENT, "capacity below blob count");
  for (int b = 0; b < m->m.nblobs(); ++b) sizes[b] = m->m.blob_sizes[b];
  return LLAMA_OK;
}

int64_t llama_record_count(const llama_mapping* m) { return m ? (int64_t)m->m.N : -1; }

int32_t llama_leaf_types(const llama_mapping* m, llama_scalar* types, int32_t capacity) {
  if (!m) return -1;
  if (types)
    for (int k = 0; k < m->m.K() && k < capacity; ++k) types[k] = m->m.types[k];
  return m->m.K();
}

llama_status llama_blob_nr_and_offset(const llama_mapping* m, const int64_t* index, int32_t leaf, int32_t* blob,
                                      uint64_t* offset) {
  if (!m || !index || !blob || !offset) return fail(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  const llb::Mapping& mm = m->m;
  if (leaf < 0 || leaf >= mm.K()) return fail(LLAMA_ERR_INVALID_ARGUMENT, "leaf out of range");
  for (size_t d = 0; d < mm.extents.size(); ++d)
    if (index[d] < 0 || index[d] >= mm.extents[d]) return fail(LLAMA_ERR_INVALID_ARGUMENT, "index out of range");
  *blob = (int32_t)mm.blob[leaf];
  *offset = mm.offset(mm.storage(index), leaf);  // linearisation, then the normal form
  return LLAMA_OK;
}

llama_status llama_plan(const llama_mapping* src_map, const llama_mapping* dst_map,
                        const llama_copy_options* options, llama_plan_info* out) {
  if (!src_map || !dst_map || !out) return fail(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  try {
    std::shared_ptr<llb::Plan> plan;
    llama_status st = get_plan(src_map->m, dst_map->m, options, &plan);
    if (st != LLAMA_OK) return st;
    *out = llama_plan_info{};
    out->path = plan->path;
    out->src_bytes = plan->src_bytes;
    out->dst_bytes = plan->dst_bytes;
    if (plan->perm) {
      out->tile_records = (int32_t)plan->perm->T;
      out->smem_bytes = plan->smem_bytes;
      out->moves = (int32_t)plan->perm->n_moves;
      out->tma = (int32_t)plan->perm->tma;
      out->word_moves = (int32_t)plan->perm->n_wmoves;
    }
    if (plan->jit) {
      out->tile_records = (int32_t)plan->jit->T;
      out->smem_bytes = plan->smem_bytes;
      out->moves = (int32_t)plan->jit->parts;
      out->tma = 1;
      out->jit = 1;
    }
    if (plan->direct) {
      out->tile_records = (int32_t)plan->direct->T;
      out->smem_bytes = plan->smem_bytes;
      out->moves = (int32_t)plan->direct->K;
      out->tma = 1;
      out->direct = 1;
    }
    if (plan->wide) {
      out->tile_records = (int32_t)(1u << (plan->wide->lty + plan->wide->ltx));
      out->smem_bytes = plan->smem_bytes;
      out->moves = (int32_t)plan->wide->mode;
      out->wide = 1;
    }
    return LLAMA_OK;
  } catch (...) {
    return fail(LLAMA_ERR_OOM, "planning failed");
  }
}

llama_status llama_plan_source(const llama_mapping* src_map, const llama_mapping* dst_map,
                               const llama_copy_options* options, char* buf, uint64_t capacity, uint64_t* length) {
  if (!src_map || !dst_map) return fail(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  try {
    std::shared_ptr<llb::Plan> plan;
    llama_status st = get_plan(src_map->m, dst_map->m, options, &plan);
    if (st != LLAMA_OK) return st;
    if (!plan->jit) return fail(LLAMA_ERR_INVALID_ARGUMENT, "the plan is not a plan-time specialised kernel");
    const std::string& src = plan->jit->source;
    if (length) *length = src.size();
    if (buf && capacity) {
      const size_t n = std::min<size_t>(src.size(), capacity - 1);
      std::memcpy(buf, src.data(), n);
      buf[n] = '\0';
    }
    return LLAMA_OK;
  } catch (...) {
    return fail(LLAMA_ERR_OOM, "planning failed");
  }
}

llama_status llama_copy_ex(const llama_mapping* src_map, void* const* src_blobs, const llama_mapping* dst_map,
                           void* const* dst_blobs, void* stream, const llama_copy_options* options) {
  if (!src_map || !dst_map) return fail(LLAMA_ERR_INVALID_ARGUMENT, "NULL mapping");
  try {
    const llb::Mapping& s = src_map->m;
    const llb::Mapping& d = dst_map->m;
    std::string err;
    llama_status st = llb::check_compatible(s, d, &err);
    if (st != LLAMA_OK) return fail(st, err);
    if ((st = check_blobs(s, src_blobs, "src_blobs")) != LLAMA_OK) return st;
    if ((st = check_blobs(d, dst_blobs, "dst_blobs")) != LLAMA_OK) return st;
    for (int i = 0; i < s.nblobs(); ++i) {  // in-situ copies are out of scope (reading #15)
      if (!s.blob_sizes[i]) continue;
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(src_blobs[i]), a1 = a0 + s.blob_sizes[i];
      for (int j = 0; j < d.nblobs(); ++j) {
        if (!d.blob_sizes[j]) continue;
        const uintptr_t b0 = reinterpret_cast<uintptr_t>(dst_blobs[j]), b1 = b0 + d.blob_sizes[j];
        if (a0 < b1 && b0 < a1)
          return fail(LLAMA_ERR_OVERLAP, "src blob " + std::to_string(i) + " overlaps dst blob " + std::to_string(j));
      }
    }
    for (int i = 0; i < d.nblobs(); ++i) {
      for (int j = i + 1; j < d.nblobs(); ++j) {
        if (!d.blob_sizes[i] || !d.blob_sizes[j]) continue;
        const uintptr_t a0 = reinterpret_cast<uintptr_t>(dst_blobs[i]), a1 = a0 + d.blob_sizes[i];
        const uintptr_t b0 = reinterpret_cast<uintptr_t>(dst_blobs[j]), b1 = b0 + d.blob_sizes[j];
        if (a0 < b1 && b0 < a1)
          return fail(LLAMA_ERR_OVERLAP, "dst blobs " + std::to_string(i) + " and " + std::to_string(j) + " overlap");
      }
    }
    std::shared_ptr<llb::Plan> plan;
    if ((st = get_plan(s, d, options, &plan)) != LLAMA_OK) return st;
    if (plan->empty) return LLAMA_OK;

    int e = 0;
    switch (plan->path) {
      case LLAMA_PATH_NAIVE:
      case LLAMA_PATH_TRANSPOSE: {
        if (plan->jit) {
          e = llb::launch_jit(*plan->jit, s, src_blobs, d, dst_blobs, plan->pdl, stream);
          break;
        }
        if (plan->wide) {
          if (plan->naive_zero_fill) {
            llb::FillParams f = *plan->fill;
            for (int b = 0; b < f.nb; ++b) f.ptr[b] = static_cast<uint8_t*>(dst_blobs[b]);
            if ((e = llb::launch_fill(f, stream))) return cuda_fail(e, "fill launch");
          }
          llb::WideParams w = *plan->wide;
          for (int b = 0; b < s.nblobs(); ++b) w.sb[b] = static_cast<const uint8_t*>(src_blobs[b]);
          for (int b = 0; b < d.nblobs(); ++b) w.db[b] = static_cast<uint8_t*>(dst_blobs[b]);
          for (uint32_t j = 0; j < w.K; ++j) {  // uniform E sides: blob + base + F per leaf
            const int k = w.order[j];
            w.leaf[j].sp = const_cast<uint8_t*>(w.sb[s.blob[k]]) + s.base[k] + s.F[k];
            w.leaf[j].dp = w.db[d.blob[k]] + d.base[k] + d.F[k];
          }
          e = llb::launch_transpose_wide(w, stream);
          break;
        }
        if (plan->naive_zero_fill) {
          llb::FillParams f = *plan->fill;
          for (int b = 0; b < f.nb; ++b) f.ptr[b] = static_cast<uint8_t*>(dst_blobs[b]);
          if ((e = llb::launch_fill(f, stream))) return cuda_fail(e, "fill launch");
        }
        llb::NaiveParams p = *plan->naive;
        for (int b = 0; b < s.nblobs(); ++b) p.sb[b] = static_cast<const uint8_t*>(src_blobs[b]);
        for (int b = 0; b < d.nblobs(); ++b) p.db[b] = static_cast<uint8_t*>(dst_blobs[b]);
        e = plan->path == LLAMA_PATH_TRANSPOSE ? llb::launch_transpose2d(p, stream) : llb::launch_naive(p, stream);
        break;
      }
      case LLAMA_PATH_BLOBCOPY: {
        if (plan->bulkcopy) {
          llb::BulkCopyParams p = *plan->bulkcopy;
          for (int b = 0; b < p.nb; ++b) {
            if (p.seg) {
              p.src[b] = static_cast<const uint8_t*>(src_blobs[p.sblob[b]]) + p.soff[b];
              p.dst[b] = static_cast<uint8_t*>(dst_blobs[p.dblob[b]]) + p.doff[b];
            } else {
              p.src[b] = static_cast<const uint8_t*>(src_blobs[b]);
              p.dst[b] = static_cast<uint8_t*>(dst_blobs[b]);
            }
          }
          e = llb::launch_bulkcopy(p, stream);
          break;
        }
        llb::BlobCopyParams p = *plan->blobcopy;
        for (int b = 0; b < p.nb; ++b) {
          p.src[b] = static_cast<const uint8_t*>(src_blobs[b]);
          p.dst[b] = static_cast<uint8_t*>(dst_blobs[b]);
        }
        e = llb::launch_blobcopy(p, stream);
        break;
      }
      case LLAMA_PATH_RUN: {
        llb::RunParams p = *plan->run;
        for (int b = 0; b < s.nblobs(); ++b) p.sb[b] = static_cast<const uint8_t*>(src_blobs[b]);
        for (int b = 0; b < d.nblobs(); ++b) p.db[b] = static_cast<uint8_t*>(dst_blobs[b]);
        e = llb::launch_run(p, stream);
        break;
      }
      case LLAMA_PATH_PERMUTE: {
        if (plan->jit) {
          e = llb::launch_jit(*plan->jit, s, src_blobs, d, dst_blobs, plan->pdl, stream);
          break;
        }
        if (plan->direct) {
          llb::DirectParams q = *plan->direct;
          for (int b = 0; b < s.nblobs(); ++b) q.blobs[0][b] = static_cast<uint8_t*>(const_cast<void*>(src_blobs[b]));
          for (int b = 0; b < d.nblobs(); ++b) q.blobs[1][b] = static_cast<uint8_t*>(dst_blobs[b]);
          for (uint32_t k = 0; k < q.K; ++k)  // the SoA side's element pointers
            q.leaf[k].gptr = q.blobs[q.a2s ? 1 : 0][q.leaf[k].blob] + q.leaf[k].gbase;
          e = llb::launch_permute_direct(q, stream);
          break;
        }
        llb::PermParams p = *plan->perm;
        for (int b = 0; b < s.nblobs(); ++b) p.blobs[0][b] = static_cast<uint8_t*>(const_cast<void*>(src_blobs[b]));
        for (int b = 0; b < d.nblobs(); ++b) p.blobs[1][b] = static_cast<uint8_t*>(dst_blobs[b]);
        e = llb::launch_permute(p, plan->smem_bytes, plan->permute_v1, plan->pdl, stream);
        break;
      }
      default:
        return fail(LLAMA_ERR_INVALID_ARGUMENT, "bad plan");
    }
    if (e) return cuda_fail(e, "copy launch");
    return LLAMA_OK;
  } catch (const std::bad_alloc&) {
    return fail(LLAMA_ERR_OOM, "out of host memory");
  } catch (...) {
    return fail(LLAMA_ERR_INVALID_ARGUMENT, "unexpected error");
  }
}

llama_status llama_copy(const llama_mapping* src_map, void* const* src_blobs, const llama_mapping* dst_map,
                        void* const* dst_blobs, void* stream) {
  return llama_copy_ex(src_map, src_blobs, dst_map, dst_blobs, stream, nullptr);
}

llama_status llama_generate(const llama_mapping* m, void* const* blobs, uint64_t seed, uint8_t pad_byte,
                            void* stream) {
  if (!m) return fail(LLAMA_ERR_INVALID_ARGUMENT, "NULL mapping");
  try {
    const llb::Mapping& mm = m->m;
    llama_status st = check_blobs(mm, blobs, "blobs");
    if (st != LLAMA_OK) return st;
    if (mm.footprint_bytes() == 0) return LLAMA_OK;
    int e;
    if (mm.has_padding()) {
      llb::FillParams f = llb::make_fill(mm, pad_byte);
      for (int b = 0; b < f.nb; ++b) f.ptr[b] = static_cast<uint8_t*>(blobs[b]);
      if ((e = llb::launch_fill(f, stream))) return cuda_fail(e, "fill launch");
    }
    std::unique_ptr<llb::GenParams> g(new llb::GenParams);
    std::memset(g.get(), 0, sizeof(*g));
    g->N = mm.N;
    g->seed = seed;
    g->K = mm.K();
    for (int k = 0; k < mm.K(); ++k) g->dl[k] = mm.dev_leaf(k);
    g->lin = mm.dev_lin();
    for (int b = 0; b < mm.nblobs(); ++b) g->db[b] = static_cast<uint8_t*>(blobs[b]);
    if ((e = llb::launch_gen(*g, stream))) return cuda_fail(e, "generate launch");
    return LLAMA_OK;
  } catch (...) {
    return fail(LLAMA_ERR_OOM, "out of host memory");
  }
}

uint64_t llama_launch_count(void) { return llb::launch_count(); }

const char* llama_status_string(llama_status s) {
  switch (s) {
    case LLAMA_OK: return "LLAMA_OK";
    case LLAMA_ERR_INVALID_ARGUMENT: return "LLAMA_ERR_INVALID_ARGUMENT";
    case LLAMA_ERR_SHAPE_MISMATCH: return "LLAMA_ERR_SHAPE_MISMATCH";
    case LLAMA_ERR_RECORD_MISMATCH: return "LLAMA_ERR_RECORD_MISMATCH";
    case LLAMA_ERR_UNSUPPORTED: return "LLAMA_ERR_UNSUPPORTED";
    case LLAMA_ERR_ALIGNMENT: return "LLAMA_ERR_ALIGNMENT";
    case LLAMA_ERR_OVERLAP: return "LLAMA_ERR_OVERLAP";
    case LLAMA_ERR_CUDA: return "LLAMA_ERR_CUDA";
    case LLAMA_ERR_OOM: return "LLAMA_ERR_OOM";
  }
  return "unknown llama_status";
}

const char* llama_last_error_message(void) { return g_err.c_str(); }

const char* llama_version(void) { return "llama_b200 0.1 (sm_100a)"; }

}  // extern "C"
