// staged.cpp -- llama_copy_staged: the staged cross-address-space copy the
// paper proposes (§3.9: "use smaller intermediate views to shuffle
// a chunk from one mapping to the other and then perform a copy of that chunk
// into the other address space, potentially overlapping shuffles and copies
// in an asynchronous workflow").
//
// The records are cut into slabs [a, b) whose bytes are contiguous ranges of
// every blob (slab boundaries on whole AoSoA blocks).  A slab is a complete
// 1-D view of its own (the normal form depends only on the flat index), so:
//   h2d stream:  DMA the slab's source ranges into a staging buffer
//   comp stream: llama_copy between the slab's 1-D views, in staging memory
//   d2h stream:  DMA the slab's destination ranges back
// with three buffers in rotation, consecutive slabs overlap the two DMA
// directions and the relayout.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "capi_internal.hpp"

namespace {

constexpr int kNB = 3;              // staging buffers in rotation
constexpr uint64_t kAlignLocal = 16;  // blob bases in staging memory (TMA needs 16 B)

uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
uint64_t gcd64(uint64_t a, uint64_t b) {
  while (b) { uint64_t t = a % b; a = b; b = t; }
  return a;
}

struct Range {       // one contiguous byte range of a slab
  int gblob;         // blob of the global view
  uint64_t goff;     // offset in the global blob
  int lblob;         // blob of the slab's 1-D view
  uint64_t loff;     // offset in the local blob
  uint64_t len;
};

// The ranges of records [a, b) of mapping g, as laid out in the slab's 1-D
// view l (same kind / lanes / alignment, extent b - a).  a is a multiple of
// g's block size when g is blocked.
void slab_ranges(const llb::Mapping& g, const llb::Mapping& l, uint64_t a, uint64_t b, std::vector<Range>* out) {
  out->clear();
  if (b <= a) return;
  if (!g.soa()) {  // AoS / AoSoA: whole blocks, one range
    const uint64_t blk0 = a / g.L, blk1 = (b + g.L - 1) / g.L;
    out->push_back(Range{0, g.base[0] + blk0 * g.B, 0, 0, (blk1 - blk0) * g.B});
    return;
  }
  for (int k = 0; k < g.K(); ++k)  // SoA: one range per leaf sub-array
    out->push_back(Range{(int)g.blob[k], g.offset(a, k), (int)l.blob[k], l.offset(0, k), (b - a) * g.sizes[k]});
}

}  // namespace

struct llama_stager {
  int device = 0;
  uint64_t cap = 0;  // bytes per side per buffer
  uint8_t* buf[kNB][2] = {};
  uint8_t* zero = nullptr;  // 4 KB of device zeros (gap fills)
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t e_in[kNB] = {}, e_comp[kNB] = {}, e_out[kNB] = {}, e_start = nullptr, e_done = nullptr;
  // slabs enqueued over the stager's lifetime: slab c uses buffer c % kNB and
  // waits for the previous user of that buffer (slab c - kNB, possibly of an
  // earlier call on another stream) to have gone back out
  uint64_t slabs = 0;
  std::map<std::tuple<uint64_t, uint64_t>, llama_mapping*> local;  // (parent id, records) -> 1-D view
  ~llama_stager() {
    if (h2d) cudaStreamSynchronize(h2d);
    if (comp) cudaStreamSynchronize(comp);
    if (d2h) cudaStreamSynchronize(d2h);
    for (auto& kv : local) llama_mapping_destroy(kv.second);
    for (int j = 0; j < kNB; ++j) {
      cudaFree(buf[j][0]);
      cudaFree(buf[j][1]);
      if (e_in[j]) cudaEventDestroy(e_in[j]);
      if (e_comp[j]) cudaEventDestroy(e_comp[j]);
      if (e_out[j]) cudaEventDestroy(e_out[j]);
    }
    cudaFree(zero);
    if (e_start) cudaEventDestroy(e_start);
    if (e_done) cudaEventDestroy(e_done);
    if (h2d) cudaStreamDestroy(h2d);
    if (comp) cudaStreamDestroy(comp);
    if (d2h) cudaStreamDestroy(d2h);
  }
  llama_mapping* view(const llama_mapping* parent, uint64_t n) {
    auto key = std::make_tuple(parent->m.id, n);
    auto it = local.find(key);
    if (it != local.end()) return it->second;
    const llb::Mapping& p = parent->m;
    const int64_t ext = (int64_t)n;
    llama_mapping_desc d{p.types.data(), p.K(), &ext, 1, p.kind, p.lanes, p.aligned ? 1 : 0};
    llama_mapping* m = nullptr;
    if (llama_mapping_create(&d, &m) != LLAMA_OK) return nullptr;
    local[key] = m;
    return m;
  }
};

namespace {

llama_status cuda_err(cudaError_t e, const char* what) {
  return llb::set_error(LLAMA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Local blob base offsets inside one staging buffer (each blob 16-B aligned);
// returns the bytes used.
uint64_t layout_local(const llb::Mapping& l, std::vector<uint64_t>* base) {
  base->assign(l.nblobs(), 0);
  uint64_t off = 0;
  for (int b = 0; b < l.nblobs(); ++b) {
    (*base)[b] = off;
    off = round_up(off + l.blob_sizes[b], kAlignLocal);
  }
  return off;
}

}  // namespace

extern "C" {

llama_status llama_stager_create(uint64_t slab_bytes, llama_stager** out) {
  if (!out) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "NULL out");
  auto* st = new (std::nothrow) llama_stager;
  if (!st) return llb::set_error(LLAMA_ERR_OOM, "out of host memory");
  st->cap = round_up(slab_bytes ? slab_bytes : (64ull << 20), kAlignLocal);
  cudaError_t e = cudaGetDevice(&st->device);
  for (int j = 0; j < kNB && e == cudaSuccess; ++j) {
    e = cudaMalloc(&st->buf[j][0], st->cap);
    if (e == cudaSuccess) e = cudaMalloc(&st->buf[j][1], st->cap);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st->e_in[j], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st->e_comp[j], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st->e_out[j], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaMalloc(&st->zero, 4096);
  if (e == cudaSuccess) e = cudaMemset(st->zero, 0, 4096);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st->e_start, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&st->e_done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st->h2d, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st->comp, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st->d2h, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete st;
    return cuda_err(e, "stager setup");
  }
  *out = st;
  return LLAMA_OK;
}

void llama_stager_destroy(llama_stager* st) { delete st; }

}  // extern "C"

namespace {

// One copy of a batch: validated, with its slab size.
struct StagedJob {
  const llama_mapping* sm;
  void* const* sb;
  const llama_mapping* dm;
  void* const* db;
  uint64_t n = 0;  // records per slab
  // n-body move instead of a copy (sm == dm, sb == db): in place per slab
  bool move = false;
  int32_t pos[3] = {0, 0, 0}, vel[3] = {0, 0, 0};
  float dt = 0.f;
};

llama_status prepare_job(llama_stager* st, StagedJob* jb) {
  if (!jb->sm || !jb->dm || !jb->sb || !jb->db) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  const llb::Mapping& s = jb->sm->m;
  const llb::Mapping& d = jb->dm->m;
  if (s.types != d.types) return llb::set_error(LLAMA_ERR_RECORD_MISMATCH, "record dimensions differ");
  if (s.extents != d.extents) return llb::set_error(LLAMA_ERR_SHAPE_MISMATCH, "array extents differ");
  for (int b = 0; b < s.nblobs(); ++b)
    if (s.blob_sizes[b] && !jb->sb[b]) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "NULL src blob");
  for (int b = 0; b < d.nblobs(); ++b)
    if (d.blob_sizes[b] && !jb->db[b]) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "NULL dst blob");
  const uint64_t N = s.N;
  if (d.collides())
    return llb::set_error(LLAMA_ERR_UNSUPPORTED, "destination maps several records onto one location");
  if (s.trace || d.trace)
    return llb::set_error(LLAMA_ERR_UNSUPPORTED, "staged copy of a traced view (use llama_copy)");
  if (s.lin != d.lin)  // equal storage orders: slabs of storage positions correspond
    return llb::set_error(LLAMA_ERR_UNSUPPORTED, "staged copy between differently linearised views");
  if (!s.uniform || !d.uniform || s.kind == LLAMA_ONE || d.kind == LLAMA_ONE)
    return llb::set_error(LLAMA_ERR_UNSUPPORTED, "staged copy of a split / one mapping (copy its blobs, then llama_copy)");
  if (d.footprint_bytes() == 0) return LLAMA_OK;
  // slab unit: whole blocks of every blocked side (lcm of the lane counts)
  uint64_t unit = 1;
  for (const llb::Mapping* m : {&s, &d})
    if (!m->soa()) unit = unit / gcd64(unit, m->L) * m->L;
  // slab size from the per-record footprint, then shrunk until both 1-D
  // views fit one staging buffer
  const uint64_t per = std::max<uint64_t>(1, std::max(s.footprint_bytes(), d.footprint_bytes()) / std::max<uint64_t>(N, 1));
  uint64_t n = std::max<uint64_t>(unit, st->cap / per / unit * unit);
  if (n > N) n = (N + unit - 1) / unit * unit;
  std::vector<uint64_t> lbs, lbd;
  for (;;) {
    const uint64_t nn = std::min(n, N);
    llama_mapping* ls = st->view(jb->sm, nn);
    llama_mapping* ld = st->view(jb->dm, nn);
    if (!ls || !ld) return llb::set_error(LLAMA_ERR_UNSUPPORTED, "cannot build slab views");
    if (layout_local(ls->m, &lbs) <= st->cap && layout_local(ld->m, &lbd) <= st->cap) break;
    if (n <= unit) return llb::set_error(LLAMA_ERR_UNSUPPORTED, "one slab of whole AoSoA blocks exceeds the staging buffer");
    n = std::max(unit, (n / 2) / unit * unit);
  }
  jb->n = n;
  return LLAMA_OK;
}

// Enqueues the slabs of one job; c counts slabs over the stager's lifetime, so
// the three buffers keep rotating from one job (and call) into the next (no
// drain between), and every reuse of a buffer waits for its previous slab.
llama_status enqueue_job(llama_stager* st, const StagedJob& jb, uint64_t* c) {
  const llb::Mapping& s = jb.sm->m;
  const llb::Mapping& d = jb.dm->m;
  if (jb.n == 0) return LLAMA_OK;  // nothing to write
  const uint64_t N = s.N, n = jb.n;
  cudaError_t e;
  // destination padding outside every slab range: gaps between aligned
  // SoA single-blob sub-arrays (reading #9) -> zero them from the device
  if (d.kind == LLAMA_SOA_SINGLE_BLOB && d.aligned) {
    uint64_t end = 0;
    for (int k = 0; k < d.K(); ++k) {
      if (d.base[k] > end) {
        e = cudaMemcpyAsync(static_cast<uint8_t*>(jb.db[0]) + end, st->zero, d.base[k] - end, cudaMemcpyDefault,
                            st->d2h);
        if (e != cudaSuccess) return cuda_err(e, "gap fill");
      }
      end = d.base[k] + d.N * d.sizes[k];
    }
  }
  std::vector<uint64_t> lbs, lbd;
  std::vector<Range> rs, rd;
  for (uint64_t a = 0; a < N; a += n, ++*c) {
    const uint64_t b = std::min(N, a + n);
    const int j = (int)(*c % kNB);
    llama_mapping* ls = st->view(jb.sm, b - a);
    llama_mapping* ld = st->view(jb.dm, b - a);
    if (!ls || !ld) return llb::set_error(LLAMA_ERR_UNSUPPORTED, "cannot build slab views");
    layout_local(ls->m, &lbs);
    layout_local(ld->m, &lbd);
    slab_ranges(s, ls->m, a, b, &rs);
    slab_ranges(d, ld->m, a, b, &rd);
    // h2d: buffer j is free once the slab that used it has gone back out
    if (*c >= (uint64_t)kNB && (e = cudaStreamWaitEvent(st->h2d, st->e_out[j], 0)) != cudaSuccess)
      return cuda_err(e, "h2d wait");
    for (const Range& r : rs) {
      e = cudaMemcpyAsync(st->buf[j][0] + lbs[r.lblob] + r.loff, static_cast<const uint8_t*>(jb.sb[r.gblob]) + r.goff,
                          r.len, cudaMemcpyDefault, st->h2d);
      if (e != cudaSuccess) return cuda_err(e, "h2d copy");
    }
    if ((e = cudaEventRecord(st->e_in[j], st->h2d)) != cudaSuccess) return cuda_err(e, "h2d event");
    // relayout of the slab's 1-D views in staging memory
    if ((e = cudaStreamWaitEvent(st->comp, st->e_in[j], 0)) != cudaSuccess) return cuda_err(e, "comp wait");
    std::vector<void*> ps(ls->m.nblobs()), pd(ld->m.nblobs());
    for (int q = 0; q < ls->m.nblobs(); ++q) ps[q] = st->buf[j][0] + lbs[q];
    for (int q = 0; q < ld->m.nblobs(); ++q) pd[q] = st->buf[j][jb.move ? 0 : 1] + lbd[q];
    llama_status cs = jb.move ? llama_nbody_move(ls, ps.data(), jb.pos, jb.vel, jb.dt, st->comp)
                              : llama_copy(ls, ps.data(), ld, pd.data(), st->comp);
    if (cs != LLAMA_OK) return cs;
    if ((e = cudaEventRecord(st->e_comp[j], st->comp)) != cudaSuccess) return cuda_err(e, "comp event");
    // d2h
    if ((e = cudaStreamWaitEvent(st->d2h, st->e_comp[j], 0)) != cudaSuccess) return cuda_err(e, "d2h wait");
    for (const Range& r : rd) {
      e = cudaMemcpyAsync(static_cast<uint8_t*>(jb.db[r.gblob]) + r.goff,
                          st->buf[j][jb.move ? 0 : 1] + lbd[r.lblob] + r.loff, r.len, cudaMemcpyDefault, st->d2h);
      if (e != cudaSuccess) return cuda_err(e, "d2h copy");
    }
    if ((e = cudaEventRecord(st->e_out[j], st->d2h)) != cudaSuccess) return cuda_err(e, "d2h event");
  }
  return LLAMA_OK;
}

}  // namespace

extern "C" {

llama_status llama_copy_staged_batch(llama_stager* st, int32_t count, const llama_mapping* const* src_maps,
                                     void* const* const* src_blobs, const llama_mapping* const* dst_maps,
                                     void* const* const* dst_blobs, void* stream) {
  if (!st || count < 0 || (count > 0 && (!src_maps || !src_blobs || !dst_maps || !dst_blobs)))
    return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  try {
    std::vector<StagedJob> jobs(count);
    for (int i = 0; i < count; ++i) {  // every copy is validated before anything is enqueued
      jobs[i] = StagedJob{src_maps[i], src_blobs[i], dst_maps[i], dst_blobs[i], 0};
      llama_status s = prepare_job(st, &jobs[i]);
      if (s != LLAMA_OK) return s;
    }
    cudaError_t e = cudaEventRecord(st->e_start, (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st->h2d, st->e_start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st->comp, st->e_start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st->d2h, st->e_start, 0);
    if (e != cudaSuccess) return cuda_err(e, "stream ordering");
    for (const StagedJob& jb : jobs) {
      llama_status s = enqueue_job(st, jb, &st->slabs);
      if (s != LLAMA_OK) return s;
    }
    if ((e = cudaEventRecord(st->e_done, st->d2h)) != cudaSuccess) return cuda_err(e, "done event");
    if ((e = cudaStreamWaitEvent((cudaStream_t)stream, st->e_done, 0)) != cudaSuccess) return cuda_err(e, "join");
    return LLAMA_OK;
  } catch (...) {
    return llb::set_error(LLAMA_ERR_OOM, "staged copy failed");
  }
}

llama_status llama_copy_staged(llama_stager* st, const llama_mapping* src_map, void* const* src_blobs,
                               const llama_mapping* dst_map, void* const* dst_blobs, void* stream) {
  return llama_copy_staged_batch(st, 1, &src_map, &src_blobs, &dst_map, &dst_blobs, stream);
}

llama_status llama_nbody_move_staged(llama_stager* st, const llama_mapping* m, void* const* blobs,
                                     const int32_t* pos_leaves, const int32_t* vel_leaves, float dt, void* stream) {
  if (!st || !m || !blobs || !pos_leaves || !vel_leaves) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  try {
    for (int c = 0; c < 3; ++c)
      for (int32_t k : {pos_leaves[c], vel_leaves[c]})
        if (k < 0 || k >= m->m.K() || m->m.sizes[k] != 4)
          return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "Pos / Vel leaves must be 4-byte leaf indices");
    StagedJob jb{m, blobs, m, blobs, 0};
    jb.move = true;
    for (int c = 0; c < 3; ++c) {
      jb.pos[c] = pos_leaves[c];
      jb.vel[c] = vel_leaves[c];
    }
    jb.dt = dt;
    llama_status s = prepare_job(st, &jb);
    if (s != LLAMA_OK) return s;
    cudaError_t e = cudaEventRecord(st->e_start, (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st->h2d, st->e_start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st->comp, st->e_start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st->d2h, st->e_start, 0);
    if (e != cudaSuccess) return cuda_err(e, "stream ordering");
    if ((s = enqueue_job(st, jb, &st->slabs)) != LLAMA_OK) return s;
    if ((e = cudaEventRecord(st->e_done, st->d2h)) != cudaSuccess) return cuda_err(e, "done event");
    if ((e = cudaStreamWaitEvent((cudaStream_t)stream, st->e_done, 0)) != cudaSuccess) return cuda_err(e, "join");
    return LLAMA_OK;
  } catch (...) {
    return llb::set_error(LLAMA_ERR_OOM, "staged move failed");
  }
}

}  // extern "C"
