// trace.cpp -- Trace / Heatmap instrumentation (SURVEY
// §8(f) f4): device counters owned by a traced mapping, and their C ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "capi_internal.hpp"

namespace llb {

TraceBuffers::~TraceBuffers() {
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) return;  // CUDA already torn down
  cudaSetDevice(device);
  if (hits) cudaFree(hits);
  if (heat) cudaFree(heat);
  cudaSetDevice(cur);
}

DevTrace dev_trace(const Mapping& m) {
  DevTrace t;
  std::memset(&t, 0, sizeof(t));
  if (!m.trace) return t;
  t.hits = m.trace->hits;
  t.heat = m.trace->heat;
  for (size_t b = 0; b < m.trace->heat_base.size(); ++b) t.heat_base[b] = m.trace->heat_base[b];
  return t;
}

}  // namespace llb

namespace {

// Counters are read after ALL work on the counters' device: a traced copy may
// sit on a non-blocking stream (torch's streams, a stager's), which the
// legacy-stream cudaMemcpy below would not wait for.
cudaError_t sync_trace_device(const llb::TraceBuffers& t) {
  int cur = 0;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return e;
  if (cur != t.device && (e = cudaSetDevice(t.device)) != cudaSuccess) return e;
  e = cudaDeviceSynchronize();
  if (cur != t.device) cudaSetDevice(cur);
  return e;
}

}  // namespace

extern "C" {

llama_status llama_mapping_create_traced(const llama_mapping* inner, int32_t kinds, llama_mapping** out) {
  if (!inner || !out) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  if (kinds <= 0 || (kinds & ~(LLAMA_TRACE_FIELDS | LLAMA_TRACE_BYTES)))
    return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "kinds: LLAMA_TRACE_FIELDS and/or LLAMA_TRACE_BYTES");
  try {
    auto* m = new llama_mapping(*inner);
    auto tb = std::make_shared<llb::TraceBuffers>();
    cudaGetDevice(&tb->device);
    cudaError_t e = cudaSuccess;
    if (kinds & LLAMA_TRACE_FIELDS) {
      e = cudaMalloc(&tb->hits, sizeof(unsigned long long) * (size_t)std::max(1, m->m.K()));
      if (e == cudaSuccess) e = cudaMemset(tb->hits, 0, sizeof(unsigned long long) * (size_t)std::max(1, m->m.K()));
    }
    if (e == cudaSuccess && (kinds & LLAMA_TRACE_BYTES)) {
      for (uint64_t s : m->m.blob_sizes) {
        tb->heat_base.push_back(tb->heat_count);
        tb->heat_count += s;
      }
      e = cudaMalloc(&tb->heat, sizeof(uint32_t) * (size_t)std::max<uint64_t>(1, tb->heat_count));
      if (e == cudaSuccess) e = cudaMemset(tb->heat, 0, sizeof(uint32_t) * (size_t)std::max<uint64_t>(1, tb->heat_count));
    }
    if (e != cudaSuccess) {
      delete m;
      return llb::set_error(LLAMA_ERR_CUDA, std::string("trace counters: ") + cudaGetErrorString(e));
    }
    m->m.trace = tb;
    m->m.id = llb::next_mapping_id();  // a different mapping for the plan cache
    *out = m;
    return LLAMA_OK;
  } catch (...) {
    return llb::set_error(LLAMA_ERR_OOM, "out of host memory");
  }
}

llama_status llama_trace_field_hits(const llama_mapping* m, uint64_t* hits, int32_t capacity) {
  if (!m || !hits) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!m->m.trace || !m->m.trace->hits) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "mapping not traced with FIELDS");
  const int n = std::min(capacity, m->m.K());
  if (n <= 0) return LLAMA_OK;
  cudaError_t e = sync_trace_device(*m->m.trace);
  if (e == cudaSuccess) e = cudaMemcpy(hits, m->m.trace->hits, sizeof(uint64_t) * (size_t)n, cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? LLAMA_OK : llb::set_error(LLAMA_ERR_CUDA, cudaGetErrorString(e));
}

llama_status llama_trace_byte_hits(const llama_mapping* m, int32_t blob, uint32_t* hits, uint64_t capacity) {
  if (!m || !hits) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!m->m.trace || !m->m.trace->heat) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "mapping not traced with BYTES");
  if (blob < 0 || blob >= m->m.nblobs()) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "blob out of range");
  const uint64_t n = m->m.blob_sizes[blob];
  if (capacity < n) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "capacity below the blob size");
  if (n == 0) return LLAMA_OK;
  cudaError_t e = sync_trace_device(*m->m.trace);
  if (e == cudaSuccess) e = cudaMemcpy(hits, m->m.trace->heat + m->m.trace->heat_base[blob], sizeof(uint32_t) * n,
                             cudaMemcpyDeviceToHost);
  return e == cudaSuccess ? LLAMA_OK : llb::set_error(LLAMA_ERR_CUDA, cudaGetErrorString(e));
}

llama_status llama_trace_reset(const llama_mapping* m, void* stream) {
  if (!m) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!m->m.trace) return llb::set_error(LLAMA_ERR_INVALID_ARGUMENT, "mapping not traced");
  cudaError_t e = cudaSuccess;
  const auto& t = *m->m.trace;
  if (t.hits) e = cudaMemsetAsync(t.hits, 0, sizeof(unsigned long long) * (size_t)std::max(1, m->m.K()), (cudaStream_t)stream);
  if (e == cudaSuccess && t.heat)
    e = cudaMemsetAsync(t.heat, 0, sizeof(uint32_t) * (size_t)std::max<uint64_t>(1, t.heat_count), (cudaStream_t)stream);
  return e == cudaSuccess ? LLAMA_OK : llb::set_error(LLAMA_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
