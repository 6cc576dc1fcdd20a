/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain C, no intrinsics,
 * no blocking or fusion: each function is the definition it cites, written out.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int log2_exact(int64_t e) { /* -1 unless e is a power of two */
  int b = 0;
  if (e < 1) return -1;
  while ((1ll << b) < e) ++b;
  return (1ll << b) == e ? b : -1;
}

int oracle_validate(const oracle_mapping* m) {
  if (!m || m->n_leaves < 1 || !m->leaf_size || m->rank < 1 || !m->extents) return -1;
  for (int32_t k = 0; k < m->n_leaves; ++k) {
    int32_t s = m->leaf_size[k];
    if (s != 1 && s != 2 && s != 4 && s != 8) return -1;
  }
  for (int32_t d = 0; d < m->rank; ++d)
    if (m->extents[d] < 0) return -1;
  if (m->kind < ORACLE_AOS || m->kind > ORACLE_SPLIT) return -1;
  if (m->lin < ORACLE_ROW_MAJOR || m->lin > ORACLE_MORTON || m->rank > 16) return -1;
  if (m->lin == ORACLE_MORTON) /* all extents equal and a power of two */
    for (int32_t d = 0; d < m->rank; ++d)
      if (m->extents[d] != m->extents[0] || log2_exact(m->extents[0]) < 0) return -1;
  if (m->kind == ORACLE_AOSOA && m->lanes < 1) return -1;
  if (m->kind == ORACLE_SPLIT) {
    /* inner_a maps the selected leaves, inner_b the rest; both
     * over the same extents; neither part may be empty. */
    const oracle_mapping* a = m->inner_a;
    const oracle_mapping* b = m->inner_b;
    if (!a || !b || !m->leaves_a || m->n_a < 1 || m->n_a >= m->n_leaves) return -1;
    if (oracle_validate(a) || oracle_validate(b)) return -1;
    if (a->n_leaves != m->n_a || b->n_leaves != m->n_leaves - m->n_a) return -1;
    if (a->rank != m->rank || b->rank != m->rank) return -1;
    for (int32_t d = 0; d < m->rank; ++d)
      if (a->extents[d] != m->extents[d] || b->extents[d] != m->extents[d]) return -1;
    int32_t ja = 0, jb = 0;
    for (int32_t k = 0; k < m->n_leaves; ++k) {
      if (ja < m->n_a && m->leaves_a[ja] == k) {
        if (a->leaf_size[ja] != m->leaf_size[k]) return -1;
        ++ja;
      } else {
        if (b->leaf_size[jb] != m->leaf_size[k]) return -1;
        ++jb;
      }
    }
    if (ja != m->n_a) return -1; /* leaves_a not increasing or out of range */
  }
  return 0;
}

/* Split: which part leaf k of a split belongs to (1 = inner_a) and
 * its leaf index inside that part (the coordinate re-indexed into the part). */
static int split_part(const oracle_mapping* m, int32_t k, int32_t* j) {
  int32_t ja = 0, jb = 0;
  for (int32_t q = 0; q < k; ++q) {
    if (ja < m->n_a && m->leaves_a[ja] == q) ++ja;
    else ++jb;
  }
  if (ja < m->n_a && m->leaves_a[ja] == k) { *j = ja; return 1; }
  *j = jb;
  return 0;
}

/* product of the extents. */
int64_t oracle_record_count(const oracle_mapping* m) {
  int64_t n = 1;
  for (int32_t d = 0; d < m->rank; ++d) n *= m->extents[d];
  return n;
}

int64_t oracle_linearize(const oracle_mapping* m, const int64_t* index) {
  for (int32_t d = 0; d < m->rank; ++d)
    if (index[d] < 0 || index[d] >= m->extents[d]) return -1;
  int64_t flat = 0;
  if (m->lin == ORACLE_COL_MAJOR) { /* first index fastest */
    for (int32_t d = m->rank - 1; d >= 0; --d) flat = flat * m->extents[d] + index[d];
    return flat;
  }
  if (m->lin == ORACLE_MORTON) { /* interleave the index bits */
    int bits = log2_exact(m->extents[0]);
    for (int b = 0; b < bits; ++b)
      for (int32_t d = 0; d < m->rank; ++d)
        flat |= ((index[d] >> b) & 1) << (b * m->rank + (m->rank - 1 - d));
    return flat;
  }
  /* P:414-416 (enumeration {0,0},{0,1},{0,2},{1,0}...): last index fastest */
  for (int32_t d = 0; d < m->rank; ++d) flat = flat * m->extents[d] + index[d];
  return flat;
}

/* Storage position of the record whose array index has row-major rank i. */
static uint64_t storage_index(const oracle_mapping* m, uint64_t i) {
  if (m->lin == ORACLE_ROW_MAJOR || m->kind == ORACLE_SPLIT) return i;
  int64_t index[16];
  uint64_t r = i;
  for (int32_t d = m->rank - 1; d >= 0; --d) { /* row-major rank -> index */
    index[d] = (int64_t)(r % (uint64_t)m->extents[d]);
    r /= (uint64_t)m->extents[d];
  }
  return (uint64_t)oracle_linearize(m, index);
}

/* S:60-66 sizeOfPacked / offsetOf(packed): leaves one after another, no padding. */
uint64_t oracle_packed_offsets(const oracle_mapping* m, uint64_t* offsets) {
  uint64_t off = 0;
  for (int32_t k = 0; k < m->n_leaves; ++k) {
    if (offsets) offsets[k] = off;
    off += (uint64_t)m->leaf_size[k];
  }
  return off;
}

/* S:69-77 sizeOfAligned / offsetOf(aligned): each leaf starts at the next
 * multiple of its alignment (= its size); the record size is rounded up to
 * the maximum leaf alignment. */
uint64_t oracle_aligned_offsets(const oracle_mapping* m, uint64_t* offsets) {
  uint64_t off = 0, max_align = 1;
  for (int32_t k = 0; k < m->n_leaves; ++k) {
    uint64_t a = (uint64_t)m->leaf_size[k];
    while (off % a != 0) off += 1;
    if (offsets) offsets[k] = off;
    off += a;
    if (a > max_align) max_align = a;
  }
  while (off % max_align != 0) off += 1;
  return off;
}

static uint64_t record_offsets(const oracle_mapping* m, uint64_t* offsets) {
  return m->aligned ? oracle_aligned_offsets(m, offsets) : oracle_packed_offsets(m, offsets);
}

/* SoA single blob: leaf sub-arrays one after another in leaf order.
 * With aligned=1 each sub-array start is rounded up to the leaf's size
 * (reading #9).  starts[k] = byte start of leaf k's sub-array;
 * returns the blob size. */
static uint64_t soa_sb_starts(const oracle_mapping* m, uint64_t* starts) {
  uint64_t n = (uint64_t)oracle_record_count(m);
  uint64_t off = 0;
  for (int32_t k = 0; k < m->n_leaves; ++k) {
    uint64_t s = (uint64_t)m->leaf_size[k];
    if (m->aligned)
      while (off % s != 0) off += 1;
    if (starts) starts[k] = off;
    off += n * s;
  }
  return off;
}

/* "a compile time blob count". */
int32_t oracle_blob_count(const oracle_mapping* m) {
  /* a split's blobs are inner_a's followed by inner_b's */
  if (m->kind == ORACLE_SPLIT) return oracle_blob_count(m->inner_a) + oracle_blob_count(m->inner_b);
  return m->kind == ORACLE_SOA_MB ? m->n_leaves : 1; /* SoA MB blobCount = leafCount */
}

/* "for each blob the size in bytes can be queried". Closed forms from
 * S:247 (AoS), S:263 (SoA MB), S:277 (SoA SB), S:281 (AoSoA, final block padded). */
void oracle_blob_sizes(const oracle_mapping* m, uint64_t* sizes) {
  uint64_t n = (uint64_t)oracle_record_count(m);
  switch (m->kind) {
    case ORACLE_AOS:
      sizes[0] = n * record_offsets(m, NULL);
      break;
    case ORACLE_SOA_MB:
      for (int32_t k = 0; k < m->n_leaves; ++k) sizes[k] = n * (uint64_t)m->leaf_size[k];
      break;
    case ORACLE_SOA_SB:
      sizes[0] = soa_sb_starts(m, NULL);
      break;
    case ORACLE_AOSOA: {
      uint64_t L = (uint64_t)m->lanes;
      uint64_t blocks = (n + L - 1) / L;
      sizes[0] = blocks * L * record_offsets(m, NULL);
      break;
    }
    case ORACLE_ONE: /* blobSize(0) = sizeOfAligned(dim), whatever the extents */
      sizes[0] = oracle_aligned_offsets(m, NULL);
      break;
    case ORACLE_SPLIT: /* inner_a's blob sizes, then inner_b's */
      oracle_blob_sizes(m->inner_a, sizes);
      oracle_blob_sizes(m->inner_b, sizes + oracle_blob_count(m->inner_a));
      break;
  }
}

/* blobNrAndOffset, one case per mapping of P:460-473, written from the
 * formulas of S:244-286:
 *   AoS: blob 0, off = i*S + offsetOf(k)
 *   SoA MB: blob k, off = i*s_k
 *   SoA SB:     blob 0, off = start_k + i*s_k
 *   AoSoA L: blob 0, off = (i/L)*L*S + offsetOf(k)*L + (i%L)*s_k
 *   One: blob 0, off = offsetOf_aligned(k), for every i
 *   Split: the part's own answer for the re-indexed
 *             leaf, blob number + blobCount(inner_a) for the inner_b part
 * where S / offsetOf are the packed or aligned record layout. */
int oracle_blob_nr_and_offset(const oracle_mapping* m, int64_t i, int32_t k,
                              int32_t* blob, uint64_t* offset) {
  if (k < 0 || k >= m->n_leaves) return -1;
  if (i < 0 || i >= oracle_record_count(m)) return -1;
  uint64_t s_k = (uint64_t)m->leaf_size[k];
  uint64_t ui = storage_index(m, (uint64_t)i);
  switch (m->kind) {
    case ORACLE_AOS: {
      uint64_t* offs = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)m->n_leaves);
      uint64_t S = record_offsets(m, offs);
      *blob = 0;
      *offset = ui * S + offs[k];
      free(offs);
      return 0;
    }
    case ORACLE_SOA_MB:
      *blob = k;
      *offset = ui * s_k;
      return 0;
    case ORACLE_SOA_SB: {
      uint64_t* starts = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)m->n_leaves);
      soa_sb_starts(m, starts);
      *blob = 0;
      *offset = starts[k] + ui * s_k;
      free(starts);
      return 0;
    }
    case ORACLE_AOSOA: {
      uint64_t* offs = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)m->n_leaves);
      uint64_t S = record_offsets(m, offs);
      uint64_t L = (uint64_t)m->lanes;
      uint64_t block = ui / L, lane = ui % L; /* i -> (i/L, i mod L) */
      *blob = 0;
      *offset = block * L * S + offs[k] * L + lane * s_k;
      free(offs);
      return 0;
    }
    case ORACLE_ONE: {
      uint64_t* offs = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)m->n_leaves);
      oracle_aligned_offsets(m, offs);
      *blob = 0;
      *offset = offs[k]; /* independent of i */
      free(offs);
      return 0;
    }
    case ORACLE_SPLIT: {
      int32_t j;
      if (split_part(m, k, &j)) return oracle_blob_nr_and_offset(m->inner_a, i, j, blob, offset);
      int rc = oracle_blob_nr_and_offset(m->inner_b, i, j, blob, offset);
      *blob += oracle_blob_count(m->inner_a);
      return rc;
    }
  }
  return -1;
}

/* A faster, equivalent evaluation of oracle_blob_nr_and_offset for the copy
 * loops: the per-leaf record offsets / sub-array starts are computed once
 * instead of per call.  The arithmetic per kind is the same as above. */
typedef struct addr_ctx {
  const oracle_mapping* m;
  uint64_t S;
  uint64_t* offs;   /* record offsets (AoS/AoSoA/One) or sub-array starts (SoA SB) */
  /* split: per leaf its part (1 = inner_a) and index in the part */
  struct addr_ctx* a;
  struct addr_ctx* b;
  int32_t* part;
  int32_t* idx;
  int32_t blobs_a;
} addr_ctx;

static void addr_ctx_init(addr_ctx* c, const oracle_mapping* m) {
  c->m = m;
  c->offs = (uint64_t*)calloc((size_t)m->n_leaves, sizeof(uint64_t));
  c->S = 0;
  c->a = c->b = NULL;
  c->part = c->idx = NULL;
  c->blobs_a = 0;
  if (m->kind == ORACLE_AOS || m->kind == ORACLE_AOSOA) c->S = record_offsets(m, c->offs);
  if (m->kind == ORACLE_SOA_SB) soa_sb_starts(m, c->offs);
  if (m->kind == ORACLE_ONE) c->S = oracle_aligned_offsets(m, c->offs);
  if (m->kind == ORACLE_SPLIT) {
    c->a = (addr_ctx*)malloc(sizeof(addr_ctx));
    c->b = (addr_ctx*)malloc(sizeof(addr_ctx));
    addr_ctx_init(c->a, m->inner_a);
    addr_ctx_init(c->b, m->inner_b);
    c->part = (int32_t*)malloc(sizeof(int32_t) * (size_t)m->n_leaves);
    c->idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)m->n_leaves);
    for (int32_t k = 0; k < m->n_leaves; ++k) c->part[k] = split_part(m, k, &c->idx[k]);
    c->blobs_a = oracle_blob_count(m->inner_a);
  }
}

static void addr_ctx_free(addr_ctx* c) {
  free(c->offs);
  if (c->a) { addr_ctx_free(c->a); free(c->a); }
  if (c->b) { addr_ctx_free(c->b); free(c->b); }
  free(c->part);
  free(c->idx);
}

static void addr_of(const addr_ctx* c, uint64_t i, int32_t k, int32_t* blob, uint64_t* offset) {
  const oracle_mapping* m = c->m;
  uint64_t s_k = (uint64_t)m->leaf_size[k];
  i = storage_index(m, i); /* i: row-major rank of the array index */
  switch (m->kind) {
    case ORACLE_ONE:
      *blob = 0;
      *offset = c->offs[k];
      return;
    case ORACLE_SPLIT:
      if (c->part[k]) {
        addr_of(c->a, i, c->idx[k], blob, offset);
      } else {
        addr_of(c->b, i, c->idx[k], blob, offset);
        *blob += c->blobs_a;
      }
      return;
    case ORACLE_AOS:
      *blob = 0;
      *offset = i * c->S + c->offs[k];
      return;
    case ORACLE_SOA_MB:
      *blob = k;
      *offset = i * s_k;
      return;
    case ORACLE_SOA_SB:
      *blob = 0;
      *offset = c->offs[k] + i * s_k;
      return;
    default: { /* ORACLE_AOSOA */
      uint64_t L = (uint64_t)m->lanes;
      *blob = 0;
      *offset = (i / L) * L * c->S + c->offs[k] * L + (i % L) * s_k;
      return;
    }
  }
}

/* splitmix64 output function (Steele, Lea, Flood 2014): the generator's mixer. */
uint64_t oracle_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void oracle_generate(const oracle_mapping* m, uint8_t* const* blobs,
                     const uint64_t* base, uint64_t seed, int64_t i0, int64_t i1) {
  addr_ctx c;
  addr_ctx_init(&c, m);
  uint64_t K = (uint64_t)m->n_leaves;
  for (int64_t i = i0; i < i1; ++i) {
    for (int32_t k = 0; k < m->n_leaves; ++k) {
      uint64_t v = oracle_splitmix64(seed ^ ((uint64_t)i * K + (uint64_t)k));
      int32_t b;
      uint64_t off;
      addr_of(&c, (uint64_t)i, k, &b, &off);
      uint8_t* p = blobs[b] + (off - (base ? base[b] : 0));
      for (int32_t j = 0; j < m->leaf_size[k]; ++j) p[j] = (uint8_t)(v >> (8 * j));
    }
  }
  addr_ctx_free(&c);
}

static int check_pair(const oracle_mapping* src, const oracle_mapping* dst) {
  if (oracle_validate(src) || oracle_validate(dst)) return -1;
  /* identical record dims and identical extents, else usage error. */
  if (src->n_leaves != dst->n_leaves) return -3;
  for (int32_t k = 0; k < src->n_leaves; ++k)
    if (src->leaf_size[k] != dst->leaf_size[k]) return -3;
  if (src->rank != dst->rank) return -2;
  for (int32_t d = 0; d < src->rank; ++d)
    if (src->extents[d] != dst->extents[d]) return -2;
  return 0;
}

/* "nested loops over the array and record dimensions and copies field-wise". */
static void copy_records(const addr_ctx* cs, const uint8_t* const* src_blobs, const uint64_t* src_base,
                         const addr_ctx* cd, uint8_t* const* dst_blobs, const uint64_t* dst_base,
                         int64_t i0, int64_t i1) {
  int32_t K = cs->m->n_leaves;
  for (int64_t i = i0; i < i1; ++i) {        /* array dimensions: outer loop */
    for (int32_t k = 0; k < K; ++k) {        /* record leaves: inner loop */
      int32_t bs, bd;
      uint64_t os, od;
      addr_of(cs, (uint64_t)i, k, &bs, &os);
      addr_of(cd, (uint64_t)i, k, &bd, &od);
      memcpy(dst_blobs[bd] + (od - (dst_base ? dst_base[bd] : 0)),
             src_blobs[bs] + (os - (src_base ? src_base[bs] : 0)),
             (size_t)cs->m->leaf_size[k]); /* bytes, never typed loads */
    }
  }
}

int oracle_copy_range(const oracle_mapping* src, const uint8_t* const* src_blobs,
                      const uint64_t* src_base, const oracle_mapping* dst,
                      uint8_t* const* dst_blobs, const uint64_t* dst_base,
                      int64_t i0, int64_t i1) {
  int rc = check_pair(src, dst);
  if (rc) return rc;
  int64_t n = oracle_record_count(src);
  if (i0 < 0 || i1 > n || i0 > i1) return -1;
  addr_ctx cs, cd;
  addr_ctx_init(&cs, src);
  addr_ctx_init(&cd, dst);
  copy_records(&cs, src_blobs, src_base, &cd, dst_blobs, dst_base, i0, i1);
  addr_ctx_free(&cs);
  addr_ctx_free(&cd);
  return 0;
}

int oracle_copy(const oracle_mapping* src, const uint8_t* const* src_blobs,
                const oracle_mapping* dst, uint8_t* const* dst_blobs, int32_t nthreads) {
  int rc = check_pair(src, dst);
  if (rc) return rc;
  /* Destination padding := 0 (reading #12): clear every dst blob first. */
  int32_t nb = oracle_blob_count(dst);
  uint64_t* sizes = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)nb);
  oracle_blob_sizes(dst, sizes);
  for (int32_t b = 0; b < nb; ++b) memset(dst_blobs[b], 0, (size_t)sizes[b]);
  free(sizes);

  addr_ctx cs, cd;
  addr_ctx_init(&cs, src);
  addr_ctx_init(&cd, dst);
  int64_t n = oracle_record_count(src);
  if (nthreads <= 1) {
    copy_records(&cs, src_blobs, NULL, &cd, dst_blobs, NULL, 0, n);
  } else {
    /* (p) variant: the array loop split into contiguous ranges,
     * one per thread. Result is independent of the partition. */
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads)
    {
      int64_t t = omp_get_thread_num(), T = omp_get_num_threads();
      int64_t a = n * t / T, b = n * (t + 1) / T;
      copy_records(&cs, src_blobs, NULL, &cd, dst_blobs, NULL, a, b);
    }
#else
    copy_records(&cs, src_blobs, NULL, &cd, dst_blobs, NULL, 0, n);
#endif
  }
  addr_ctx_free(&cs);
  addr_ctx_free(&cd);
  return 0;
}

/* Listing P:643-645: particles(i)(Pos{}) += particles(i)(Vel{}) * TIMESTEP, per
 * component, FP = float.  ONE rounding: p + v * dt as a fused
 * multiply-add (reading #25): the paper built its CPU n-body with -ffast-math
 * -mfma and its GPU n-body with nvcc --use_fast_math, both of
 * which contract the multiply-add.  C99 fmaf is correctly rounded on every
 * host (the file is built with -ffp-contract=off, so no other expression is
 * fused). */
int oracle_nbody_move(const oracle_mapping* m, uint8_t* const* blobs, const int32_t* pos, const int32_t* vel,
                      float dt, int64_t i0, int64_t i1) {
  if (oracle_validate(m)) return -1;
  int64_t n = oracle_record_count(m);
  if (i0 < 0 || i1 > n || i0 > i1) return -1;
  for (int c = 0; c < 3; ++c) {
    if (pos[c] < 0 || pos[c] >= m->n_leaves || vel[c] < 0 || vel[c] >= m->n_leaves) return -1;
    if (m->leaf_size[pos[c]] != 4 || m->leaf_size[vel[c]] != 4) return -1;
  }
  addr_ctx c;
  addr_ctx_init(&c, m);
  for (int64_t i = i0; i < i1; ++i) {
    for (int k = 0; k < 3; ++k) {
      int32_t bp, bv;
      uint64_t op, ov;
      addr_of(&c, (uint64_t)i, pos[k], &bp, &op);
      addr_of(&c, (uint64_t)i, vel[k], &bv, &ov);
      float p, v;
      memcpy(&p, blobs[bp] + op, 4);
      memcpy(&v, blobs[bv] + ov, 4);
      p = fmaf(v, dt, p);
      memcpy(blobs[bp] + op, &p, 4);
    }
  }
  addr_ctx_free(&c);
  return 0;
}

static void count(const oracle_mapping* m, const addr_ctx* c, uint64_t i, int32_t k, uint64_t* hits,
                  uint32_t* const* heat) {
  if (hits) hits[k] += 1;
  if (heat) {
    int32_t b;
    uint64_t o;
    addr_of(c, i, k, &b, &o);
    for (int32_t j = 0; j < m->leaf_size[k]; ++j) heat[b][o + (uint64_t)j] += 1;
  }
}

int oracle_copy_counted(const oracle_mapping* src, const uint8_t* const* src_blobs, const oracle_mapping* dst,
                        uint8_t* const* dst_blobs, uint64_t* src_hits, uint64_t* dst_hits,
                        uint32_t* const* src_heat, uint32_t* const* dst_heat) {
  int rc = oracle_copy(src, src_blobs, dst, dst_blobs, 1);
  if (rc) return rc;
  addr_ctx cs, cd;
  addr_ctx_init(&cs, src);
  addr_ctx_init(&cd, dst);
  int64_t n = oracle_record_count(src);
  for (int64_t i = 0; i < n; ++i)
    for (int32_t k = 0; k < src->n_leaves; ++k) {
      count(src, &cs, (uint64_t)i, k, src_hits, src_heat); /* the read of (i, k) */
      count(dst, &cd, (uint64_t)i, k, dst_hits, dst_heat); /* the write of (i, k) */
    }
  addr_ctx_free(&cs);
  addr_ctx_free(&cd);
  return 0;
}

int oracle_nbody_move_counted(const oracle_mapping* m, uint8_t* const* blobs, const int32_t* pos,
                              const int32_t* vel, float dt, uint64_t* hits, uint32_t* const* heat) {
  int64_t n = oracle_record_count(m);
  int rc = oracle_nbody_move(m, blobs, pos, vel, dt, 0, n);
  if (rc) return rc;
  addr_ctx c;
  addr_ctx_init(&c, m);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      count(m, &c, (uint64_t)i, pos[k], hits, heat); /* Pos_c += ...: one resolution */
      count(m, &c, (uint64_t)i, vel[k], hits, heat); /* ... Vel_c * dt: one resolution */
    }
  addr_ctx_free(&c);
  return 0;
}
