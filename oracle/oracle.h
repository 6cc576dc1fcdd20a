/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the LLAMA layout-aware
 * copy (arXiv 2106.04284), used as the parity oracle for the CUDA path in
 * paper_2106_04284_b200/.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or constant with the CUDA path, and must never be called
 * from the product path.
 *
 * Citation convention: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
 *
 * What it computes (§3.9 "Copying between views", §4.2 "naive copy"):
 *   for every array index i (row-major) and every leaf k (DFS order,
 *   P:296-309): dst[blob_d(i,k)][off_d(i,k) .. +s_k) = src[blob_s(i,k)][off_s(i,k) .. +s_k)
 * where (blob, off) is the mapping's blobNrAndOffset (§3.7), written
 * out per mapping kind directly from the definitions;
 * destination padding bytes are written as 0 (reading #12).
 *
 * Parity status: every function here is pinned by tests/test_oracle_pins.py
 * (worked examples, closed forms, C-compiler / numpy layouts, special cases,
 * invariants, brute force).  No function is "parity unpinned".
 */
#ifndef LLAMA_ORACLE_H
#define LLAMA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mapping kinds. */
enum { ORACLE_AOS = 0, ORACLE_SOA_SB = 1, ORACLE_SOA_MB = 2, ORACLE_AOSOA = 3, ORACLE_ONE = 4, ORACLE_SPLIT = 5 };

/* Linearisations of the array index ("storage order ... row- or
 * column-major ... space filling curves such as Morton codes"). */
enum { ORACLE_ROW_MAJOR = 0, ORACLE_COL_MAJOR = 1, ORACLE_MORTON = 2 };

/* A mapping as the oracle sees it: the flattened leaf sizes (DFS order; each
 * leaf's alignment equals its size), the array extents (row-major),
 * the kind, the AoSoA lane count L (ignored otherwise) and packed/aligned.
 * ORACLE_ONE always uses the aligned record layout.
 * ORACLE_SPLIT: the leaves listed in leaves_a[0..n_a)
 * (increasing) are mapped by inner_a -- a mapping of just those leaves, in
 * order -- and the others by inner_b; the other fields of a split describe
 * the full record (leaf sizes, extents); lanes / aligned are ignored. */
typedef struct oracle_mapping {
  int32_t n_leaves;
  const int32_t* leaf_size; /* bytes, each in {1,2,4,8} */
  int32_t rank;
  const int64_t* extents;
  int32_t kind;
  int64_t lanes;
  int32_t aligned; /* 0 = tightly packed, 1 = natural alignment */
  const struct oracle_mapping* inner_a; /* ORACLE_SPLIT only */
  const struct oracle_mapping* inner_b;
  const int32_t* leaves_a;
  int32_t n_a;
  int32_t lin; /* ORACLE_ROW_MAJOR (default) / COL_MAJOR / MORTON; a split's parts carry their own */
} oracle_mapping;

/* Returns 0 if the mapping is well formed, -1 otherwise. */
int oracle_validate(const oracle_mapping* m);

/* Number of records = product of extents. */
int64_t oracle_record_count(const oracle_mapping* m);

/* The mapping's linearisation of an array index (its storage position):
 *   row-major, last index fastest;
 *   column-major, first index fastest;
 *   Morton: bit b of index[d] goes to bit b*rank + (rank-1-d) of the code
 *   (all extents equal powers of two; reading #26).
 * Returns -1 on an out-of-range index.  Records are otherwise identified
 * everywhere in this oracle by their array index's ROW-MAJOR rank i (the
 * iteration order); the address functions below apply the
 * mapping's linearisation to it. */
int64_t oracle_linearize(const oracle_mapping* m, const int64_t* index);

/* Record-level offsets.  offsets[k] of leaf k within
 * one record; return value = record size.  packed: sum of sizes, no padding.
 * aligned: each leaf starts at the next multiple of its size; the record size
 * is rounded up to the largest leaf alignment. */
uint64_t oracle_packed_offsets(const oracle_mapping* m, uint64_t* offsets);
uint64_t oracle_aligned_offsets(const oracle_mapping* m, uint64_t* offsets);

/* Blob count and sizes. */
int32_t oracle_blob_count(const oracle_mapping* m);
void oracle_blob_sizes(const oracle_mapping* m, uint64_t* sizes);

/* blobNrAndOffset for flat index i and leaf k. Returns 0 / -1. */
int oracle_blob_nr_and_offset(const oracle_mapping* m, int64_t i, int32_t k,
                              int32_t* blob, uint64_t* offset);

/* The seeded input generator (an input recipe, not the method): byte b of leaf
 * k of record i is byte b (little endian) of splitmix64(seed ^ (i*K + k)).
 * Writes the leaves of records [i0,i1) through the oracle's own address
 * function.  Blob pointers are windows: blobs[b] holds the bytes starting at
 * global blob offset base[b] (base may be NULL = all zero). */
uint64_t oracle_splitmix64(uint64_t x);
void oracle_generate(const oracle_mapping* m, uint8_t* const* blobs,
                     const uint64_t* base, uint64_t seed, int64_t i0, int64_t i1);

/* The copy (P:757 naive copy: array loop outer, leaf loop inner, one s_k-byte
 * element copy per (i,k) via both mappings' blobNrAndOffset).  Copies records
 * [i0,i1) only; does NOT clear dst (the caller supplies zeroed windows).
 * Returns 0, or -2 shape mismatch (extents), -3 record mismatch (leaf sizes),
 * -1 invalid. */
int oracle_copy_range(const oracle_mapping* src, const uint8_t* const* src_blobs,
                      const uint64_t* src_base, const oracle_mapping* dst,
                      uint8_t* const* dst_blobs, const uint64_t* dst_base,
                      int64_t i0, int64_t i1);

/* Whole-view copy: zero-fills every dst blob (padding := 0), then copies all
 * records. nthreads > 1 runs the paper's "(p)" variant: the array loop is
 * split over OpenMP threads. */
int oracle_copy(const oracle_mapping* src, const uint8_t* const* src_blobs,
                const oracle_mapping* dst, uint8_t* const* dst_blobs, int32_t nthreads);

/* n-body move (Listing P:643-645, §4.1), FP = float
 * (P:618): for every particle i in [i0, i1) and c in {X, Y, Z}
 *   Pos_c(i) = Pos_c(i) + Vel_c(i) * dt
 * in f32 with one rounding (a fused multiply-add, fmaf; DESIGN.md reading
 * #25), reading and writing through the oracle's own address function.
 * pos[3] / vel[3] are the leaf indices of Pos.{X,Y,Z} / Vel.{X,Y,Z}; those
 * leaves must be 4 bytes.  Every other byte is left as it is.
 * Returns 0, or -1 for an invalid mapping / leaf / range. */
int oracle_nbody_move(const oracle_mapping* m, uint8_t* const* blobs, const int32_t* pos, const int32_t* vel,
                      float dt, int64_t i0, int64_t i1);

/* Trace and Heatmap: the
 * whole-view copy and the move, counting every address resolution.
 * *_hits[k] += 1 per resolution of leaf k (NULL: not counted);
 * *_heat[b][o] += 1 for every byte o of the resolved range in blob b (NULL:
 * not counted).  The copy resolves each (i, k) once on each side; the move
 * resolves Pos_c once (the compound +=) and Vel_c once per particle. */
int oracle_copy_counted(const oracle_mapping* src, const uint8_t* const* src_blobs, const oracle_mapping* dst,
                        uint8_t* const* dst_blobs, uint64_t* src_hits, uint64_t* dst_hits,
                        uint32_t* const* src_heat, uint32_t* const* dst_heat);
int oracle_nbody_move_counted(const oracle_mapping* m, uint8_t* const* blobs, const int32_t* pos,
                              const int32_t* vel, float dt, uint64_t* hits, uint32_t* const* heat);

#ifdef __cplusplus
}
#endif
#endif
