// mapping.hpp -- the runtime mapping descriptor (§3.7) in the AoSoA
// normal form, plus the record-dimension schema parser.
#pragma once
#include <stdint.h>

#include <memory>
#include <string>
#include <vector>

#include "llama_b200.h"
#include "params.hpp"

namespace llb {

uint32_t scalar_size(llama_scalar t);

// Parses the schema grammar of S:122-126 and flattens it depth-first
// (P:290 static arrays -> n fields; P:296-309 declaration order).
// Returns false with a message on a malformed schema.
bool parse_schema(const std::string& schema, std::vector<llama_scalar>* leaves, std::string* err);

// A part of a mapping: leaves that share one uniform normal form (the whole
// mapping for the classic kinds; each inner mapping of a Split).
struct Part {
  llama_kind kind = LLAMA_AOS;
  bool aligned = false;
  uint64_t L = 1, B = 0, E = 0;
  uint64_t record_bytes = 0;  // the part's record size S (AoS / AoSoA)
  std::vector<int> leaves;    // leaf indices of the full record, increasing
  bool soa() const { return kind == LLAMA_SOA_SINGLE_BLOB || kind == LLAMA_SOA_MULTI_BLOB; }
};

// Device counters of a traced mapping (Trace / Heatmap); shared
// by the copies of a mapping handle, freed with the last one.
struct TraceBuffers {
  unsigned long long* hits = nullptr;  // one per leaf
  uint32_t* heat = nullptr;            // one per blob byte, blobs back to back
  std::vector<uint64_t> heat_base;     // start of each blob's counters
  uint64_t heat_count = 0;
  int device = 0;
  ~TraceBuffers();
};

struct Mapping {
  uint64_t id = 0;  // unique per process, keys the plan cache
  std::vector<llama_scalar> types;
  std::vector<uint32_t> sizes;
  std::vector<int64_t> extents;
  llama_kind kind = LLAMA_AOS;
  int64_t lanes = 1;
  bool aligned = false;

  uint64_t N = 0;            // product of extents
  uint64_t record_bytes = 0; // S (packed or aligned record size)
  std::vector<uint64_t> rec_off;  // leaf offsets inside one record

  // normal form: off(i,k) = base_k + (i / L_k) * B_k + F_k + (i % L_k) * s_k.
  // L / B are the mapping-wide values of the four uniform kinds; Lk / Bk
  // hold them per leaf (they differ between the parts of a Split).
  uint64_t L = 1, B = 0;
  bool uniform = true;  // every leaf shares L and B (not a Split)
  llama_linearizer lin = LLAMA_ROW_MAJOR;  // storage order of the array index
  std::vector<uint64_t> Lk, Bk;
  std::vector<uint64_t> base, F;
  std::vector<uint32_t> blob;
  std::vector<uint64_t> blob_sizes;
  uint64_t E = 0;            // records covered by the blobs (blocked: nblocks*L; SoA: N)
  std::vector<Part> parts;   // one for the classic kinds; a split's parts in blob order
  std::shared_ptr<TraceBuffers> trace;  // non-null: instrumented (Trace / Heatmap)

  int K() const { return (int)sizes.size(); }
  int nblobs() const { return (int)blob_sizes.size(); }
  bool soa() const { return kind == LLAMA_SOA_SINGLE_BLOB || kind == LLAMA_SOA_MULTI_BLOB; }
  // a leaf maps several records onto one location (One, or a One part of a Split)
  bool collides() const {
    for (int k = 0; k < K(); ++k)
      if (Bk[k] == 0 && Lk[k] < N && N > 1) return true;
    return false;
  }
  uint64_t payload_bytes() const;   // N * sum s_k
  uint64_t footprint_bytes() const; // sum of blob sizes
  bool has_padding() const { return footprint_bytes() != payload_bytes(); }
  uint64_t offset(uint64_t i, int k) const { return base[k] + (i / Lk[k]) * Bk[k] + F[k] + (i % Lk[k]) * sizes[k]; }
  DevSide dev_side() const;
  DevLeaf dev_leaf(int k) const;
  DevLin dev_lin() const;
  // storage position of an array index (row-major rank -> linearisation)
  uint64_t storage(const int64_t* index) const;
};

// Builds the descriptor; returns LLAMA_OK or an error with *err set.
llama_status build_mapping(const llama_mapping_desc& d, Mapping* m, std::string* err);

uint64_t next_mapping_id();
DevTrace dev_trace(const Mapping& m);  // trace.cpp; zeros when not traced

// Sets the linearisation (validated; a new id for the plan cache).
llama_status set_linearizer(Mapping* m, llama_linearizer lin, std::string* err);

// Split: leaves_a of the full record go to a, the rest to b.
llama_status build_split(const Mapping& a, const Mapping& b, const int32_t* leaves_a, int32_t n_a, Mapping* m,
                         std::string* err);

}  // namespace llb
