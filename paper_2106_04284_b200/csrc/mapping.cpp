// mapping.cpp -- schema parser, record offsets and the AoSoA normal form.
#include "mapping.hpp"

#include <algorithm>
#include <atomic>
#include <cctype>

namespace llb {

uint32_t scalar_size(llama_scalar t) {
  switch (t) {
    case LLAMA_BOOL: case LLAMA_I8: case LLAMA_U8: return 1;
    case LLAMA_I16: case LLAMA_U16: return 2;
    case LLAMA_I32: case LLAMA_U32: case LLAMA_F32: return 4;
    case LLAMA_I64: case LLAMA_U64: case LLAMA_F64: return 8;
  }
  return 0;
}

// ----------------------------------------------------------------- schema
namespace {

struct SchemaParser {
  std::string s;
  size_t p = 0;
  std::string err;

  bool fail(const std::string& m) {
    if (err.empty()) err = m + " at position " + std::to_string(p);
    return false;
  }
  char peek() const { return p < s.size() ? s[p] : '\0'; }
  bool ident(std::string* out) {
    size_t st = p;
    while (p < s.size() && (std::isalnum((unsigned char)s[p]) || s[p] == '_')) ++p;
    if (st == p) return fail("expected a name");
    *out = s.substr(st, p - st);
    return true;
  }
  static bool scalar(const std::string& n, llama_scalar* t) {
    static const struct { const char* n; llama_scalar t; } tab[] = {
        {"bool", LLAMA_BOOL}, {"i8", LLAMA_I8},   {"u8", LLAMA_U8},   {"i16", LLAMA_I16},
        {"u16", LLAMA_U16},   {"i32", LLAMA_I32}, {"u32", LLAMA_U32}, {"i64", LLAMA_I64},
        {"u64", LLAMA_U64},   {"f32", LLAMA_F32}, {"f64", LLAMA_F64}};
    for (auto& e : tab)
      if (n == e.n) { *t = e.t; return true; }
    return false;
  }
  // A parsed node: a list of leaves (already flattened) -- arrays replicate it.
  bool array_dims(std::vector<int>* dims) {
    while (peek() == '[') {
      ++p;
      size_t st = p;
      while (std::isdigit((unsigned char)peek())) ++p;
      if (st == p) return fail("expected an array extent");
      long n = std::stol(s.substr(st, p - st));
      if (n < 1) return fail("zero-extent array");
      if (peek() != ']') return fail("expected ']'");
      ++p;
      dims->push_back((int)n);
    }
    return true;
  }
  bool replicate(std::vector<llama_scalar>* node, const std::vector<int>& dims) {
    size_t total = node->size();
    for (int n : dims) total *= (size_t)n;
    if (total > 100000) return fail("record too large");
    std::vector<llama_scalar> one = *node;
    for (auto it = dims.rbegin(); it != dims.rend(); ++it) {  // T[a][b] = record of a records of b T
      std::vector<llama_scalar> rep;
      for (int j = 0; j < *it; ++j) rep.insert(rep.end(), one.begin(), one.end());
      one.swap(rep);
    }
    node->swap(one);
    return true;
  }
  bool body(std::vector<llama_scalar>* out) {  // '{' field (',' field)* '}'
    if (peek() != '{') return fail("expected '{'");
    ++p;
    std::vector<std::string> tags;
    for (;;) {
      std::string tag;
      if (!ident(&tag)) return false;
      for (auto& t : tags)
        if (t == tag) return fail("duplicate tag '" + tag + "'");
      tags.push_back(tag);
      std::vector<llama_scalar> node;
      if (peek() == ':') {
        ++p;
        std::string name;
        if (!ident(&name)) return false;
        if (peek() == '{') {
          if (!body(&node)) return false;
        } else {
          llama_scalar t;
          if (!scalar(name, &t)) return fail("unknown scalar type '" + name + "'");
          node.push_back(t);
        }
      } else if (peek() == '{') {
        if (!body(&node)) return false;
      } else {
        return fail("expected ':' or '{' after tag '" + tag + "'");
      }
      std::vector<int> dims;
      if (!array_dims(&dims)) return false;
      if (!dims.empty() && !replicate(&node, dims)) return false;
      out->insert(out->end(), node.begin(), node.end());
      if (peek() == ',') { ++p; continue; }
      if (peek() == '}') { ++p; return true; }
      return fail("expected ',' or '}'");
    }
  }
};

}  // namespace

bool parse_schema(const std::string& schema, std::vector<llama_scalar>* leaves, std::string* err) {
  SchemaParser ps;
  for (char c : schema)
    if (!std::isspace((unsigned char)c)) ps.s.push_back(c);
  std::string name;
  leaves->clear();
  bool ok = ps.ident(&name);
  if (ok) {
    llama_scalar t;
    if (ps.peek() == '{') ok = ps.body(leaves);
    else if (SchemaParser::scalar(name, &t)) leaves->push_back(t);
    else ok = ps.fail("expected a record or a scalar");
  }
  if (ok && ps.p != ps.s.size()) ok = ps.fail("trailing text");
  if (!ok && err) *err = "schema: " + ps.err;
  return ok;
}

// ---------------------------------------------------------------- mapping
namespace {
std::atomic<uint64_t> g_next_id{1};

bool mul_ok(uint64_t a, uint64_t b, uint64_t* out) { return !__builtin_mul_overflow(a, b, out); }
uint64_t round_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }
}  // namespace

uint64_t Mapping::payload_bytes() const {
  uint64_t s = 0;
  for (auto v : sizes) s += v;
  return N * s;
}

uint64_t Mapping::footprint_bytes() const {
  uint64_t s = 0;
  for (auto v : blob_sizes) s += v;
  return s;
}

DevSide Mapping::dev_side() const {
  DevSide d{};
  d.L = L;
  d.B = B;
  d.lshift = (L & (L - 1)) == 0 ? (uint32_t)__builtin_ctzll(L) : kNoShift;
  return d;
}

DevLeaf Mapping::dev_leaf(int k) const {
  DevLeaf l{};
  l.base = base[k];
  l.F = F[k];
  l.L = Lk[k];
  l.B = Bk[k];
  l.blob = blob[k];
  l.size = sizes[k];
  if (Bk[k] == 0 && Lk[k] >= N) l.lshift = 63;  // a single block: i / L == 0 for every valid i
  else l.lshift = (Lk[k] & (Lk[k] - 1)) == 0 ? (uint32_t)__builtin_ctzll(Lk[k]) : kNoShift;
  return l;
}

uint64_t next_mapping_id() { return g_next_id.fetch_add(1); }

DevLin Mapping::dev_lin() const {
  DevLin l{};
  l.kind = (uint32_t)lin;
  l.rank = (uint32_t)extents.size();
  for (size_t d = 0; d < extents.size(); ++d) l.ext[d] = (uint64_t)extents[d];
  if (lin == LLAMA_MORTON && !extents.empty()) {
    while ((1ull << l.bits) < (uint64_t)extents[0]) ++l.bits;
  }
  return l;
}

uint64_t Mapping::storage(const int64_t* index) const {
  const size_t r = extents.size();
  uint64_t f = 0;
  if (lin == LLAMA_COL_MAJOR) {
    for (size_t d = r; d-- > 0;) f = f * (uint64_t)extents[d] + (uint64_t)index[d];
  } else if (lin == LLAMA_MORTON) {
    const DevLin l = dev_lin();
    for (uint32_t b = 0; b < l.bits; ++b)
      for (uint32_t d = 0; d < l.rank; ++d) f |= (((uint64_t)index[d] >> b) & 1ull) << (b * l.rank + (l.rank - 1 - d));
  } else {
    for (size_t d = 0; d < r; ++d) f = f * (uint64_t)extents[d] + (uint64_t)index[d];
  }
  return f;
}

llama_status set_linearizer(Mapping* m, llama_linearizer lin, std::string* err) {
  if (lin < LLAMA_ROW_MAJOR || lin > LLAMA_MORTON) { *err = "bad linearizer"; return LLAMA_ERR_INVALID_ARGUMENT; }
  if (lin == LLAMA_MORTON) {
    for (int64_t e : m->extents)
      if (e != m->extents[0] || e < 1 || (e & (e - 1)) != 0) {
        *err = "MORTON needs equal power-of-two extents (S:176)";
        return LLAMA_ERR_INVALID_ARGUMENT;
      }
  }
  m->lin = lin;
  m->id = g_next_id.fetch_add(1);
  return LLAMA_OK;
}

llama_status build_split(const Mapping& a, const Mapping& b, const int32_t* leaves_a, int32_t n_a, Mapping* m,
                         std::string* err) {
  const int K = a.K() + b.K();
  if (n_a != a.K()) { *err = "leaves_a must list exactly a's leaves"; return LLAMA_ERR_INVALID_ARGUMENT; }
  if (K > LLAMA_MAX_LEAVES) { *err = "more than LLAMA_MAX_LEAVES leaves"; return LLAMA_ERR_UNSUPPORTED; }
  if (a.extents != b.extents) { *err = "a and b must have the same extents"; return LLAMA_ERR_INVALID_ARGUMENT; }
  if (a.lin != b.lin) { *err = "a and b must have the same linearizer"; return LLAMA_ERR_INVALID_ARGUMENT; }
  if (a.nblobs() + b.nblobs() > LLAMA_MAX_BLOBS) { *err = "more than LLAMA_MAX_BLOBS blobs"; return LLAMA_ERR_UNSUPPORTED; }
  std::vector<int> in_a(K, -1);
  for (int j = 0; j < n_a; ++j) {
    if (leaves_a[j] < 0 || leaves_a[j] >= K || (j > 0 && leaves_a[j] <= leaves_a[j - 1])) {
      *err = "leaves_a must be strictly increasing leaf indices";
      return LLAMA_ERR_INVALID_ARGUMENT;
    }
    in_a[leaves_a[j]] = j;
  }
  *m = Mapping();
  m->extents = a.extents;
  m->N = a.N;
  m->kind = LLAMA_SPLIT;
  m->uniform = false;
  m->lin = a.lin;
  m->E = std::max(a.E, b.E);  // records the blobs cover: the largest of the parts
  int ib = 0;
  for (int k = 0; k < K; ++k) {
    const bool A = in_a[k] >= 0;
    const Mapping& s = A ? a : b;
    const int j = A ? in_a[k] : ib++;
    m->types.push_back(s.types[j]);
    m->sizes.push_back(s.sizes[j]);
    m->rec_off.push_back(0);
    m->Lk.push_back(s.Lk[j]);
    m->Bk.push_back(s.Bk[j]);
    m->base.push_back(s.base[j]);
    m->F.push_back(s.F[j]);
    m->blob.push_back(s.blob[j] + (A ? 0u : (uint32_t)a.nblobs()));
  }
  m->blob_sizes = a.blob_sizes;
  m->blob_sizes.insert(m->blob_sizes.end(), b.blob_sizes.begin(), b.blob_sizes.end());
  std::vector<int> full_b;  // leaf j of b is leaf full_b[j] of the split
  for (int k = 0; k < K; ++k)
    if (in_a[k] < 0) full_b.push_back(k);
  for (int X = 0; X < 2; ++X)
    for (const Part& q : (X == 0 ? a : b).parts) {
      Part r = q;
      for (int& l : r.leaves) l = X == 0 ? leaves_a[l] : full_b[l];
      m->parts.push_back(r);
    }
  m->id = g_next_id.fetch_add(1);
  return LLAMA_OK;
}

llama_status build_mapping(const llama_mapping_desc& d, Mapping* m, std::string* err) {
  if (!d.leaf_types || !d.extents) { *err = "NULL leaf_types or extents"; return LLAMA_ERR_INVALID_ARGUMENT; }
  if (d.n_leaves < 1 || d.rank < 1) { *err = "n_leaves and rank must be >= 1"; return LLAMA_ERR_INVALID_ARGUMENT; }
  if (d.n_leaves > LLAMA_MAX_LEAVES) { *err = "more than LLAMA_MAX_LEAVES leaves"; return LLAMA_ERR_UNSUPPORTED; }
  if (d.rank > LLAMA_MAX_RANK) { *err = "rank above LLAMA_MAX_RANK"; return LLAMA_ERR_UNSUPPORTED; }
  if (d.kind < LLAMA_AOS || d.kind > LLAMA_ONE) { *err = "bad kind"; return LLAMA_ERR_INVALID_ARGUMENT; }
  if (d.kind == LLAMA_AOSOA && d.lanes < 1) { *err = "AoSoA lanes must be >= 1"; return LLAMA_ERR_INVALID_ARGUMENT; }
  m->types.assign(d.leaf_types, d.leaf_types + d.n_leaves);
  m->sizes.clear();
  for (auto t : m->types) {
    uint32_t s = scalar_size(t);
    if (!s) { *err = "bad leaf type"; return LLAMA_ERR_INVALID_ARGUMENT; }
    m->sizes.push_back(s);
  }
  m->extents.assign(d.extents, d.extents + d.rank);
  uint64_t N = 1;
  for (auto e : m->extents) {
    if (e < 0) { *err = "negative extent"; return LLAMA_ERR_INVALID_ARGUMENT; }
    if (!mul_ok(N, (uint64_t)e, &N)) { *err = "record count overflows"; return LLAMA_ERR_UNSUPPORTED; }
  }
  if (N > (1ull << 40)) { *err = "more than 2^40 records"; return LLAMA_ERR_UNSUPPORTED; }
  m->N = N;
  m->kind = d.kind;
  m->lanes = d.kind == LLAMA_AOSOA ? d.lanes : 1;
  m->aligned = d.aligned != 0 || d.kind == LLAMA_ONE;  // One stores one aligned record
  const int K = d.n_leaves;

  // record offsets: packed or natural alignment
  m->rec_off.assign(K, 0);
  uint64_t off = 0, maxa = 1;
  for (int k = 0; k < K; ++k) {
    uint64_t s = m->sizes[k];
    if (m->aligned) off = round_up(off, s);
    m->rec_off[k] = off;
    off += s;
    if (s > maxa) maxa = s;
  }
  if (m->aligned) off = round_up(off, maxa);
  m->record_bytes = off;

  m->base.assign(K, 0);
  m->F.assign(K, 0);
  m->blob.assign(K, 0);
  m->blob_sizes.clear();
  uint64_t tmp;
  switch (d.kind) {
    case LLAMA_AOS:
    case LLAMA_AOSOA: {
      const uint64_t L = (uint64_t)m->lanes;
      m->L = L;
      if (!mul_ok(L, m->record_bytes, &m->B)) { *err = "block too large"; return LLAMA_ERR_UNSUPPORTED; }
      for (int k = 0; k < K; ++k) m->F[k] = L * m->rec_off[k];
      uint64_t nblocks = (N + L - 1) / L;  // tail block padded (reading #7)
      if (!mul_ok(nblocks, m->B, &tmp) || !mul_ok(nblocks, L, &m->E)) { *err = "blob size overflows"; return LLAMA_ERR_UNSUPPORTED; }
      m->blob_sizes.push_back(tmp);
      break;
    }
    case LLAMA_SOA_MULTI_BLOB:
      m->L = N > 0 ? N : 1;
      m->B = 0;
      m->E = N;
      for (int k = 0; k < K; ++k) {
        m->blob[k] = (uint32_t)k;
        if (!mul_ok(N, m->sizes[k], &tmp)) { *err = "blob size overflows"; return LLAMA_ERR_UNSUPPORTED; }
        m->blob_sizes.push_back(tmp);
      }
      if (K > LLAMA_MAX_BLOBS) { *err = "more than LLAMA_MAX_BLOBS blobs"; return LLAMA_ERR_UNSUPPORTED; }
      break;
    case LLAMA_ONE:  // every record at the same place (L = 1, B = 0)
      m->L = 1;
      m->B = 0;
      m->E = N;
      for (int k = 0; k < K; ++k) m->F[k] = m->rec_off[k];
      m->blob_sizes.push_back(m->record_bytes);
      break;
    case LLAMA_SOA_SINGLE_BLOB: {
      m->L = N > 0 ? N : 1;
      m->B = 0;
      m->E = N;
      uint64_t start = 0;
      for (int k = 0; k < K; ++k) {
        if (m->aligned) start = round_up(start, m->sizes[k]);  // reading #9
        m->base[k] = start;
        if (!mul_ok(N, m->sizes[k], &tmp)) { *err = "blob size overflows"; return LLAMA_ERR_UNSUPPORTED; }
        start += tmp;
      }
      m->blob_sizes.push_back(start);
      break;
    }
  }
  m->Lk.assign(K, m->L);
  m->Bk.assign(K, m->B);
  Part whole;
  whole.kind = m->kind;
  whole.aligned = m->aligned;
  whole.L = m->L;
  whole.B = m->B;
  whole.E = m->E;
  whole.record_bytes = m->record_bytes;
  for (int k = 0; k < K; ++k) whole.leaves.push_back(k);
  m->parts.assign(1, whole);
  m->id = g_next_id.fetch_add(1);
  return LLAMA_OK;
}

}  // namespace llb
