// plan.cpp -- chooses the kernel path for a mapping pair and precomputes its
// parameter block.
#include "plan.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>

namespace llb {

namespace {

constexpr uint64_t kAosLikeMaxBlock = 16384;  // larger AoSoA blocks are tiled inside a block
constexpr int kBarBytes = 128;

// Tuning knobs (llama_knob, include/llama_b200.h): the defaults written at
// each use below are the measured choices on B200; a caller overrides them
// only explicitly through llama_copy_options.knobs (the plan cache keys on
// the values), never through the environment.

uint64_t gcd64(uint64_t a, uint64_t b) {
  while (b) { uint64_t t = a % b; a = b; b = t; }
  return a;
}
uint64_t lcm64(uint64_t a, uint64_t b) { return a / gcd64(a, b) * b; }
uint64_t lowbit(uint64_t x) { return x ? (x & (~x + 1)) : (1ull << 62); }
uint64_t align16(uint64_t x) { return (x + 15) & ~15ull; }
uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

bool same_layout(const Mapping& s, const Mapping& d) {
  if (s.Lk != d.Lk || s.Bk != d.Bk || s.blob_sizes != d.blob_sizes) return false;
  for (int k = 0; k < s.K(); ++k)
    if (s.base[k] != d.base[k] || s.F[k] != d.F[k] || s.blob[k] != d.blob[k]) return false;
  return true;
}

}  // namespace

llama_status check_compatible(const Mapping& s, const Mapping& d, std::string* err) {
  if (s.types != d.types) {
    *err = "record dimensions differ (leaf type lists are not identical)";
    return LLAMA_ERR_RECORD_MISMATCH;
  }
  if (s.extents != d.extents) {
    *err = "array extents differ";
    return LLAMA_ERR_SHAPE_MISMATCH;
  }
  return LLAMA_OK;
}

FillParams make_fill(const Mapping& m, uint8_t value) {
  FillParams f;
  std::memset(&f, 0, sizeof(f));
  f.nb = m.nblobs();
  f.value = value;
  f.vstart[0] = 0;
  for (int b = 0; b < f.nb; ++b) {
    f.bytes[b] = m.blob_sizes[b];
    f.vstart[b + 1] = f.vstart[b] + ceil_div(m.blob_sizes[b], 16);
  }
  return f;
}

void plan_naive(const Mapping& s, const Mapping& d, Plan* p) {
  p->path = LLAMA_PATH_NAIVE;
  p->naive.reset(new NaiveParams);
  NaiveParams& n = *p->naive;
  std::memset(&n, 0, sizeof(n));
  n.N = s.N;
  n.K = s.K();
  n.relin = s.lin != d.lin ? 1 : 0;
  n.slin = s.dev_lin();
  n.dlin = d.dev_lin();
  n.traced = (s.trace || d.trace) ? 1 : 0;
  n.tr[0] = dev_trace(s);
  n.tr[1] = dev_trace(d);
  for (int k = 0; k < s.K(); ++k) {
    n.sl[k] = s.dev_leaf(k);
    n.dl[k] = d.dev_leaf(k);
  }
  p->naive_zero_fill = d.has_padding();  // padding := 0 (reading #12)
  if (p->naive_zero_fill) p->fill.reset(new FillParams(make_fill(d, 0)));
}

// 2-d views of different linearisations, records small enough for 32x32
// tiles in <= 48 KB of shared memory, not traced.
bool plan_transpose(const Mapping& s, const Mapping& d, const Knobs& kn, Plan* p, std::string* why) {
  if (s.trace || d.trace) { *why = "traced views count through the naive kernel"; return false; }
  if (s.lin == d.lin) { *why = "equal linearisations"; return false; }
  if (s.extents.size() != 2) { *why = "TRANSPOSE is for 2-d views"; return false; }
  uint64_t smem = 0;
  uint32_t base[kMaxLeaves];
  for (int k = 0; k < s.K(); ++k) {
    smem = (smem + 7) & ~7ull;
    base[k] = (uint32_t)smem;
    smem += 32ull * 32 * s.sizes[k];  // 32 x 32 swizzled tile (k_simple.cu tile_slot)
  }
  if (smem > 48 * 1024) { *why = "records too wide for 32x32 tiles"; return false; }
  plan_naive(s, d, p);
  p->path = LLAMA_PATH_TRANSPOSE;
  NaiveParams& n = *p->naive;
  n.H = (uint64_t)s.extents[0];
  n.W = (uint64_t)s.extents[1];
  n.tsmem = (uint32_t)smem;
  for (int k = 0; k < s.K(); ++k) n.tbase[k] = base[k];
  n.tuniform = (s.uniform && d.uniform) ? 1 : 0;
  // linear sides: L = 1 (AoS, One) or one block of all records (SoA); the
  // kernel then locates leaf elements with one 32-bit multiply-add
  n.tlinear = n.tuniform && s.N < (1ull << 32);
  for (const Mapping* m : {&s, &d})
    for (int k = 0; k < m->K(); ++k)
      if (!((m->Lk[k] == 1 && m->Bk[k] < (1ull << 32)) || m->Lk[k] >= m->N)) n.tlinear = 0;
  if (!kn.get(LLAMA_KNOB_TRANSPOSE_LINEAR, 1)) n.tlinear = 0;
  n.raw_typed = (uint32_t)kn.get(LLAMA_KNOB_TRANSPOSE_RAW_TYPED, 1);
  if (n.tlinear) {  // one leaf size of 4 or 8 bytes: the two-leaf pass (k_simple.cu lin_tile_fixed)
    const uint64_t z = s.sizes[0];
    bool same = (z == 4 || z == 8) && kn.get(LLAMA_KNOB_TRANSPOSE_FIXED, 1);
    for (int k = 0; k < s.K(); ++k) same = same && s.sizes[k] == z;
    n.tlinear = same ? (uint32_t)z : 1;
  }
  // plain AoS sides move whole tiles as 16-byte vectors through a raw record
  // buffer: every 32-record row / column segment (a 1024-record Morton tile)
  // must start 16-byte aligned
  uint64_t raw_bytes = 0;
  for (int X = 0; X < 2; ++X) {
    const Mapping& m = X == 0 ? s : d;
    const uint64_t S = m.B;
    bool ok = m.uniform && m.kind == LLAMA_AOS && m.L == 1 && m.base[0] % 16 == 0 && (32 * S) % 16 == 0 &&
              kn.get(LLAMA_KNOB_TRANSPOSE_RAW, 1);
    if (m.lin == LLAMA_ROW_MAJOR) ok = ok && ((uint64_t)m.extents[1] * S) % 16 == 0;
    if (m.lin == LLAMA_COL_MAJOR) ok = ok && ((uint64_t)m.extents[0] * S) % 16 == 0;
    if (ok) {
      if (X == 1) n.dpad = m.has_padding() ? 1 : 0;
      (X == 0 ? n.sraw : n.draw) = 1;
      (X == 0 ? n.sS : n.dS) = (uint32_t)S;
      raw_bytes = std::max<uint64_t>(raw_bytes, 1024 * S);
    }
  }
  // measured (4096^2 Particle7): raw on both sides 1.54 -> 2.37 TB/s; one
  // raw side next to an element-wise SoA side is slower than element-wise
  // on both (2.52 -> 2.22 TB/s: the raw code's registers cost occupancy)
  if (!(n.sraw && n.draw) && !(n.tlinear && kn.get(LLAMA_KNOB_TRANSPOSE_RAW1, 1))) n.sraw = n.draw = 0, raw_bytes = 0;
  if (raw_bytes) {
    smem = (smem + 15) & ~15ull;
    n.rawoff = (uint32_t)smem;
    smem += raw_bytes;
    if (smem > 100 * 1024) {  // keep two CTAs per SM; else element-wise sides
      smem = n.rawoff;
      n.sraw = n.draw = 0;
      n.rawoff = 0;
    }
    n.tsmem = (uint32_t)smem;
  }
  // per-CTA leaf table of both sides (k_simple.cu LinEnt, 16 B per leaf);
  // not next to a raw buffer (Particle7: 56 KB of tile + raw buffer fill a
  // quarter SM exactly, the table would cost a CTA per SM: -17%)
  if (n.tlinear && !n.sraw && !n.draw && kn.get(LLAMA_KNOB_TRANSPOSE_TABLE, 1)) {
    smem = (smem + 15) & ~15ull;
    n.linoff = (uint32_t)smem;
    smem += 2ull * 16 * s.K();
    n.tsmem = (uint32_t)smem;
  }
  n.taligned = 1;  // blobs are 16-B aligned: check the normal forms
  for (const Mapping* m : {&s, &d})
    for (int k = 0; k < m->K(); ++k) {
      const uint64_t z = m->sizes[k];
      const bool one_block = m->Bk[k] == 0 && m->Lk[k] >= m->N;
      if ((m->base[k] + m->F[k]) % z || (!one_block && m->Bk[k] % z)) n.taligned = 0;
    }
  return true;
}

// ------------------------------------------------ wide transposing copy (f4)
// Rank-2 views of different storage orders with records too wide for the JIT
// transpose's TY x 32 tiles (k_transpose_wide.cu).  A side is "A" (plain AoS:
// one part, L = 1, stride S % 4 == 0) or "E" (anything else, element-wise).
namespace {

// (r2) AoSoA-L sides (L a power of two <= 64) are image sides too when the
// tile's runs hold whole blocks (checked against the tile shape below)
bool wide_a_side(const Mapping& m) {
  const bool pow2 = m.L >= 1 && (m.L & (m.L - 1)) == 0;
  return m.uniform && m.parts.size() == 1 && (m.kind == LLAMA_AOS || m.kind == LLAMA_AOSOA) && pow2 && m.L <= 64 &&
         m.B > 0 && m.B % 4 == 0 && m.B / m.L <= 4096 && (m.B / m.L) * m.L == m.B;
}

// alignment (power of two <= 16) of every element address of leaf k on an E side
uint32_t wide_e_align(const Mapping& m, int k) {
  uint64_t a = gcd64(16, m.base[k] + m.F[k]);
  a = gcd64(a, m.sizes[k]);
  if (m.Lk[k] < m.N) a = gcd64(a, m.Bk[k]);
  return (uint32_t)a;
}

// largest chunk (16, 8, 4) dividing every run start and full-run length of
// an A side whose runs hold 2^lrun records
uint32_t wide_chunk(const Mapping& m, uint32_t lrun) {
  // (bytes per record position of a run: B / L for AoSoA-L images)
  const uint64_t S = m.B / m.L, H = (uint64_t)m.extents[0], W = (uint64_t)m.extents[1];
  for (uint32_t c : {16u, 8u, 4u}) {
    bool ok = m.base[0] % c == 0 && ((S << lrun) % c == 0);
    if (m.lin == LLAMA_ROW_MAJOR) ok = ok && (W * S) % c == 0;
    if (m.lin == LLAMA_COL_MAJOR) ok = ok && (H * S) % c == 0;
    if (ok) return c;
  }
  return 4;
}

// host copies of the kernel's tile orders (k_transpose_wide.cu t_rc / rc_t)
uint32_t h_compact(uint32_t x) {
  uint32_t r = 0;
  for (int b = 0; b < 16; ++b) r |= ((x >> (2 * b)) & 1u) << b;
  return r;
}
uint32_t h_part(uint32_t x) {
  uint32_t r = 0;
  for (int b = 0; b < 16; ++b) r |= ((x >> b) & 1u) << (2 * b);
  return r;
}
void h_t_rc(uint32_t lin, uint32_t t, uint32_t lty, uint32_t ltx, uint32_t& r, uint32_t& c) {
  if (lin == LLAMA_ROW_MAJOR) r = t >> ltx, c = t & ((1u << ltx) - 1);
  else if (lin == LLAMA_COL_MAJOR) c = t >> lty, r = t & ((1u << lty) - 1);
  else c = h_compact(t), r = h_compact(t >> 1);
}
uint32_t h_rc_t(uint32_t lin, uint32_t r, uint32_t c, uint32_t lty, uint32_t ltx) {
  if (lin == LLAMA_ROW_MAJOR) return (r << ltx) | c;
  if (lin == LLAMA_COL_MAJOR) return (c << lty) | r;
  return h_part(c) | (h_part(r) << 1);
}

// Shared-memory wavefronts of one warp's 4-byte accesses at byte offsets `off`
// (the most distinct words that fall into one bank).
uint32_t wavefronts(const std::vector<uint64_t>& off) {
  std::vector<std::vector<uint64_t>> bank(32);
  for (uint64_t o : off) {
    auto& b = bank[(o / 4) % 32];
    if (std::find(b.begin(), b.end(), o / 4) == b.end()) b.push_back(o / 4);
  }
  size_t w = 1;
  for (auto& b : bank) w = std::max(w, b.size());
  return (uint32_t)w;
}

// Image pitch of an A side: the run bytes rounded up to the chunk, then the
// candidate (within 16 chunks) whose warp accesses of the move phase take the
// fewest wavefronts.  `lanes(i)` gives warp 0's records (indices along the A
// side's own order) of access i.
template <typename Lanes>
uint32_t wide_pitch(uint64_t run_bytes, uint32_t chunk, uint32_t nruns, uint32_t S, uint32_t lrun, int n_acc,
                    Lanes lanes) {
  const uint64_t p0 = (run_bytes + chunk - 1) / chunk * chunk;
  if (nruns <= 1) return (uint32_t)p0;
  uint64_t best = p0;
  uint32_t best_w = ~0u;
  for (uint64_t p = p0; p < p0 + 16 * chunk; p += chunk) {
    uint32_t w = 0;
    for (int i = 0; i < n_acc; ++i) {
      std::vector<uint64_t> off;
      for (uint32_t t : lanes(i)) off.push_back((t >> lrun) * p + (t & ((1u << lrun) - 1)) * (uint64_t)S);
      w += wavefronts(off);
    }
    if (w < best_w) best_w = w, best = p;
  }
  return (uint32_t)best;
}

uint32_t ilog2(uint64_t x) {
  uint32_t r = 0;
  while ((1ull << (r + 1)) <= x) ++r;
  return r;
}

}  // namespace

static bool plan_wide_impl(const Mapping& s, const Mapping& d, const Knobs& kn, Plan* p, std::string* why) {
  if (s.trace || d.trace) { *why = "traced views count through the naive kernel"; return false; }
  if (s.lin == d.lin) { *why = "equal linearisations"; return false; }
  if (s.extents.size() != 2) { *why = "the wide transposing copy is for 2-d views"; return false; }
  if (!kn.get(LLAMA_KNOB_WIDE, 1)) { *why = "knob wide = 0"; return false; }
  bool sA = wide_a_side(s), dA = wide_a_side(d);
  const uint64_t H = (uint64_t)s.extents[0], W = (uint64_t)s.extents[1];
  const bool morton = s.lin == LLAMA_MORTON || d.lin == LLAMA_MORTON;
  uint32_t lty = 5, ltx = 5;  // E -> E: 32 x 32
  for (int pass = 0; pass < 3; ++pass) {  // (an AoSoA side whose runs would split blocks is demoted to E)
  lty = 5, ltx = 5;
  if (sA || dA) {
    // 128 records per tile while the images stay <= 64 KB (HEP100 aligned: 61 KB)
    bool same = sA && dA && s.B == d.B && s.L == 1 && d.L == 1 && !d.has_padding();
    for (int k = 0; k < s.K() && same; ++k) same = s.F[k] == d.F[k];
    const uint64_t S = (sA ? s.B / s.L : 0) + (dA && !same ? d.B / d.L : 0);
    uint32_t lt = 7;
    while (lt > 5 && (S << lt) > 64 * 1024) --lt;
    // the E side's storage runs span the tile: 32 records along a row /
    // column side; a Morton tile is 2^a x 2^a or 2^a x 2^(a+1) (contiguous codes)
    const Mapping* e = !sA ? &s : !dA ? &d : nullptr;
    // E -> A staged through shared memory (knob wide_stage, off: measured
    // over the 30 HEP100 E -> A pairs, median 0.46 -> 0.39 -- the scatter out
    // of the staging area into a packed image costs more than the register
    // loads it replaces): 64-record tiles keep image + staging area <= 64 KB
    if (!sA && dA && kn.get(LLAMA_KNOB_WIDE_STAGE, 0) && s.uniform && (s.L >= s.N || s.L % 4 == 0) &&
        (s.lin != LLAMA_ROW_MAJOR || W % 4 == 0) && (s.lin != LLAMA_COL_MAJOR || H % 4 == 0))
      lt = std::min<uint32_t>(lt, 6);
    if (morton || !e) lty = lt / 2, ltx = lt - lt / 2;
    else if (e->lin == LLAMA_ROW_MAJOR) ltx = 5, lty = lt - 5;
    else lty = 5, ltx = lt - 5;
  }
  if (morton) {  // extents equal powers of two: clip the tile (stays square or 1 x 2)
    const uint32_t b = ilog2(H);
    lty = std::min(lty, b);
    ltx = std::min(ltx, b);
  }
  // AoSoA-L image sides: every run of the tile starts at a multiple of L and
  // holds whole blocks
  bool demoted = false;
  for (int X = 0; X < 2; ++X) {
    const Mapping& m = X == 0 ? s : d;
    bool& A = X == 0 ? sA : dA;
    if (!A || m.L == 1) continue;
    const uint64_t run = m.lin == LLAMA_ROW_MAJOR ? 1ull << ltx : m.lin == LLAMA_COL_MAJOR ? 1ull << lty
                                                                                      : 1ull << (lty + ltx);
    bool ok = run % m.L == 0 && kn.get(LLAMA_KNOB_WIDE_AOSOA_IMG, 1);
    // an AoSoA destination next to a plain AoS source image stays element-wise
    // (measured, 1024^2 HEP100: AoS -> AoSoA8 median 0.92x as image -> image
    // moves; AoSoA8 <-> SoA 1.16-1.57x, AoSoA8 -> AoSoA8 1.7x, AoSoA8 -> AoS 1.11x)
    if (X == 1 && sA && s.L == 1 && kn.get(LLAMA_KNOB_WIDE_AOSOA_IMG, 1) < 2) ok = false;
    if (m.lin == LLAMA_ROW_MAJOR) ok = ok && W % m.L == 0;
    if (m.lin == LLAMA_COL_MAJOR) ok = ok && H % m.L == 0;
    if (!ok) A = false, demoted = true;
  }
  if (!demoted) break;
  }
  const uint32_t lt = lty + ltx, n = 1u << lt;
  p->wide.reset(new WideParams);
  WideParams& w = *p->wide;
  std::memset(&w, 0, sizeof(w));
  w.H = H;
  w.W = W;
  w.lty = lty;
  w.ltx = ltx;
  w.K = (uint32_t)s.K();
  w.ntx = ceil_div(W, 1ull << ltx);
  const uint64_t n_tiles = ceil_div(H, 1ull << lty) * w.ntx;
  if (sA && dA) {
    bool same = s.B == d.B && s.L == 1 && d.L == 1 && !d.has_padding();
    for (int k = 0; k < s.K() && same; ++k) same = s.F[k] == d.F[k];
    w.mode = same ? 3 : 2;
  } else {
    w.mode = sA ? 0 : dA ? 1 : 4;
  }
  uint64_t smem = 0;
  for (int X = 0; X < 2; ++X) {
    const Mapping& m = X == 0 ? s : d;
    WideSide& sd = w.side[X];
    sd.lin = (uint32_t)m.lin;
    sd.A = (X == 0 ? sA : dA) ? 1 : 0;
    if (sd.A) {
      const bool image = !(X == 1 && sA && w.mode == 3);  // mode 3 flushes from the source image
      sd.S = (uint32_t)(m.B / m.L);  // bytes per record position of a run (AoSoA: B / L)
      sd.B = (uint32_t)m.B;
      sd.lL = ilog2(m.L);
      sd.blob = m.blob[0];
      sd.base = m.base[0];
      sd.lrun = m.lin == LLAMA_ROW_MAJOR ? ltx : m.lin == LLAMA_COL_MAJOR ? lty : lt;
      sd.chunk = wide_chunk(m, sd.lrun);
      const uint32_t nruns = 1u << (lt - sd.lrun);
      sd.pitch = (uint32_t)(((uint64_t)sd.S << sd.lrun) + sd.chunk - 1) / sd.chunk * sd.chunk;  // (re-chosen below)
      if (image) {
        sd.img = (uint32_t)smem;
        sd.img_bytes = (uint32_t)align16((uint64_t)nruns * sd.pitch);
        smem += sd.img_bytes;
      }
    } else {
      sd.uni = m.uniform ? 1 : 0;
      sd.L = m.L;
      sd.B = m.B;
      sd.lshift = m.L >= m.N ? 63u : (m.L & (m.L - 1)) == 0 ? ilog2(m.L) : kNoShift;
      if (sd.lshift == kNoShift) {  // division by L through a multiplier (k_transpose_wide.cu esplit)
        sd.mshift = ilog2(m.L) + 1;  // ceil(log2 L), L not a power of two
        const unsigned __int128 two64 = (unsigned __int128)1 << 64;
        sd.magic = (uint64_t)(two64 * (((unsigned __int128)1 << sd.mshift) - m.L) / m.L) + 1;
      }
    }
  }
  w.dzero = (dA && d.has_padding()) ? 1 : 0;
  // 4-record groups along the E side (modes 0 / 1, knob wide_group): the
  // group of 4 consecutive storage positions starts at a multiple of 4 and
  // lies in one block, so leaf k's 4 elements are one 4 * s_k-byte range
  auto group_ok = [&](const Mapping& e) {
    bool ok = e.uniform && (e.L >= e.N || e.L % 4 == 0) && lt >= 2;
    if (e.lin == LLAMA_ROW_MAJOR) ok = ok && ltx >= 2 && W % 4 == 0;
    if (e.lin == LLAMA_COL_MAJOR) ok = ok && lty >= 2 && H % 4 == 0;
    return ok;
  };
  // group vectors: leaf k's 4 elements of a group, aligned to min(16, 4 s_k)
  auto group_vec = [&](const Mapping& e, int k) {
    uint64_t a = gcd64(gcd64(16, e.base[k] + e.F[k]), 4ull * e.sizes[k]);
    if (e.L < e.N) a = gcd64(a, e.B);
    return a >= std::min<uint64_t>(16, 4ull * e.sizes[k]);
  };
  if (kn.get(LLAMA_KNOB_WIDE_GROUP, 1)) {
    if (w.mode <= 1) w.grp = group_ok(w.mode == 0 ? d : s) ? 1 : 0;
    if (w.mode == 4) w.grp = group_ok(s) && group_ok(d) ? 1 : 0;
  }
  // image pitches by simulated bank conflicts of warp 0's move accesses
  // (before the images are placed: a pitch changes the image size)
  {
    uint64_t off = 0;
    for (int X = 0; X < 2; ++X) {
      WideSide& sd = w.side[X];
      if (!sd.A || sd.img_bytes == 0) continue;
      const uint32_t nruns = 1u << (lt - sd.lrun);
      // (r2) tensor-map TMA (knob wide_tma): one box op per tile and side
      // (SASS UTMALDG / UTMASTG); the image is the dense box
      const Mapping& m = X == 0 ? s : d;
      if (kn.get(LLAMA_KNOB_WIDE_TMA, 1) && m.lin == LLAMA_MORTON && m.base[0] % 16 == 0 &&
          ((uint64_t)sd.S << lt) % 16 == 0 && ((uint64_t)sd.S << lt) < (1ull << 20)) {
        // a Morton tile is one contiguous run starting at a multiple of n
        // records: one 1-d bulk copy (UBLKCP) per tile and side
        sd.tma = 1;
        sd.pitch = (uint32_t)((uint64_t)sd.S << lt);
        off = (off + 127) & ~127ull;
        sd.img = (uint32_t)off;
        sd.img_bytes = sd.box_bytes = sd.pitch;
        off += align16(sd.img_bytes);
        continue;
      }
      if (kn.get(LLAMA_KNOB_WIDE_TMA, 1) && m.lin != LLAMA_MORTON && m.base[0] % 16 == 0) {
        const uint64_t S = sd.S;
        uint32_t g = 1, e = 0;
        uint64_t inner = 0;  // bytes of the box's innermost row
        if (m.lin == LLAMA_ROW_MAJOR) {
          inner = S << ltx;
          if ((W * S) % 16) inner = 0;
        } else {
          for (uint32_t gg = 1u << lty; gg >= 1; gg >>= 1)
            if ((gg * S) % 16 == 0 && gg * S <= 2048 && H % gg == 0) { g = gg; break; }
          inner = (g * S) % 16 == 0 && g * S <= 2048 && H % g == 0 && (H * S) % 16 == 0 ? g * S : 0;
        }
        if (inner && inner % 16 == 0)
          for (uint32_t ee : {8u, 4u, 2u, 1u})
            if (inner % ee == 0 && inner / ee <= 256) { e = ee; break; }
        if (e) {
          sd.tma = m.lin == LLAMA_ROW_MAJOR ? 2 : 3;
          sd.elsz = e;
          sd.g = g;
          sd.pitch = (uint32_t)(S << sd.lrun);  // dense runs
          off = (off + 127) & ~127ull;          // (the TMA destination / source in shared memory)
          sd.img = (uint32_t)off;
          sd.img_bytes = sd.box_bytes = nruns * sd.pitch;
          off += align16(sd.img_bytes);
          continue;
        }
      }
      const uint32_t ord = w.mode == 1 ? w.side[0].lin : w.side[1].lin;  // the order the lanes run along
      const bool g = w.grp && w.mode <= 1;
      auto lanes = [&](int i) {
        std::vector<uint32_t> v;
        for (uint32_t l = 0; l < 32 && l < (g ? n / 4 : n); ++l) {
          uint32_t r, c;
          h_t_rc(ord, g ? 4 * l + i : l, lty, ltx, r, c);
          v.push_back(h_rc_t(sd.lin, r, c, lty, ltx));
        }
        return v;
      };
      // (r2) a 4-byte chunk allows odd-word pitches: the 4 records of a group
      // sit in runs 4 apart, which a 16-byte multiple pitch folds onto 8 banks
      // (4-way conflicts); take the chunk with the fewest wavefronts, the
      // larger on a tie (fewer cp.async / store instructions)
      uint32_t best_p = 0, best_c = sd.chunk, best_w = ~0u;
      for (uint32_t c : {sd.chunk, 4u}) {
        if (c > sd.chunk) continue;
        const uint32_t pc = wide_pitch((uint64_t)sd.S << sd.lrun, c, nruns, sd.S, sd.lrun, g ? 4 : 1, lanes);
        uint32_t wf = 0;
        for (int i = 0; i < (g ? 4 : 1); ++i) {
          std::vector<uint64_t> o;
          for (uint32_t t : lanes(i)) o.push_back((t >> sd.lrun) * (uint64_t)pc + (t & ((1u << sd.lrun) - 1)) * (uint64_t)sd.S);
          wf += wavefronts(o);
        }
        if (wf < best_w) best_w = wf, best_p = pc, best_c = c;
      }
      if (kn.get(LLAMA_KNOB_WIDE_CHUNK4, 0) == 0) best_p = wide_pitch((uint64_t)sd.S << sd.lrun, sd.chunk, nruns, sd.S,
                                                                     sd.lrun, g ? 4 : 1, lanes), best_c = sd.chunk;
      sd.pitch = best_p;
      sd.chunk = best_c;
      sd.img = (uint32_t)off;
      sd.img_bytes = (uint32_t)align16((uint64_t)nruns * sd.pitch);
      off += sd.img_bytes;
    }
    if (w.mode != 4) smem = off;
  }
  w.bar = (uint32_t)((smem + 7) & ~7ull);  // the TMA mbarrier
  smem = w.bar + 8;
  // leaf positions in class order: size, then unit, then the group vector flag, descending
  struct LeafInfo { int k; uint32_t size, unit; };
  std::vector<LeafInfo> li;
  for (int k = 0; k < s.K(); ++k) {
    uint32_t u = s.sizes[k];
    for (int X = 0; X < 2; ++X) {
      const Mapping& m = X == 0 ? s : d;
      const WideSide& sd = w.side[X];
      const uint32_t a = sd.A ? (uint32_t)gcd64(gcd64(16, sd.pitch), gcd64(sd.B, m.F[k])) : wide_e_align(m, k);
      u = std::min(u, a);
    }
    if (w.grp && w.mode <= 1 && group_vec(w.mode == 0 ? d : s, k)) u |= 256;  // (f64: two 16-byte pieces)
    li.push_back({k, s.sizes[k], u});
  }
  std::stable_sort(li.begin(), li.end(), [](const LeafInfo& a, const LeafInfo& b) {
    return a.size != b.size ? a.size > b.size : a.unit > b.unit;  // (unit | 256 for vector groups)
  });
  for (size_t j = 0; j < li.size(); ++j) {
    const int k = li[j].k;
    WideLeaf& l = w.leaf[j];
    l.size = (uint16_t)li[j].size;
    l.unit = (uint16_t)li[j].unit;  // the class keeps the vector flag; leaves take the scalar unit
    const uint16_t cls_unit = l.unit;
    l.unit &= 0xFF;
    l.soff = (uint32_t)s.F[k];
    l.doff = (uint32_t)d.F[k];
    w.order[j] = (uint16_t)k;
    if (w.grp && w.mode == 4) l.vec = (group_vec(s, k) ? 1u : 0u) | (group_vec(d, k) ? 2u : 0u);
    w.sl[j] = s.dev_leaf(k);
    w.dl[j] = d.dev_leaf(k);
    if (w.n_cls == 0 || w.cls[w.n_cls - 1].size != l.size || w.cls[w.n_cls - 1].unit != cls_unit) {
      if (w.n_cls == 16) { *why = "too many leaf classes"; return false; }
      w.cls[w.n_cls++] = WideClass{(uint16_t)j, (uint16_t)j, l.size, cls_unit};
    }
    w.cls[w.n_cls - 1].j1 = (uint16_t)(j + 1);
  }
  if (w.mode == 4) {  // leaf batches of element buffers (n + n / 32 elements each) within 40 KB
    const uint64_t budget = 40 * 1024;
    w.buf = (uint32_t)align16(smem);
    uint64_t used = 0;
    w.nbatch = 0;
    w.bstart[0] = 0;
    for (size_t j = 0; j < li.size(); ++j) {
      const uint64_t bytes = align16((uint64_t)(w.grp ? n : n + n / 32) * li[j].size);  // (grp: swizzled, unpadded)
      if (used && used + bytes > budget) {
        w.bstart[++w.nbatch] = (uint16_t)j;
        used = 0;
      }
      w.leaf[j].buf = (uint32_t)used;
      used += bytes;
      smem = std::max<uint64_t>(smem, w.buf + used);
    }
    w.bstart[++w.nbatch] = (uint16_t)li.size();
    if (lt != 10) { *why = "E -> E tiles are 32 x 32 records"; return false; }  // 4 records per thread
  }
  w.async = w.mode == 1 && w.grp && !kn.get(LLAMA_KNOB_WIDE_STAGE, 0) && kn.get(LLAMA_KNOB_WIDE_ASYNC, 0) ? 1 : 0;  // (measured 1-5% slower: off)
  if (w.mode == 1 && w.grp && kn.get(LLAMA_KNOB_WIDE_STAGE, 0)) {  // staging area: leaf j's n elements in E order
    w.stage = 1;
    w.buf = (uint32_t)align16(smem);
    uint64_t off = 0;
    for (size_t j = 0; j < li.size(); ++j) {
      w.leaf[j].buf = (uint32_t)off;
      off += align16((uint64_t)n * li[j].size);
    }
    smem = w.buf + off;
  }
  // tile order (knob wide_torder: 0 x fastest, 1 y fastest, 2 auto): auto runs
  // the tiles along a column-major E side's storage order, so consecutive
  // tiles continue the same columns (contiguous DRAM streams on that side)
  {
    const int64_t to = kn.get(LLAMA_KNOB_WIDE_TORDER, 2);
    const Mapping& e = w.mode == 0 ? d : s;  // (mode 4: the source)
    w.yfast = to == 1 || (to == 2 && (w.mode == 0 || w.mode == 1 || w.mode == 4) && e.lin == LLAMA_COL_MAJOR);
    w.nty = ceil_div(H, 1ull << lty);
  }
  w.n_items = n_tiles * (w.mode == 4 ? w.nbatch : 1);
  if (w.n_items >= (1ull << 31)) { *why = "more than 2^31 tiles"; return false; }  // 32-bit tile loop
  if (w.mode == 3) w.u3 = (uint32_t)gcd64(gcd64(16, w.side[0].S), gcd64(w.side[0].pitch, w.side[1].chunk));
  if (smem > 200 * 1024) { *why = "tile images exceed shared memory"; return false; }
  w.smem = (uint32_t)align16(std::max<uint64_t>(smem, 16));
  p->path = LLAMA_PATH_TRANSPOSE;
  p->smem_bytes = (int)w.smem;
  // E destinations with padding (aligned SoA SB gaps, aligned / tail AoSoA
  // lanes) are zero-filled first; A destinations zero their images
  p->naive_zero_fill = !dA && d.has_padding();
  if (p->naive_zero_fill) p->fill.reset(new FillParams(make_fill(d, 0)));
  return true;
}

bool plan_wide(const Mapping& s, const Mapping& d, const Knobs& kn, Plan* p, std::string* why) {
  if (plan_wide_impl(s, d, kn, p, why)) return true;
  p->wide.reset();
  return false;
}

// Every leaf one contiguous run of N * s_k bytes in the mapping (SoA single /
// multi blob, a part of one block), starting 16-byte aligned.
static bool single_runs(const Mapping& m) {
  for (int k = 0; k < m.K(); ++k) {
    const bool run = m.Lk[k] >= m.N || m.Bk[k] == m.Lk[k] * m.sizes[k];
    if (!run || (m.base[k] + m.F[k]) % 16) return false;
  }
  return true;
}

// Different layouts whose leaves are single runs on both sides (SoA SB <-> MB):
// one bulk-copy range per leaf (each leaf's array moves as it is).
static bool plan_segments(const Mapping& s, const Mapping& d, const Knobs& kn, Plan* p, std::string* why) {
  if (!single_runs(s) || !single_runs(d)) { *why = "leaves are not single contiguous runs"; return false; }
  if (d.has_padding()) { *why = "layout has padding (must be written as 0)"; return false; }
  if (s.K() > kMaxBlobs) { *why = "too many leaves"; return false; }
  const uint64_t ch = kn.get(LLAMA_KNOB_BULK_CHUNK, 65536) & ~15ull;
  const uint32_t ns = (uint32_t)std::min<uint64_t>(8, std::max<uint64_t>(2, kn.get(LLAMA_KNOB_BULK_STAGES, 3)));
  if (ch < 16 || 128 + (uint64_t)ns * ch > 227ull * 1024) {
    *why = "bulk_chunk x bulk_stages exceed 227 KB of shared memory";
    return false;
  }
  p->path = LLAMA_PATH_BLOBCOPY;
  p->bulkcopy.reset(new BulkCopyParams);
  BulkCopyParams& b = *p->bulkcopy;
  std::memset(&b, 0, sizeof(b));
  b.seg = 1;
  b.nb = s.K();
  b.CH = (uint32_t)ch;
  b.NS = ns;
  for (int k = 0; k < s.K(); ++k) {
    b.bytes[k] = s.N * s.sizes[k];
    b.sblob[k] = s.blob[k];
    b.soff[k] = s.base[k] + s.F[k];
    b.dblob[k] = d.blob[k];
    b.doff[k] = d.base[k] + d.F[k];
    b.cstart[k + 1] = b.cstart[k] + ceil_div(b.bytes[k], b.CH);
  }
  return true;
}

bool plan_blobcopy(const Mapping& s, const Mapping& d, const Knobs& kn, Plan* p, std::string* why) {
  if (!same_layout(s, d)) return plan_segments(s, d, kn, p, why);
  if (d.has_padding()) { *why = "layout has padding (must be written as 0)"; return false; }
  p->path = LLAMA_PATH_BLOBCOPY;
  if (kn.get(LLAMA_KNOB_BLOBCOPY_LSU, 0)) {  // thread (LDG/STG) variant, for comparison
    p->blobcopy.reset(new BlobCopyParams);
    BlobCopyParams& b = *p->blobcopy;
    std::memset(&b, 0, sizeof(b));
    b.nb = d.nblobs();
    for (int j = 0; j < b.nb; ++j) {
      b.bytes[j] = d.blob_sizes[j];
      b.vstart[j + 1] = b.vstart[j] + ceil_div(d.blob_sizes[j], 16);
    }
    return true;
  }
  p->bulkcopy.reset(new BulkCopyParams);
  BulkCopyParams& b = *p->bulkcopy;
  std::memset(&b, 0, sizeof(b));
  b.nb = d.nblobs();
  const uint64_t ch = kn.get(LLAMA_KNOB_BULK_CHUNK, 65536) & ~15ull;  // 64 KB x 3 stages: measured best on B200
  b.NS = (uint32_t)std::min<uint64_t>(8, std::max<uint64_t>(2, kn.get(LLAMA_KNOB_BULK_STAGES, 3)));
  b.CH = (uint32_t)std::min<uint64_t>(ch, 1u << 30);
  // the ring (bulk_chunk x bulk_stages) must fit one CTA's shared memory
  if (ch < 16 || 128 + (uint64_t)b.NS * ch > 227ull * 1024) {
    *why = "bulk_chunk x bulk_stages exceed 227 KB of shared memory";
    p->bulkcopy.reset();
    return false;
  }
  for (int j = 0; j < b.nb; ++j) {
    b.bytes[j] = d.blob_sizes[j];
    b.cstart[j + 1] = b.cstart[j] + ceil_div(d.blob_sizes[j], b.CH);
  }
  return true;
}

bool plan_run(const Mapping& s, const Mapping& d, Plan* p, std::string* why) {
  if (d.has_padding()) { *why = "destination has padding"; return false; }
  const Mapping* side[2] = {&s, &d};
  for (int k = 0; k < s.K(); ++k) {
    const uint64_t sz = s.sizes[k];
    // records per common run ("min(N,M)"; gcd for lane counts that do
    // not divide each other); a single block counts as L = N
    const uint64_t n1 = std::max<uint64_t>(s.N, 1);
    const uint64_t g = gcd64(std::min(s.Lk[k], n1), std::min(d.Lk[k], n1));
    const bool single_run = g >= s.N;    // the whole leaf is one run on both sides
    if (!single_run && (g * sz) % 16 != 0) { *why = "common runs shorter than 16 B"; return false; }
    for (int X = 0; X < 2; ++X) {
      const Mapping& m = *side[X];
      if ((m.base[k] + m.F[k]) % 16 != 0 || (!single_run && (m.base[k] % 16 || m.F[k] % 16))) {
        *why = "run starts not 16-B aligned";
        return false;
      }
      if (!single_run && m.N > m.Lk[k] && m.Bk[k] % 16 != 0) { *why = "block stride not 16-B aligned"; return false; }
    }
  }
  p->path = LLAMA_PATH_RUN;
  p->run.reset(new RunParams);
  RunParams& r = *p->run;
  std::memset(&r, 0, sizeof(r));
  r.N = s.N;
  r.K = s.K();
  // chunk = C records, a multiple of 16 (every leaf's chunk part is whole
  // 16-byte vectors) sized to ~32 KB of source bytes
  uint64_t S = 0;
  for (int k = 0; k < s.K(); ++k) S += s.sizes[k];
  uint64_t C = std::max<uint64_t>(16, (32768 / S) / 16 * 16);
  r.C = C;
  r.n_chunks = ceil_div(s.N, C);
  r.cvstart[0] = 0;
  for (int k = 0; k < s.K(); ++k) {
    r.sl[k] = s.dev_leaf(k);
    r.dl[k] = d.dev_leaf(k);
    r.cvstart[k + 1] = r.cvstart[k] + (uint32_t)(C * s.sizes[k] / 16);
  }
  r.chunk_vecs = r.cvstart[s.K()];
  return true;
}

// AoS <-> SoA with many leaves (measured on HEP100): the AoS side
// through a TMA ring, the SoA side element-wise with coalesced accesses.
bool plan_direct(const Mapping& s, const Mapping& d, int tile_records, const Knobs& kn, Plan* p, std::string* why) {
  const uint64_t mode = kn.get(LLAMA_KNOB_DIRECT, 1);  // 0: off; 2: any leaf count (tests)
  if (mode == 0) { *why = "disabled"; return false; }
  if (!s.uniform || !d.uniform) { *why = "split"; return false; }
  const bool a2s = s.kind == LLAMA_AOS && d.soa();
  const bool s2a = s.soa() && d.kind == LLAMA_AOS;
  if (!a2s && !s2a) { *why = "not AoS <-> SoA"; return false; }
  if (s.K() <= 16 && mode != 2) { *why = "few leaves: the tile permute"; return false; }
  const Mapping& A = a2s ? s : d;
  const Mapping& So = a2s ? d : s;
  const uint64_t S = A.B;
  if (S == 0 || A.L != 1) { *why = "AoS stride"; return false; }
  // measured on HEP100: AoS -> SoA wins for packed and aligned records (2.8 ->
  // 5.2 TB/s packed; misaligned leaves are funnel-shifted out of aligned
  // words); SoA -> AoS for naturally aligned records, and for packed ones
  // only with the staged misaligned classes (2.92 -> 3.18 TB/s; scattered from
  // registers in 1-2 byte pieces they lost: 2.9 -> 2.0)
  // (with a record stride that is a multiple of 4 the misaligned 4- / 8-byte
  // leaves are staged by cp.async and scattered in compile-time pieces)
  const bool staging = s2a && S % 4 == 0 && kn.get(LLAMA_KNOB_DIRECT_ASYNC, 1) && kn.get(LLAMA_KNOB_DIRECT_PHASE, 1) &&
                       kn.get(LLAMA_KNOB_DIRECT_STAGING, 1);
  if (mode != 2 && s2a && !staging)
    for (int k = 0; k < A.K(); ++k)
      if (A.F[k] % A.sizes[k] || S % A.sizes[k]) { *why = "packed AoS: the tile permute"; return false; }
  // T = 64 records per tile (two per lane); stages measured on HEP100: AoS ->
  // SoA 3 (aligned 5.25 -> 5.83 TB/s over 2), SoA -> AoS 2 (3.92 vs 2.88 at 3)
  const uint64_t T = 64;
  if (tile_records > 0 && tile_records != 64) { *why = "the direct variant uses 64-record tiles"; return false; }
  const uint64_t stage = align16(T * S);
  const uint64_t ns = std::min<uint64_t>(8, std::max<uint64_t>(2, kn.get(LLAMA_KNOB_DIRECT_STAGES, a2s ? 3 : 2)));
  if (ns * stage > 200 * 1024) { *why = "record too wide"; return false; }
  p->direct.reset(new DirectParams);
  DirectParams& dp = *p->direct;
  std::memset(&dp, 0, sizeof(dp));
  dp.N = s.N;
  dp.T = (uint32_t)T;
  dp.K = (uint32_t)s.K();
  dp.S = (uint32_t)S;
  dp.a2s = a2s ? 1 : 0;
  dp.ns = (uint32_t)ns;
  dp.stage = (uint32_t)stage;
  dp.n_tiles = ceil_div(s.N, T);
  // an even record stride in words puts one leaf of 32 records on few banks
  dp.mix = ((S / 4) % 2 == 0 && S % 4 == 0 && kn.get(LLAMA_KNOB_DIRECT_MIX, 1)) ? 1 : 0;
  // SoA -> AoS: aligned 4- / 8-byte elements land in the image by cp.async
  dp.async = (!a2s && kn.get(LLAMA_KNOB_DIRECT_ASYNC, 1)) ? 1 : 0;
  dp.abase = A.base[0];
  dp.ablob = A.blob[0];
  auto lb = [](uint64_t x) { return x ? (x & (~x + 1)) : 16ull; };
  for (int k = 0; k < s.K(); ++k) {
    DirectLeaf& l = dp.leaf[k];
    l.gbase = So.base[k] + So.F[k];
    l.blob = So.blob[k];
    l.F = (uint32_t)A.F[k];
    l.size = (uint16_t)s.sizes[k];
    l.a_img = (uint8_t)std::min<uint64_t>(8, std::min(lb(S), lb(A.F[k])));
    l.a_glob = (uint8_t)std::min<uint64_t>(8, std::min<uint64_t>(lb(l.gbase), 16));
  }
  // leaf classes: (size, image aligned, global aligned), leaves grouped
  {
    std::vector<int> idx(s.K());
    for (int k = 0; k < s.K(); ++k) idx[k] = k;
    auto kind = [&](int k) {
      const DirectLeaf& l = dp.leaf[k];
      uint32_t kd = (uint32_t)l.size | (l.a_img >= l.size ? 16u : 0u) | (l.a_glob >= l.size ? 32u : 0u);
      // record stride a multiple of 4: a misaligned leaf sits at the same
      // word phase F % 4 in every record (compile-time funnel shifts / pieces)
      if (S % 4 == 0 && l.a_img < l.size && l.size >= 2 && kn.get(LLAMA_KNOB_DIRECT_PHASE, 1))
        kd |= 64u | ((l.F & 3u) << 7);
      // SoA -> AoS, image-aligned 1- / 2-byte leaf with 16-byte aligned SoA
      // runs: staged as 16-byte cp.async chunks (full tiles)
      // (measured: chunk-staging the aligned 4- / 8-byte classes too, instead
      // of their element cp.asyncs into the image, lost 2-33%)
      if (staging && l.size <= 2 && l.a_img >= l.size && l.gbase % 16 == 0 && (T * l.size) % 16 == 0 &&
          kn.get(LLAMA_KNOB_DIRECT_CHUNKS, 1))
        kd |= 512u;
      return kd;
    };
    // SoA -> AoS with cp.async: classes ordered by how the kernel moves them
    // (k_permute_direct.cu direct_tile): 0 chunk-staged, 1 staged, 2 cp.async
    // into the image, 3 registers; each pass walks its own class range
    const bool use_async = !a2s && kn.get(LLAMA_KNOB_DIRECT_ASYNC, 1);
    auto cat = [&](int k) -> uint32_t {
      const uint32_t kd = kind(k), z = kd & 15;
      if (!use_async) return 3;
      if (kd & 512) return 0;
      if (staging && (kd & 96) == 96 && (z == 4 || z == 8)) return 1;
      if ((kd & 48) == 48 && (z == 4 || z == 8)) return 2;
      return 3;
    };
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) {
      return cat(x) != cat(y) ? cat(x) < cat(y) : kind(x) < kind(y);
    });
    for (int i = 0; i < s.K(); ++i) {
      dp.order[i] = (uint16_t)idx[i];
      if (i == 0 || kind(idx[i]) != kind(idx[i - 1])) {
        if (dp.n_cls >= 16) { *why = "too many leaf classes"; return false; }
        dp.cls[dp.n_cls++] = DirectClass{(uint16_t)i, (uint16_t)(i + 1), kind(idx[i])};
      } else {
        dp.cls[dp.n_cls - 1].k1 = (uint16_t)(i + 1);
      }
    }
    for (uint32_t c = 0; c < 3; ++c) {
      dp.cat_end[c] = 0;
      for (uint32_t ci = 0; ci < dp.n_cls; ++ci)
        if (cat(idx[dp.cls[ci].k0]) <= c) dp.cat_end[c] = ci + 1;
    }
  }
  if (staging) {  // staging area of the misaligned (phase) 4- / 8-byte classes, T elements per leaf
    uint64_t off = 0;
    for (uint32_t ci = 0; ci < dp.n_cls; ++ci) {
      const DirectClass& c = dp.cls[ci];
      const uint32_t z = c.kind & 15;
      if (!(c.kind & 512) && ((c.kind & 96) != 96 || (z != 4 && z != 8))) continue;
      for (uint32_t i = c.k0; i < c.k1; ++i) {
        dp.leaf[dp.order[i]].stg = (uint32_t)off;
        off += align16(T * z);
      }
    }
    dp.stg_bytes = (uint32_t)off;
  }
  if (a2s && d.has_padding()) {  // aligned SoA SB: the gaps between sub-arrays
    if (d.kind != LLAMA_SOA_SINGLE_BLOB) { *why = "padded destination"; return false; }
    uint64_t end = 0;
    for (int k = 0; k < d.K(); ++k) {
      if (d.base[k] > end) {
        dp.gap_blob[dp.n_gaps] = d.blob[k];
        dp.gap_off[dp.n_gaps] = end;
        dp.gap_len[dp.n_gaps] = (uint32_t)(d.base[k] - end);
        ++dp.n_gaps;
      }
      end = d.base[k] + d.N * d.sizes[k];
    }
  }
  p->path = LLAMA_PATH_PERMUTE;
  p->smem_bytes = (int)(128 + ns * stage + 16 + 16 * s.K() + dp.stg_bytes);
  return true;
}

bool plan_permute(const Mapping& s, const Mapping& d, int tile_records, const Knobs& kn, Plan* p, std::string* why) {
  // every part must spread its records over its blobs (not One)
  for (const Mapping* m : {&s, &d}) {
    if ((int)m->parts.size() > kMaxParts) { *why = "too many split parts"; return false; }
    for (const Part& q : m->parts)
      if (q.kind == LLAMA_ONE) { *why = "one mapping"; return false; }
  }
  const Mapping* side[2] = {&s, &d};
  std::vector<bool> soa_like[2];  // per part
  uint64_t Tmult = 32;
  std::vector<uint64_t> Tdiv;
  uint64_t rec_img[2] = {0, 0};
  for (int X = 0; X < 2; ++X) {
    const Mapping& m = *side[X];
    for (const Part& q : m.parts) {
      bool sl;
      if (q.soa()) {
        sl = true;
      } else if (q.B <= kAosLikeMaxBlock) {
        sl = false;
        Tmult = lcm64(Tmult, q.L);
      } else {
        sl = true;  // huge AoSoA blocks: a tile stays inside one block
        Tdiv.push_back(q.L);
      }
      soa_like[X].push_back(sl);
      uint64_t sum = 0;
      for (int k : q.leaves) sum += m.sizes[k];
      rec_img[X] += sl ? sum : q.record_bytes;
    }
  }
  if (Tmult > 8192) { *why = "lane counts need tiles above 8192 records"; return false; }
  const uint64_t R = d.E;  // records the destination blobs cover
  uint64_t T;
  if (tile_records > 0) {
    T = (uint64_t)tile_records;
    if (T % Tmult || (T > 256 && T % 256)) {
      *why = "tile_records must be a multiple of 32 and of every AoS-like lane count, and <= 256 or a multiple of 256";
      return false;
    }
  } else {
    // measured on B200 with the warp-specialised kernel (DESIGN.md "Tile
    // size"): small records (<= 128 B src + dst) -> 64 KB tiles (T = 1024
    // for Particle7) with a deep ring in one CTA per SM; wide records (whose
    // permute costs more per tile) -> the largest tile that still leaves two
    // CTAs per SM (budget below)
    const uint64_t per = rec_img[0] + rec_img[1];
    const uint64_t def_tile = per <= 128 ? 64 * 1024 : 48 * 1024;
    uint64_t c = std::max<uint64_t>(1, kn.get(LLAMA_KNOB_TILE_BYTES, def_tile) / (per * Tmult));
    const uint64_t cmax = std::max<uint64_t>(1, ceil_div(R, Tmult));
    c = std::min(c, cmax);
    T = 0;
    for (; c >= 1; --c) {
      const uint64_t t = c * Tmult;
      // <= 256 records, or 512 / 1024 (whole passes of 256 threads, R = 2 / 4
      // records per thread; measured: other multiples and > 116 KB of shared
      // memory per CTA run markedly slower on B200)
      bool ok = t <= 256 || t == 512 || t == 1024;
      for (auto L : Tdiv) ok = ok && (L % t == 0);
      // wide records: the tile must leave room for two CTAs per SM with two
      // source stages (measured: one CTA per SM starves the permute of warps)
      const uint64_t est = 256 + 64ull * s.K() + 2 * (t * rec_img[0] + 16ull * s.K()) + 2 * (t * rec_img[1] + 16ull * s.K());
      if (per > 128 && c > 1 && est > kn.get(LLAMA_KNOB_SMEM_BUDGET, 112 * 1000)) ok = false;
      if (ok) { T = t; break; }
    }
    if (!T) { *why = "no tile size divides the AoSoA lane count"; return false; }
  }
  for (auto L : Tdiv)
    if (L % T) { *why = "tile must divide the lane count of a large-block AoSoA side"; return false; }

  p->perm.reset(new PermParams);
  PermParams& pp = *p->perm;
  std::memset(&pp, 0, sizeof(pp));
  pp.N = s.N;
  pp.T = (uint32_t)T;
  pp.K = (uint32_t)s.K();
  pp.n_tiles = ceil_div(R, T);
  bool tma = true;
  std::vector<uint32_t> imgF[2] = {std::vector<uint32_t>(s.K()), std::vector<uint32_t>(s.K())};
  std::vector<int> part_of[2] = {std::vector<int>(s.K()), std::vector<int>(s.K())};
  std::vector<int> geo_of[2] = {std::vector<int>(s.K()), std::vector<int>(s.K())};
  uint64_t full_src = 0;  // TMA bytes of a full tile's source segments (16-B multiples: T % 32 == 0)
  for (int X = 0; X < 2; ++X) {
    const Mapping& m = *side[X];
    PermSide& ps = pp.side[X];
    ps.E = m.E;
    ps.n_parts = (uint32_t)m.parts.size();
    ps.linear = 1;
    for (int k = 0; k < m.K(); ++k) pp.leaf[X][k] = m.dev_leaf(k);
    uint64_t off = 0;  // the side image: its parts' images one after another
    uint32_t ns = 0;
    for (size_t j = 0; j < m.parts.size(); ++j) {
      const Part& q = m.parts[j];
      PermPart& pq = pp.part[X][j];
      pq.g.L = q.L;
      pq.g.B = q.B;
      pq.g.lshift = q.soa() ? 63u : (q.L & (q.L - 1)) == 0 ? (uint32_t)__builtin_ctzll(q.L) : kNoShift;
      pq.E = q.E;
      pq.soa_like = soa_like[X][j] ? 1 : 0;
      if (soa_like[X][j] && !q.soa()) ps.linear = 0;  // large AoSoA blocks: segment starts jump per block
      // the part's image geometry; parts with equal geometry share one entry
      PermGeo g{};
      if (!soa_like[X][j]) {
        g.Limg = (uint32_t)q.L;
        g.limg_shift = (q.L & (q.L - 1)) == 0 ? (uint32_t)__builtin_ctzll(q.L) : kNoShift;
        g.Bimg = (uint32_t)q.B;
      } else {
        g.Limg = (uint32_t)T;
        g.limg_shift = 31;  // r < T: one image block
        g.Bimg = 0;
      }
      uint32_t gi = 0;
      while (gi < ps.n_geo && !(pp.geo[X][gi].Limg == g.Limg && pp.geo[X][gi].Bimg == g.Bimg)) ++gi;
      if (gi == ps.n_geo) pp.geo[X][ps.n_geo++] = g;
      for (int k : q.leaves) {
        part_of[X][k] = (int)j;
        geo_of[X][k] = (int)gi;
      }
      off = align16(off);
      if (!soa_like[X][j]) {
        const uint64_t img = T / q.L * q.B;
        for (int k : q.leaves) imgF[X][k] = (uint32_t)(off + m.F[k]);
        pp.seg[X][ns++] = PermSeg{(uint16_t)j, (uint16_t)q.leaves[0], (uint32_t)off};
        if (m.base[q.leaves[0]] % 16 || img % 16) tma = false;
        if (X == 0) full_src += img;
        off += img;
      } else {
        for (int k : q.leaves) {
          off = align16(off);
          imgF[X][k] = (uint32_t)off;
          pp.seg[X][ns++] = PermSeg{(uint16_t)j, (uint16_t)k, (uint32_t)off};
          off += T * m.sizes[k];
          if (m.base[k] % 16) tma = false;
          if (!q.soa() && (m.F[k] % 16 || q.B % 16)) tma = false;
          if (X == 0) full_src += T * m.sizes[k];
        }
      }
    }
    ps.n_segs = ns;
    ps.img_bytes = (uint32_t)align16(off);
  }
  if (kn.get(LLAMA_KNOB_NO_TMA, 0)) tma = false;
  pp.tma = tma ? 1 : 0;
  pp.src_tile_tma = (uint32_t)full_src;
  pp.src_stage = (uint32_t)align16(pp.side[0].img_bytes);
  pp.dst_stage = (uint32_t)align16(pp.side[1].img_bytes);
  // per-record move table: leaf k moves in units of the widest power of two
  // that divides its size and both image offsets for every record; classes
  // by (src geometry, dst geometry, unit, leaf size): within a class the
  // record-dependent part of an image offset is the same for every move, so
  // the kernel hoists it, and recomputes it only when the geometries change
  std::vector<Move> mv[kMaxParts][kMaxParts][4][4];  // [src geo][dst geo][unit][size]
  auto lg = [](uint64_t v) { return v == 8 ? 0 : v == 4 ? 1 : v == 2 ? 2 : 3; };
  for (int k = 0; k < s.K(); ++k) {
    uint64_t unit = std::min<uint64_t>(8, s.sizes[k]);
    for (int X = 0; X < 2; ++X) {
      const PermGeo& pq = pp.geo[X][geo_of[X][k]];
      uint64_t a = std::min<uint64_t>(16, lowbit(imgF[X][k]));
      if (pq.Limg > 1) a = std::min<uint64_t>(a, lowbit(s.sizes[k]));
      if (T / pq.Limg > 1) a = std::min<uint64_t>(a, lowbit(pq.Bimg));
      unit = std::min(unit, a);
    }
    for (uint64_t j = 0; j < s.sizes[k] / unit; ++j) {
      Move m;
      m.soff = (uint32_t)(imgF[0][k] + j * unit);
      m.doff = (uint32_t)(imgF[1][k] + j * unit);
      m.size = (uint16_t)s.sizes[k];
      m.unit = (uint8_t)unit;
      m.pad_ = 0;
      mv[geo_of[0][k]][geo_of[1][k]][lg(unit)][lg(s.sizes[k])].push_back(m);
    }
  }
  uint32_t nm = 0;
  pp.n_classes = 0;
  for (int a = 0; a < kMaxParts; ++a)
    for (int b = 0; b < kMaxParts; ++b)
      for (int c = 0; c < 4; ++c)
        for (int z = 0; z < 4; ++z) {
          if (mv[a][b][c][z].empty()) continue;
          if (pp.n_classes >= (uint32_t)kMaxClasses) { *why = "too many move classes"; return false; }
          MoveClass& mc = pp.classes[pp.n_classes++];
          mc.m0 = nm;
          for (auto& m : mv[a][b][c][z]) {
            if (nm >= (uint32_t)kMaxMoves) { *why = "move table too long"; return false; }
            pp.moves[nm++] = m;
          }
          mc.m1 = nm;
          mc.unit = (uint16_t)(8u >> c);
          mc.size = (uint16_t)(8u >> z);
          mc.sp = (uint16_t)a;
          mc.dp = (uint16_t)b;
        }
  // AoS <-> AoS word mode for wide records (both sides plain AoS, strides
  // multiples of 4, >= 64 destination words per record): each destination
  // word is built from a <= 12-byte source window; lanes own words, so both
  // images are read/written contiguously (no bank conflicts at any stride).
  pp.n_wmoves = 0;
  if (s.parts.size() == 1 && d.parts.size() == 1 && !soa_like[0][0] && !soa_like[1][0] && s.L == 1 &&
      d.L == 1 && s.B % 4 == 0 && d.B % 4 == 0 &&
      kn.get(LLAMA_KNOB_WORD_MODE, 1)) {
    std::vector<int64_t> src_of(d.B, -1);
    for (int k = 0; k < s.K(); ++k)
      for (uint32_t b = 0; b < s.sizes[k]; ++b) src_of[d.F[k] + b] = (int64_t)(s.F[k] + b);
    std::vector<WordMove> wm;
    bool ok = true;
    for (uint64_t w = 0; w < d.B / 4 && ok; ++w) {
      int64_t lo = -1;
      for (int b = 0; b < 4; ++b)
        if (src_of[4 * w + b] >= 0 && (lo < 0 || src_of[4 * w + b] < lo)) lo = src_of[4 * w + b];
      if (lo < 0) continue;  // all padding: the zeroed image already holds it
      const int64_t ws = lo & ~3ll;
      uint32_t sel1 = 0, sel2 = 0, mask = 0;
      for (int b = 0; b < 4; ++b) {
        const int64_t q = src_of[4 * w + b];
        const int64_t idx = q < 0 ? 0 : q - ws;
        if (idx > 11) { ok = false; break; }
        if (q >= 0) mask |= 0xFFu << (8 * b);
        sel1 |= (uint32_t)(idx < 8 ? idx : 0) << (4 * b);
        sel2 |= (uint32_t)(idx < 8 ? b : 4 + (idx - 8)) << (4 * b);
      }
      wm.push_back(WordMove{(uint16_t)(4 * w), (uint16_t)ws, (uint16_t)sel1, (uint16_t)sel2, mask});
    }
    if (ok && wm.size() >= 64 && wm.size() <= (size_t)kMaxWordMoves && d.B < 65536 && s.B < 65536) {
      pp.n_wmoves = (uint32_t)wm.size();
      for (size_t j = 0; j < wm.size(); ++j) pp.wmoves[j] = wm[j];
    }
  }
  // SSeg tables (24 B each, padded) + the word-move table copy
  pp.tab_bytes = (uint32_t)(align16(2ull * 32 * s.K()) + align16(sizeof(WordMove) * pp.n_wmoves));
  if (pp.n_wmoves) pp.src_stage += 16;  // word windows may read up to 8 B past a tile's last record
  pp.nd = 2;
  uint64_t smem = 0;
  const uint64_t per_rec = rec_img[0] + rec_img[1];
  const uint64_t budget = kn.get(LLAMA_KNOB_SMEM_BUDGET, per_rec <= 128 ? 230 * 1000 : 112 * 1000);
  // small records: a deep (4-stage) ring; wide records: 2 stages, so more CTAs fit per SM
  const uint32_t ns_max =
      (uint32_t)std::min<uint64_t>(4, std::max<uint64_t>(2, kn.get(LLAMA_KNOB_STAGES, per_rec <= 128 ? 4 : 2)));
  for (uint32_t ns = ns_max; ns >= 2; --ns) {
    smem = kBarBytes + pp.tab_bytes + (uint64_t)ns * pp.src_stage + 2ull * pp.dst_stage;
    pp.ns = ns;
    // measured on B200: one CTA with 116-160 KB of shared memory runs far
    // slower than both 108 KB and 172 KB (C4: 3.5 vs 6.0 TB/s); skip the window
    const bool window = smem > 116 * 1024 && smem < 160 * 1024 && !kn.given(LLAMA_KNOB_STAGES);
    if (smem <= budget && !(window && ns > 2)) break;
  }
  if (smem > 227 * 1024) { *why = "tile images exceed shared memory"; return false; }
  pp.order = (uint32_t)kn.get(LLAMA_KNOB_WS_ORDER, 2);
  // a third destination buffer keeps one tile's store in flight while the
  // consumers fill the next (warp-specialised kernel only; measured on B200:
  // +2-5% for small records, C2 6.44 -> 6.57 TB/s; slower for wide records
  // with two CTAs per SM, and never into the 116-160 KB window above)
  const uint64_t nd_req =
      std::min<uint64_t>(4, std::max<uint64_t>(2, kn.get(LLAMA_KNOB_DST_BUFS, per_rec <= 128 ? 3 : 2)));
  while (pp.tma && pp.nd < nd_req && smem + pp.dst_stage <= std::min<uint64_t>(budget, 227 * 1024) &&
         !(smem + pp.dst_stage > 116 * 1024 && smem + pp.dst_stage < 160 * 1024)) {
    smem += pp.dst_stage;
    ++pp.nd;
  }
  pp.n_moves = nm;

  // destination padding no tile segment covers: the gaps between aligned
  // SoA single-blob sub-arrays (reading #9); blocked SoA-like parts with
  // padding (tail block, aligned records) are left to the naive path
  for (size_t j = 0; j < d.parts.size(); ++j) {
    const Part& q = d.parts[j];
    if (!soa_like[1][j] || q.kind == LLAMA_SOA_MULTI_BLOB) continue;
    if (q.kind != LLAMA_SOA_SINGLE_BLOB) {
      uint64_t sum = 0;
      for (int k : q.leaves) sum += d.sizes[k];
      if (q.E != d.N || q.record_bytes != sum) { *why = "padded large-block destination"; return false; }
      continue;
    }
    uint64_t end = 0;
    for (int k : q.leaves) {
      if (d.base[k] > end) {
        pp.gap_blob[pp.n_gaps] = d.blob[k];
        pp.gap_off[pp.n_gaps] = end;
        pp.gap_len[pp.n_gaps] = (uint32_t)(d.base[k] - end);
        ++pp.n_gaps;
      }
      end = d.base[k] + d.N * d.sizes[k];
    }
  }
  p->path = LLAMA_PATH_PERMUTE;
  p->smem_bytes = (int)smem;
  return true;
}

// The plan-time specialised permute (jit.cpp) for wide records and splits.
bool plan_jit_path(const Mapping& s, const Mapping& d, int tile_records, const Knobs& kn, Plan* p, std::string* why) {
  std::unique_ptr<JitPlan> jp(new JitPlan);
  if (!plan_jit(s, d, tile_records, kn, jp.get(), why)) {
#ifdef LLB_DEBUG_JIT
    std::fprintf(stderr, "plan_jit: %s\n", why->c_str());
#endif
    return false;
  }
  p->path = LLAMA_PATH_PERMUTE;
  p->smem_bytes = (int)jp->smem;
  p->jit = std::move(jp);
  return true;
}

llama_status make_plan(const Mapping& s, const Mapping& d, llama_path path, int tile_records, const Knobs& kn,
                       Plan* out, std::string* err) {
  out->permute_v1 = kn.get(LLAMA_KNOB_PERMUTE_V1, 0) != 0;
  out->pdl = kn.get(LLAMA_KNOB_NO_PDL, 0) == 0;
  llama_status st = check_compatible(s, d, err);
  if (st != LLAMA_OK) return st;
  if (d.collides()) {  // the copy's result would depend on the order of the writes
    *err = "destination maps several records onto one location (One / a One part of a Split)";
    return LLAMA_ERR_UNSUPPORTED;
  }
  out->src_bytes = s.footprint_bytes();
  out->dst_bytes = d.footprint_bytes();
  if (out->dst_bytes == 0) {
    out->empty = true;
    out->path = path == LLAMA_PATH_AUTO ? LLAMA_PATH_BLOBCOPY : path;
    return LLAMA_OK;
  }
  std::string why;
  // record (index) -> record (index) across storage orders, or counting every
  // address resolution (Trace / Heatmap): the element-wise kernel only
  if (s.lin != d.lin || s.trace || d.trace) {
    const bool tr = path == LLAMA_PATH_AUTO || path == LLAMA_PATH_TRANSPOSE;
    if (tr && kn.get(LLAMA_KNOB_WIDE, 1) == 2 && plan_wide(s, d, kn, out, &why)) return LLAMA_OK;
    if (path == LLAMA_PATH_AUTO || path == LLAMA_PATH_TRANSPOSE) {
      std::unique_ptr<JitPlan> jp(new JitPlan);
      if (plan_jit2d(s, d, kn, jp.get(), &why)) {
        out->path = LLAMA_PATH_TRANSPOSE;
        out->smem_bytes = (int)jp->smem;
        out->jit = std::move(jp);
        return LLAMA_OK;
      }
#ifdef LLB_DEBUG_JIT
      std::fprintf(stderr, "plan_jit2d: %s\n", why.c_str());
#endif
    }
    if (tr && plan_transpose(s, d, kn, out, &why)) return LLAMA_OK;
    if (tr && plan_wide(s, d, kn, out, &why)) return LLAMA_OK;
    if (path != LLAMA_PATH_AUTO && path != LLAMA_PATH_NAIVE) {
      *err = "path not applicable to this mapping pair: linearised differently or traced: " + why;
      return LLAMA_ERR_UNSUPPORTED;
    }
    plan_naive(s, d, out);
    return LLAMA_OK;
  }
  if (path == LLAMA_PATH_TRANSPOSE) {
    *err = "path not applicable to this mapping pair: TRANSPOSE needs differently linearised views";
    return LLAMA_ERR_UNSUPPORTED;
  }
  switch (path) {
    case LLAMA_PATH_AUTO:
      // the warp-specialised TMA permute measured fastest on B200 for every
      // pair it applies to -- identities (6.25-6.40 vs 6.14-6.20 TB/s for the
      // bulk blob copy) and run pairs (SoA <-> AoSoA) included
      // identities of SoA layouts with many leaves (many blobs / segments): the bulk blob copy
      // (HEP SoA MB: 6.4 TB/s vs 1.8 for 200 TMA segment ops per tile)
      // and SoA layouts with many leaves into each other (one range per leaf:
      // HEP100 SoA SB <-> MB 5.0 TB/s through the JIT program -> see DESIGN.md)
      if (s.K() > 16 && (s.soa() || (single_runs(s) && single_runs(d))) && plan_blobcopy(s, d, kn, out, &why))
        return LLAMA_OK;
      if (plan_jit_path(s, d, tile_records, kn, out, &why)) return LLAMA_OK;
      if (plan_direct(s, d, tile_records, kn, out, &why)) return LLAMA_OK;
      if (plan_permute(s, d, tile_records, kn, out, &why)) return LLAMA_OK;
      if (plan_blobcopy(s, d, kn, out, &why)) return LLAMA_OK;
      if (plan_run(s, d, out, &why)) return LLAMA_OK;
      plan_naive(s, d, out);
      return LLAMA_OK;
    case LLAMA_PATH_NAIVE:
      plan_naive(s, d, out);
      return LLAMA_OK;
    case LLAMA_PATH_BLOBCOPY:
      if (plan_blobcopy(s, d, kn, out, &why)) return LLAMA_OK;
      break;
    case LLAMA_PATH_RUN:
      if (plan_run(s, d, out, &why)) return LLAMA_OK;
      break;
    case LLAMA_PATH_PERMUTE:
      if (plan_jit_path(s, d, tile_records, kn, out, &why)) return LLAMA_OK;
      if (plan_direct(s, d, tile_records, kn, out, &why)) return LLAMA_OK;
      if (plan_permute(s, d, tile_records, kn, out, &why)) return LLAMA_OK;
      break;
    default:
      *err = "bad path";
      return LLAMA_ERR_INVALID_ARGUMENT;
  }
  *err = "path not applicable to this mapping pair: " + why;
  return LLAMA_ERR_UNSUPPORTED;
}

}  // namespace llb
