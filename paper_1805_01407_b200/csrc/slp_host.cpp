// Host side of the C ABI: registry, scalar engine step, GF(2) polynomial
// algebra (characteristic polynomial, jump polynomials) and the substream
// initialisation plans consumed by kernel K1.
//
// Reference counterparts (paths relative to /root/reference/pkg/src/slprng/):
//   registry              generators.py:71-124
//   engine step           engines.py:100-140
//   char poly             gf2.py:418-486 (cyclic/Krylov decomposition, Cayley-Hamilton check)
//   x^e mod P             gf2.py:214-227 (square-and-multiply)
//   jump by polynomial    generators.py:315-334
//   lane doubling         generators.py:450-459 (here: radix-8 rounds, see init_plan)
#include <immintrin.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <system_error>
#include <thread>
#include <tuple>

#include "../../include/slp_b200.h"
#include "slp_internal.h"

namespace slp {

// ---------------------------------------------------------------------------
// registry

static const GenDesc kGens[SLP_NUM_GENERATORS] = {
#define SLP_X(id, name, fam, k, w, a, b, c, sc, wi, wj, S, R, T) \
  {id, #name, fam, k, w, a, b, c, sc, wi, wj, S, R, T},
    SLP_REGISTRY(SLP_X)
#undef SLP_X
};

// registered custom generators (custom_spec, generators.py:127-135), ids
// SLP_CUSTOM_ID0 + i; entries are never removed, so pointers stay valid
struct CustomGen {
  GenDesc d;
  char name[32];
};
static std::unique_ptr<CustomGen> g_custom[SLP_MAX_CUSTOM];
static std::atomic<int> g_ncustom{0};
static std::mutex g_custom_mu;

const GenDesc *gen_desc(int id) {
  if (id >= 0 && id < SLP_NUM_GENERATORS) return &kGens[id];
  if (id >= SLP_CUSTOM_ID0 && id < SLP_CUSTOM_ID0 + g_ncustom.load(std::memory_order_acquire))
    return &g_custom[id - SLP_CUSTOM_ID0]->d;
  return nullptr;
}

// the smallest registry id with the same engine, else the first registered
// custom generator with it: plans and jump tables are shared per engine
int engine_id(int id) {
  const GenDesc *g = gen_desc(id);
  if (!g) return id;
  for (int i = 0; i < SLP_NUM_GENERATORS; ++i)
    if (kGens[i].same_engine(*g)) return i;
  const int n = g_ncustom.load(std::memory_order_acquire);
  for (int i = 0; i < n; ++i)
    if (g_custom[i]->d.same_engine(*g)) return SLP_CUSTOM_ID0 + i;
  return id;
}

int rt_shape(int family, int k, int w) {
#define SLP_SHAPE_X(i, fam, kk, ww) \
  if (family == (fam) && k == (kk) && w == (ww)) return i;
  SLP_RT_SHAPES(SLP_SHAPE_X)
#undef SLP_SHAPE_X
  return -1;
}

static thread_local std::string t_last_error;
void set_last_error(const std::string &s) { t_last_error = s; }

// ---------------------------------------------------------------------------
// scalar engine step, flat view (engines.py:100-140)

static inline uint64_t rotl_w(uint64_t x, int r, int w, uint64_t mask) {
  return ((x << r) | (x >> (w - r))) & mask;
}

void engine_step(const GenDesc &g, uint64_t *s) {
  const int w = g.w, k = g.k;
  const uint64_t mask = w == 64 ? ~0ull : ((1ull << w) - 1);
  if (g.family == SLP_FAM_XOROSHIRO) {
    uint64_t x0 = s[0];
    uint64_t xl = s[k - 1] ^ x0;
    uint64_t m2 = rotl_w(x0, g.a, w, mask) ^ xl ^ ((xl << g.b) & mask);
    uint64_t m1 = rotl_w(xl, g.c, w, mask);
    for (int j = 0; j + 2 < k; ++j) s[j] = s[j + 1];
    s[k - 2] = m2;
    s[k - 1] = m1;
    return;
  }
  if (g.family == SLP_FAM_XOSHIRO && k == 4) {
    uint64_t t = (s[1] << g.a) & mask;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl_w(s[3], g.b, w, mask);
    return;
  }
  if (g.family == SLP_FAM_XOSHIRO) {
    uint64_t t = (s[1] << g.a) & mask;
    s[2] ^= s[0];
    s[5] ^= s[1];
    s[1] ^= s[2];
    s[7] ^= s[3];
    s[3] ^= s[4];
    s[4] ^= s[5];
    s[0] ^= s[6];
    s[6] ^= s[7];
    s[6] ^= t;
    s[7] = rotl_w(s[7], g.b, w, mask);
    return;
  }
  // xorshift, k = 2
  uint64_t s0 = s[0], s1 = s[1];
  uint64_t t = s0 ^ ((s0 << g.a) & mask);
  s[0] = s1;
  s[1] = t ^ (t >> g.b) ^ s1 ^ (s1 >> g.c);
}

// ---------------------------------------------------------------------------
// GF(2) polynomials

int poly_degree(const Poly &p) {
  for (int i = (int)p.size() - 1; i >= 0; --i)
    if (p[i]) return i * 64 + 63 - __builtin_clzll(p[i]);
  return -1;
}

void poly_trim(Poly &p) {
  while (!p.empty() && p.back() == 0) p.pop_back();
}

// 64 x 64 -> 128 carry-less product: PCLMULQDQ when the host CPU has it,
// else a portable 4-bit window.
__attribute__((target("pclmul,sse4.1"))) static void clmul64_hw(uint64_t a, uint64_t b, uint64_t &lo,
                                                                  uint64_t &hi) {
  const __m128i r = _mm_clmulepi64_si128(_mm_cvtsi64_si128((long long)a), _mm_cvtsi64_si128((long long)b), 0);
  lo = (uint64_t)_mm_cvtsi128_si64(r);
  hi = (uint64_t)_mm_extract_epi64(r, 1);
}

static void clmul64_sw(uint64_t a, uint64_t b, uint64_t &lo, uint64_t &hi) {
  uint64_t tbl_lo[16], tbl_hi[16];
  tbl_lo[0] = 0;
  tbl_hi[0] = 0;
  for (int v = 1; v < 16; ++v) {
    int low = __builtin_ctz(v);
    int rest = v & (v - 1);
    uint64_t sl = low ? (b << low) : b;
    uint64_t sh = low ? (b >> (64 - low)) : 0;
    tbl_lo[v] = tbl_lo[rest] ^ sl;
    tbl_hi[v] = tbl_hi[rest] ^ sh;
  }
  lo = 0;
  hi = 0;
  for (int i = 60; i >= 0; i -= 4) {
    hi = (hi << 4) | (lo >> 60);
    lo <<= 4;
    unsigned nib = (a >> i) & 15;
    lo ^= tbl_lo[nib];
    hi ^= tbl_hi[nib];
  }
}

static const bool g_has_pclmul = __builtin_cpu_supports("pclmul") && __builtin_cpu_supports("sse4.1");

static inline void clmul64(uint64_t a, uint64_t b, uint64_t &lo, uint64_t &hi) {
  if (g_has_pclmul)
    clmul64_hw(a, b, lo, hi);
  else
    clmul64_sw(a, b, lo, hi);
}

Poly poly_mul(const Poly &a, const Poly &b) {
  if (a.empty() || b.empty()) return Poly();
  Poly r(a.size() + b.size(), 0);
  for (size_t i = 0; i < a.size(); ++i) {
    if (!a[i]) continue;
    for (size_t j = 0; j < b.size(); ++j) {
      if (!b[j]) continue;
      uint64_t lo, hi;
      clmul64(a[i], b[j], lo, hi);
      r[i + j] ^= lo;
      r[i + j + 1] ^= hi;
    }
  }
  poly_trim(r);
  return r;
}

// generic long division remainder (bit-serial); used once per modulus
Poly poly_mod(Poly a, const Poly &m) {
  const int dm = poly_degree(m);
  if (dm < 0) throw std::invalid_argument("polynomial modulus is zero");
  int da = poly_degree(a);
  while (da >= dm) {
    const int sh = da - dm;
    const int ws = sh / 64, bs = sh % 64;
    for (size_t j = 0; j < m.size(); ++j) {
      uint64_t v = m[j];
      if (!v) continue;
      a[j + ws] ^= v << bs;
      if (bs && j + ws + 1 < a.size()) a[j + ws + 1] ^= v >> (64 - bs);
    }
    int wi = da / 64;
    while (wi >= 0 && a[wi] == 0) --wi;
    da = wi < 0 ? -1 : wi * 64 + 63 - __builtin_clzll(a[wi]);
  }
  poly_trim(a);
  return a;
}

// a >> s (drop the s lowest coefficients)
static Poly poly_shr(const Poly &a, int s) {
  const int ws = s / 64, bs = s % 64;
  if ((int)a.size() <= ws) return Poly();
  Poly r(a.size() - ws, 0);
  for (size_t i = 0; i < r.size(); ++i) {
    uint64_t v = a[i + ws] >> bs;
    if (bs && i + ws + 1 < a.size()) v |= a[i + ws + 1] << (64 - bs);
    r[i] = v;
  }
  poly_trim(r);
  return r;
}

// Barrett reduction modulo P of degree n: mu = x^(2n) div P; for deg A < 2n,
// A div P = ((A >> n) * mu) >> n exactly over GF(2), so A mod P costs two
// multiplications instead of n shift-xor steps.
struct Reducer {
  Poly P;
  int n;
  Poly mu;
  explicit Reducer(const Poly &m) : P(m), n(poly_degree(m)) {
    if (n < 1) throw std::invalid_argument("modulus must have degree >= 1");
    // long division of x^(2n) by P, collecting the quotient
    Poly rem((size_t)(2 * n) / 64 + 1, 0);
    rem[(2 * n) / 64] = 1ull << ((2 * n) % 64);
    mu.assign((size_t)n / 64 + 1, 0);
    int dr = 2 * n;
    while (dr >= n) {
      const int sh = dr - n;
      mu[sh / 64] |= 1ull << (sh % 64);
      const int ws = sh / 64, bs = sh % 64;
      for (size_t j = 0; j < P.size(); ++j) {
        uint64_t v = P[j];
        if (!v) continue;
        rem[j + ws] ^= v << bs;
        if (bs && j + ws + 1 < rem.size()) rem[j + ws + 1] ^= v >> (64 - bs);
      }
      int wi = dr / 64;
      while (wi >= 0 && rem[wi] == 0) --wi;
      dr = wi < 0 ? -1 : wi * 64 + 63 - __builtin_clzll(rem[wi]);
    }
    poly_trim(mu);
  }
  Poly reduce(Poly a) const {
    if (poly_degree(a) < n) return a;
    if (poly_degree(a) >= 2 * n) return poly_mod(std::move(a), P);
    const Poly q = poly_shr(poly_mul(poly_shr(a, n), mu), n);
    const Poly qp = poly_mul(q, P);
    for (size_t i = 0; i < qp.size() && i < a.size(); ++i) a[i] ^= qp[i];
    poly_trim(a);
    return a;
  }
  Poly mulmod(const Poly &a, const Poly &b) const { return reduce(poly_mul(a, b)); }
};

Poly poly_mulmod(const Poly &a, const Poly &b, const Poly &m) { return Reducer(m).mulmod(a, b); }

// squaring over GF(2) interleaves zeros between the coefficient bits
static uint16_t g_spread[256];
static const bool g_spread_init = [] {
  for (int v = 0; v < 256; ++v) {
    uint16_t r = 0;
    for (int b = 0; b < 8; ++b) r |= (uint16_t)(((v >> b) & 1) << (2 * b));
    g_spread[v] = r;
  }
  return true;
}();

static Poly poly_sqr(const Poly &a) {
  Poly r(a.size() * 2, 0);
  for (size_t i = 0; i < a.size(); ++i) {
    const uint64_t v = a[i];
    uint64_t lo = 0, hi = 0;
    for (int k = 0; k < 4; ++k) {
      lo |= (uint64_t)g_spread[(v >> (8 * k)) & 0xFF] << (16 * k);
      hi |= (uint64_t)g_spread[(v >> (32 + 8 * k)) & 0xFF] << (16 * k);
    }
    r[2 * i] = lo;
    r[2 * i + 1] = hi;
  }
  poly_trim(r);
  return r;
}

static Poly poly_mulx_mod(Poly a, const Poly &m, int dm) {
  // a * x mod m, deg a < dm
  a.resize((size_t)dm / 64 + 2, 0);
  uint64_t carry = 0;
  for (auto &v : a) {
    uint64_t nc = v >> 63;
    v = (v << 1) | carry;
    carry = nc;
  }
  if ((a[dm / 64] >> (dm % 64)) & 1ull)
    for (size_t j = 0; j < m.size(); ++j) a[j] ^= m[j];
  poly_trim(a);
  return a;
}

Poly poly_x_pow(const uint64_t *e, int ewords, const Poly &m) {
  const int dm = poly_degree(m);
  if (dm < 1) throw std::invalid_argument("modulus must have degree >= 1");
  int top = -1;
  for (int i = ewords - 1; i >= 0; --i)
    if (e[i]) {
      top = i * 64 + 63 - __builtin_clzll(e[i]);
      break;
    }
  Poly r{1};
  if (dm == 1 && (m[0] & 1) == 0) {
    // modulus x: x^e mod x
    return top < 0 ? r : Poly();
  }
  const Reducer red(m);
  r = poly_mod(r, m);
  // left-to-right: square, then multiply by x for a set bit
  for (int bit = top; bit >= 0; --bit) {
    r = red.reduce(poly_sqr(r));
    if ((e[bit / 64] >> (bit % 64)) & 1ull) r = poly_mulx_mod(r, m, dm);
  }
  return r;
}

// ---------------------------------------------------------------------------
// characteristic polynomial by cyclic decomposition of the row action
// v -> v*M (= engine step in the flat view).  Each new cyclic vector's chain
// is reduced modulo the span already found; the monic relation that closes
// the chain is the relative annihilator, and the product of those is det(xI - M).
// Same mathematics as gf2.py:418-469, written over fixed-width bitsets.

namespace {
constexpr int kMaxN = 1024;
constexpr int kVW = kMaxN / 64;      // vector words
constexpr int kPW = kMaxN / 64 + 1;  // combo words (degree <= n)

struct BitVec {
  uint64_t v[kVW];
};
struct Combo {
  uint64_t v[kPW];
};

inline int top_bit(const uint64_t *v, int nw) {
  for (int i = nw - 1; i >= 0; --i)
    if (v[i]) return i * 64 + 63 - __builtin_clzll(v[i]);
  return -1;
}

// pack flat words (k words of w bits) into bit vector: word j at bits [j*w, (j+1)*w)
void pack(const GenDesc &g, const uint64_t *words, uint64_t *bits) {
  std::memset(bits, 0, sizeof(uint64_t) * kVW);
  for (int j = 0; j < g.k; ++j) {
    for (int t = 0; t < g.w; ++t) {
      if ((words[j] >> t) & 1ull) {
        int p = j * g.w + t;
        bits[p / 64] |= 1ull << (p % 64);
      }
    }
  }
}
void unpack(const GenDesc &g, const uint64_t *bits, uint64_t *words) {
  for (int j = 0; j < g.k; ++j) {
    uint64_t x = 0;
    for (int t = 0; t < g.w; ++t) {
      int p = j * g.w + t;
      x |= ((bits[p / 64] >> (p % 64)) & 1ull) << t;
    }
    words[j] = x;
  }
}
void mul_vec(const GenDesc &g, const uint64_t *in, uint64_t *out) {
  uint64_t w[64];
  unpack(g, in, w);
  engine_step(g, w);
  pack(g, w, out);
}
}  // namespace

static Poly char_poly_compute(const GenDesc &g) {
  const int n = g.n();
  if (n > kMaxN) throw std::invalid_argument("state too large");
  const int nw = (n + 63) / 64;
  std::vector<BitVec> basis;         // vectors spanning the found invariant subspace
  std::vector<int> basis_at(n, -1);  // pivot -> basis index
  Poly result{1};
  int dim = 0, j = 0;
  while (dim < n) {
    // next unit vector outside the span
    BitVec v{};
    for (;; ++j) {
      BitVec r{};
      r.v[j / 64] = 1ull << (j % 64);
      int p;
      while ((p = top_bit(r.v, nw)) >= 0 && basis_at[p] >= 0)
        for (int i = 0; i < nw; ++i) r.v[i] ^= basis[basis_at[p]].v[i];
      if (p >= 0) {
        std::memset(&v, 0, sizeof v);
        v.v[j / 64] = 1ull << (j % 64);
        ++j;
        break;
      }
    }
    std::vector<BitVec> cvec;
    std::vector<Combo> ccomb;
    std::vector<int> chain_at(n, -1);
    BitVec u = v;
    Combo up{};
    up.v[0] = 1;
    int power = 0;
    Combo g_rel{};
    for (;;) {
      BitVec r = u;
      Combo c = up;
      int p;
      for (;;) {
        p = top_bit(r.v, nw);
        if (p < 0) break;
        if (chain_at[p] >= 0) {
          const int ci = chain_at[p];
          for (int i = 0; i < nw; ++i) r.v[i] ^= cvec[ci].v[i];
          for (int i = 0; i < kPW; ++i) c.v[i] ^= ccomb[ci].v[i];
        } else if (basis_at[p] >= 0) {
          for (int i = 0; i < nw; ++i) r.v[i] ^= basis[basis_at[p]].v[i];
        } else {
          break;
        }
      }
      if (p < 0) {
        g_rel = c;
        break;
      }
      chain_at[p] = (int)cvec.size();
      cvec.push_back(r);
      ccomb.push_back(c);
      BitVec nu{};
      mul_vec(g, u.v, nu.v);
      u = nu;
      ++power;
      if (power > n) throw std::runtime_error("char_poly: chain did not close");
      // up <<= 1
      uint64_t carry = 0;
      for (int i = 0; i < kPW; ++i) {
        uint64_t nc = up.v[i] >> 63;
        up.v[i] = (up.v[i] << 1) | carry;
        carry = nc;
      }
    }
    Poly gp(g_rel.v, g_rel.v + kPW);
    poly_trim(gp);
    result = poly_mul(result, gp);
    for (size_t i = 0; i < cvec.size(); ++i) {
      int p = top_bit(cvec[i].v, nw);
      basis_at[p] = (int)basis.size();
      basis.push_back(cvec[i]);
    }
    dim += (int)cvec.size();
  }
  poly_trim(result);
  return result;
}

// Cayley-Hamilton self-check: P(M) == 0, applied to every unit vector
// (gf2.py:472-486).
static bool cayley_hamilton_holds(const GenDesc &g, const Poly &P) {
  const int n = g.n();
  const int deg = poly_degree(P);
  std::vector<uint64_t> cur(g.k), acc(g.k), unit_bits(kVW);
  for (int i = 0; i < n; ++i) {
    std::fill(unit_bits.begin(), unit_bits.end(), 0);
    unit_bits[i / 64] = 1ull << (i % 64);
    unpack(g, unit_bits.data(), cur.data());
    std::fill(acc.begin(), acc.end(), 0);
    for (int d = 0; d <= deg; ++d) {
      if ((P[d / 64] >> (d % 64)) & 1ull)
        for (int q = 0; q < g.k; ++q) acc[q] ^= cur[q];
      if (d != deg) engine_step(g, cur.data());
    }
    for (int q = 0; q < g.k; ++q)
      if (acc[q]) return false;
  }
  return true;
}

static std::mutex g_cp_mu;
static std::map<std::tuple<int, int, int, int, int, int>, std::unique_ptr<Poly>> g_cp_cache;

const Poly &engine_char_poly(const GenDesc &g) {
  const auto key = std::make_tuple(g.family, g.k, g.w, g.a, g.b, g.c);
  {
    std::lock_guard<std::mutex> lk(g_cp_mu);
    auto it = g_cp_cache.find(key);
    if (it != g_cp_cache.end()) return *it->second;
  }
  Poly P = char_poly_compute(g);
  if (poly_degree(P) != g.n() || !cayley_hamilton_holds(g, P))
    throw AlgebraError("characteristic polynomial failed Cayley-Hamilton check");
  std::lock_guard<std::mutex> lk(g_cp_mu);
  auto res = g_cp_cache.emplace(key, std::make_unique<Poly>(std::move(P)));
  return *res.first->second;
}

const Poly &engine_char_poly(int id) { return engine_char_poly(*gen_desc(engine_id(id))); }

void host_jump(const GenDesc &g, const Poly &p, uint64_t *flat) {
  const int deg = poly_degree(p);
  uint64_t cur[64], acc[64];
  for (int i = 0; i < g.k; ++i) {
    cur[i] = flat[i];
    acc[i] = 0;
  }
  for (int d = 0; d <= deg; ++d) {
    if ((p[d / 64] >> (d % 64)) & 1ull)
      for (int i = 0; i < g.k; ++i) acc[i] ^= cur[i];
    if (d != deg) engine_step(g, cur);
  }
  for (int i = 0; i < g.k; ++i) flat[i] = acc[i];
}

// ---------------------------------------------------------------------------
// substream init plans (kernel K1).
//
// Stream i of a block is base * M^(i*J).  Launch 0 gives each of the first
// m0 = min(n, 1024) streams its own polynomial x^(iJ) mod P (one jump per
// stream, all independent, so the latency is one jump instead of the
// log2(m0) dependent rounds of the reference's doubling, generators.py:450-459).
// Later launches grow the prefix by a radix of up to 8: stream m*c + s
// (c < 8, s < m) is stream s jumped by x^(c*m*J).  Every stream is produced
// by exactly one polynomial jump, as in the reference.

static constexpr uint64_t kDirect = 1024;

// direct (launch-0) polynomials per plan: fewer for wide engines, whose
// non-uniform direct jumps are latency-bound (SLP_PLAN_DIRECT overrides, A/B)
static uint64_t plan_direct(int nbits) {
  static const long env = [] {
    const char *v = std::getenv("SLP_PLAN_DIRECT");
    return v && *v ? std::atol(v) : 0L;
  }();
  if (env > 0) return (uint64_t)env;
  return nbits <= 256 ? kDirect : (nbits <= 512 ? kDirect / 4 : kDirect / 8);
}
// Requests beyond the small direct set of a wide engine get 4096 direct
// polynomials (SLP_PLAN_DIRECT_BIG overrides): since K1 splits a wide jump
// over lanes, one launch of 4096 per-lane-polynomial jumps costs less than
// the radix-8 rounds it replaces (xoroshiro1024: 2^15 substreams 0.160 ->
// 0.088 ms, one stream of 2^28 outputs 4.29 -> 5.0 TB/s;
// profiles/round2_jump_parts.md).  Their host cost (one degree-n mulmod
// each, ~4.4 us for n = 1024) is spread over threads in init_plan.
static uint64_t plan_direct_big(int nbits) {
  static const long env = [] {
    const char *v = std::getenv("SLP_PLAN_DIRECT_BIG");
    return v && *v ? std::atol(v) : 0L;
  }();
  const uint64_t small = plan_direct(nbits);
  if (env > 0) return (uint64_t)env > small ? (uint64_t)env : small;
  return nbits <= 256 ? small : 4096;
}
static constexpr uint64_t kRadix = 8;

struct PlanKey {
  int eid;
  std::vector<uint64_t> steps;
  uint64_t n;
  bool operator<(const PlanKey &o) const { return std::tie(eid, steps, n) < std::tie(o.eid, o.steps, o.n); }
};

// bounded LRU: plans are keyed by the exact stride (segment split: T / J,
// lane_len, HWD segment lengths), so a long-running caller may see many;
// callers hold a shared_ptr for the duration of a call, so eviction never
// pulls a plan from under a launch.  Device copies are keyed by InitPlan::uid
// (slp_api.cu) and age out of their own LRU.
static constexpr size_t kMaxPlans = 256;
static std::mutex g_plan_mu;
struct PlanSlot {
  std::shared_ptr<const InitPlan> plan;
  uint64_t tick;
};
static std::map<PlanKey, PlanSlot> g_plans;
static uint64_t g_plan_tick = 0, g_plan_uid = 0;

std::shared_ptr<const InitPlan> init_plan(int id, const uint64_t *steps, int steps_words, uint64_t n_req) {
  const int eid = engine_id(id);
  std::vector<uint64_t> st(steps, steps + steps_words);
  while (!st.empty() && st.back() == 0) st.pop_back();
  // Plans are built for n = ndirect * 8^r >= n_req and serve every smaller
  // count (the launches are a prefix; the caller clips them to its n), so a
  // caller with many different counts (HWD ranges) shares O(log n) plans and
  // their device tables instead of one per count.
  const GenDesc &gd = *gen_desc(eid);
  const uint64_t nd = n_req <= plan_direct(gd.n()) ? plan_direct(gd.n()) : plan_direct_big(gd.n());
  uint64_t n = nd;
  while (n < n_req) n *= kRadix;
  PlanKey key{eid, st, n};
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto it = g_plans.find(key);
    if (it != g_plans.end()) {
      it->second.tick = ++g_plan_tick;
      return it->second.plan;
    }
  }
  const GenDesc &g = *gen_desc(eid);
  const Poly &P = engine_char_poly(eid);
  auto plan = std::make_shared<InitPlan>();
  const int pw = (g.n() + 63) / 64;
  plan->pw = pw;
  auto push = [&](const Poly &p) {
    for (int i = 0; i < pw; ++i) plan->polys.push_back(i < (int)p.size() ? p[i] : 0);
  };
  const Poly xJ = poly_x_pow(st.data(), (int)st.size(), P);
  const Reducer red(P);
  // fewer direct polynomials for wide engines: each costs a host mulmod of
  // degree-n polys (plan build time), the rounds that replace them are cheap
  const uint64_t m0 = nd;  // n = nd * 8^r
  // launch 0: x^(iJ) for i < m0.  A long chain is cut into blocks: the block
  // starts x^(kBJ) come from x^(BJ) (square-and-multiply), then one thread per
  // block multiplies by x^J.
  Poly cur{1};
  cur = poly_mod(cur, P);
  std::vector<Poly> direct(m0);
  unsigned nthr = std::thread::hardware_concurrency();
  if (nthr > 16) nthr = 16;
  if (m0 < 1024 || nthr < 2) {
    for (uint64_t i = 0; i < m0; ++i) {
      direct[i] = cur;
      cur = red.mulmod(cur, xJ);
    }
  } else {
    const uint64_t B = (m0 + nthr - 1) / nthr;
    Poly xBJ{1}, sq = xJ;  // x^(BJ)
    for (uint64_t e = B; e; e >>= 1) {
      if (e & 1) xBJ = red.mulmod(xBJ, sq);
      if (e > 1) sq = red.mulmod(sq, sq);
    }
    std::vector<Poly> starts;
    for (uint64_t lo = 0; lo < m0; lo += B) {
      starts.push_back(cur);
      cur = red.mulmod(cur, xBJ);
    }
    std::vector<Poly> ends(starts.size());
    auto work = [&](size_t k) {
      Poly c = starts[k];
      const uint64_t lo = k * B, hi = lo + B < m0 ? lo + B : m0;
      for (uint64_t i = lo; i < hi; ++i) {
        direct[i] = c;
        c = red.mulmod(c, xJ);
      }
      ends[k] = c;
    };
    std::vector<std::thread> pool;
    size_t spawned = 0;
    try {
      for (; spawned + 1 < starts.size(); ++spawned) pool.emplace_back(work, spawned);
    } catch (const std::system_error &) {
      // no more threads: the remaining blocks run here
    }
    for (size_t k = spawned; k < starts.size(); ++k) work(k);  // the last block (and any unspawned) inline
    for (auto &t : pool) t.join();
    cur = ends.back();  // x^(m0 J)
  }
  for (uint64_t i = 0; i < m0; ++i) push(direct[i]);
  plan->launches.push_back(InitLaunch{0, m0, 0, 0, false});
  // x^(m0 J) is `cur` now
  uint64_t m = m0;
  Poly xmJ = cur;  // x^(m J)
  while (m < n) {
    uint64_t radix = (n - m + m - 1) / m + 1;  // ceil(n/m)
    if (radix > kRadix) radix = kRadix;
    const uint64_t poly0 = plan->polys.size() / pw;
    Poly pc = xmJ;  // c = 1
    for (uint64_t c = 1; c < radix; ++c) {
      push(pc);
      pc = red.mulmod(pc, xmJ);
    }
    // after the loop pc = x^(radix * m * J)
    uint64_t count = (radix - 1) * m;
    if (count > n - m) count = n - m;
    plan->launches.push_back(InitLaunch{m, count, m, poly0, (m % 32) == 0});
    m += count;
    xmJ = pc;
  }
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) {  // built concurrently by another thread
    it->second.tick = ++g_plan_tick;
    return it->second.plan;
  }
  while (g_plans.size() >= kMaxPlans) {
    auto lru = g_plans.begin();
    for (auto jt = g_plans.begin(); jt != g_plans.end(); ++jt)
      if (jt->second.tick < lru->second.tick) lru = jt;
    g_plans.erase(lru);
  }
  plan->uid = ++g_plan_uid;
  std::shared_ptr<const InitPlan> cp = plan;
  g_plans.emplace(std::move(key), PlanSlot{cp, ++g_plan_tick});
  return cp;
}

}  // namespace slp

// ---------------------------------------------------------------------------
// C ABI (host part)

using namespace slp;

extern "C" {

int slp_num_generators(void) { return SLP_NUM_GENERATORS; }

int slp_generator_id(const char *name) {
  if (!name) return SLP_ERR_INVALID;
  for (int i = 0; i < SLP_NUM_GENERATORS; ++i)
    if (std::strcmp(kGens[i].name, name) == 0) return i;
  return SLP_ERR_UNKNOWN_GENERATOR;
}

int slp_generator_info(int id, slp_gen_info *out) {
  const GenDesc *g = gen_desc(id);
  if (!g) return SLP_ERR_UNKNOWN_GENERATOR;
  if (!out) return SLP_ERR_INVALID;
  std::memset(out, 0, sizeof *out);
  out->id = g->id;
  out->family = g->family;
  out->k = g->k;
  out->w = g->w;
  out->a = g->a;
  out->b = g->b;
  out->c = g->c;
  out->scrambler = g->scrambler;
  out->word_i = g->word_i;
  out->word_j = g->word_j;
  out->R = g->R;
  out->S = g->S;
  out->T = g->T;
  std::strncpy(out->name, g->name, sizeof(out->name) - 1);
  return SLP_OK;
}

static int copy_poly(const Poly &p, uint64_t *out, int words) {
  if ((int)p.size() > words) return SLP_ERR_BUFFER;
  for (int i = 0; i < words; ++i) out[i] = i < (int)p.size() ? p[i] : 0;
  return SLP_OK;
}

int slp_char_poly(int id, uint64_t *poly, int poly_words) {
  if (!gen_desc(id)) return SLP_ERR_UNKNOWN_GENERATOR;
  if (!poly || poly_words <= 0) return SLP_ERR_INVALID;
  try {
    return copy_poly(engine_char_poly(id), poly, poly_words);
  } catch (const AlgebraError &e) {
    set_last_error(e.what());
    return SLP_ERR_ALGEBRA;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return SLP_ERR_INVALID;
  }
}

int slp_jump_poly(int id, const uint64_t *steps, int steps_words, uint64_t *poly, int poly_words) {
  if (!gen_desc(id)) return SLP_ERR_UNKNOWN_GENERATOR;
  if (!poly || poly_words <= 0 || steps_words < 0 || (steps_words > 0 && !steps)) return SLP_ERR_INVALID;
  try {
    Poly p = poly_x_pow(steps, steps_words, engine_char_poly(id));
    return copy_poly(p, poly, poly_words);
  } catch (const AlgebraError &e) {
    set_last_error(e.what());
    return SLP_ERR_ALGEBRA;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return SLP_ERR_INVALID;
  }
}

int64_t slp_init_plan_poly(int id, const uint64_t *steps, int steps_words, uint64_t n, uint64_t index,
                           uint64_t *poly, int poly_words) {
  if (!gen_desc(id)) return SLP_ERR_UNKNOWN_GENERATOR;
  if (steps_words < 0 || (steps_words > 0 && !steps) || n == 0) return SLP_ERR_INVALID;
  try {
    const auto plan = init_plan(id, steps, steps_words, n);
    const uint64_t count = plan->polys.size() / (uint64_t)plan->pw;
    if (poly && index < count) {
      if (poly_words < plan->pw) return SLP_ERR_INVALID;
      for (int i = 0; i < poly_words; ++i)
        poly[i] = i < plan->pw ? plan->polys[index * (uint64_t)plan->pw + (uint64_t)i] : 0;
    }
    return (int64_t)count;
  } catch (const AlgebraError &e) {
    set_last_error(e.what());
    return SLP_ERR_ALGEBRA;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return SLP_ERR_INVALID;
  }
}

int slp_host_jump(int id, const uint64_t *poly, int poly_words, uint64_t *flat_state) {
  const GenDesc *g = gen_desc(id);
  if (!g) return SLP_ERR_UNKNOWN_GENERATOR;
  if (!poly || !flat_state || poly_words <= 0) return SLP_ERR_INVALID;
  Poly p(poly, poly + poly_words);
  poly_trim(p);
  if (p.empty()) return SLP_ERR_ZERO_STATE;  // "jump polynomial is zero"
  const uint64_t mask = g->w == 64 ? ~0ull : ((1ull << g->w) - 1);
  bool any = false;
  for (int i = 0; i < g->k; ++i) {
    if (flat_state[i] & ~mask) return SLP_ERR_INVALID;
    any |= flat_state[i] != 0;
  }
  if (!any) return SLP_ERR_ZERO_STATE;
  host_jump(*g, p, flat_state);
  return SLP_OK;
}

static int custom_desc(int family, int k, int w, int a, int b, int c, GenDesc *g) {
  // validation of engines.py:43-97 (EngineKind / _check_params)
  if (family < 0 || family > 2 || w < 2 || w > 64 || k < 2 || k * w > 1024) return SLP_ERR_INVALID;
  if (family == SLP_FAM_XOSHIRO && k != 4 && k != 8) return SLP_ERR_INVALID;
  if (family == SLP_FAM_XORSHIFT && k != 2) return SLP_ERR_INVALID;
  if (k > 64) return SLP_ERR_INVALID;
  const bool needs_c = family != SLP_FAM_XOSHIRO;
  if (!(0 < a && a < w) || !(0 < b && b < w) || (needs_c && !(0 < c && c < w))) return SLP_ERR_INVALID;
  *g = GenDesc{-1, "custom", family, k, w, a, b, needs_c ? c : 0, SLP_SC_NONE, 0, -1, 0, 0, 0};
  return SLP_OK;
}

static bool scrambler_ok(const slp_gen_info &s, int k, int w) {
  // ScramblerSpec.validate (scramblers.py:68-82)
  if (s.scrambler < SLP_SC_NONE || s.scrambler > SLP_SC_STARSTAR) return false;
  if (s.word_i < 0 || s.word_i >= k) return false;
  if ((s.scrambler == SLP_SC_PLUS || s.scrambler == SLP_SC_PLUSPLUS) && (s.word_j < 0 || s.word_j >= k)) return false;
  if ((s.scrambler == SLP_SC_STAR || s.scrambler == SLP_SC_STARSTAR) && (s.S % 2 == 0)) return false;
  if ((s.scrambler == SLP_SC_PLUSPLUS || s.scrambler == SLP_SC_STARSTAR) && !(0 < s.R && s.R < w)) return false;
  if (s.scrambler == SLP_SC_STARSTAR && s.T % 2 == 0) return false;
  return true;
}

int slp_register_generator(const slp_gen_info *spec) {
  if (!spec) return SLP_ERR_INVALID;
  GenDesc g;
  int rc = custom_desc(spec->family, spec->k, spec->w, spec->a, spec->b, spec->c, &g);
  if (rc != SLP_OK) return rc;
  if (!scrambler_ok(*spec, g.k, g.w)) return SLP_ERR_INVALID;
  const uint64_t wmask = g.w == 64 ? ~0ull : ((1ull << g.w) - 1);
  g.scrambler = spec->scrambler;
  g.word_i = spec->word_i;
  const bool uses_j = g.scrambler == SLP_SC_PLUS || g.scrambler == SLP_SC_PLUSPLUS;
  g.word_j = uses_j ? spec->word_j : -1;
  const bool uses_s = g.scrambler == SLP_SC_STAR || g.scrambler == SLP_SC_STARSTAR;
  g.S = uses_s ? spec->S & wmask : 0;  // (x * S) mod 2^w only depends on S mod 2^w
  g.R = (g.scrambler == SLP_SC_PLUSPLUS || g.scrambler == SLP_SC_STARSTAR) ? spec->R : 0;
  g.T = g.scrambler == SLP_SC_STARSTAR ? spec->T & wmask : 0;
  auto same = [&](const GenDesc &o) {
    return o.same_engine(g) && o.scrambler == g.scrambler && o.word_i == g.word_i && o.word_j == g.word_j &&
           o.S == g.S && o.R == g.R && o.T == g.T;
  };
  for (int i = 0; i < SLP_NUM_GENERATORS; ++i)
    if (same(kGens[i])) return i;  // identical to a registry generator: same kernels
  std::lock_guard<std::mutex> lk(g_custom_mu);
  const int n = g_ncustom.load(std::memory_order_relaxed);
  for (int i = 0; i < n; ++i)
    if (same(g_custom[i]->d)) return SLP_CUSTOM_ID0 + i;
  if (n >= SLP_MAX_CUSTOM) {
    set_last_error("too many registered custom generators");
    return SLP_ERR_BUFFER;
  }
  auto c = std::make_unique<CustomGen>();
  c->d = g;
  c->d.id = SLP_CUSTOM_ID0 + n;
  std::memset(c->name, 0, sizeof c->name);
  const char *nm = spec->name[0] ? spec->name : "custom";
  std::memcpy(c->name, nm, strnlen(nm, sizeof(c->name) - 1));  // spec->name need not be terminated
  c->d.name = c->name;
  g_custom[n] = std::move(c);
  g_ncustom.store(n + 1, std::memory_order_release);
  return SLP_CUSTOM_ID0 + n;
}

int slp_engine_char_poly(int family, int k, int w, int a, int b, int c, uint64_t *poly, int poly_words) {
  GenDesc g;
  int rc = custom_desc(family, k, w, a, b, c, &g);
  if (rc != SLP_OK) return rc;
  if (!poly || poly_words <= 0) return SLP_ERR_INVALID;
  try {
    return copy_poly(engine_char_poly(g), poly, poly_words);
  } catch (const AlgebraError &e) {
    set_last_error(e.what());
    return SLP_ERR_ALGEBRA;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return SLP_ERR_INVALID;
  }
}

int slp_engine_jump_poly(int family, int k, int w, int a, int b, int c, const uint64_t *steps, int steps_words,
                         uint64_t *poly, int poly_words) {
  GenDesc g;
  int rc = custom_desc(family, k, w, a, b, c, &g);
  if (rc != SLP_OK) return rc;
  if (!poly || poly_words <= 0 || steps_words < 0 || (steps_words > 0 && !steps)) return SLP_ERR_INVALID;
  try {
    return copy_poly(poly_x_pow(steps, steps_words, engine_char_poly(g)), poly, poly_words);
  } catch (const AlgebraError &e) {
    set_last_error(e.what());
    return SLP_ERR_ALGEBRA;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return SLP_ERR_INVALID;
  }
}

const char *slp_status_str(int s) {
  switch (s) {
    case SLP_OK: return "ok";
    case SLP_ERR_INVALID: return "invalid argument";
    case SLP_ERR_UNKNOWN_GENERATOR: return "unknown generator";
    case SLP_ERR_UNSUPPORTED: return "unsupported by the device path";
    case SLP_ERR_ZERO_STATE: return "all-zero state or zero jump polynomial";
    case SLP_ERR_CUDA: return "CUDA error";
    case SLP_ERR_ALGEBRA: return "GF(2) self-check failed";
    case SLP_ERR_BUFFER: return "buffer too small";
    default: return "unknown status";
  }
}

const char *slp_last_error(void) { return t_last_error.c_str(); }

}  // extern "C"
