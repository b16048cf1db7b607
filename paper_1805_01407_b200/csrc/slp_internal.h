// Internal declarations shared by the host algebra (slp_host.cpp) and the
// device launch code (slp_kernels.cu).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "slp_registry.h"

namespace slp {

// internal self-check failure (the reference raises Gf2Error, gf2.py:48-53)
struct AlgebraError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct GenDesc {
  int id;
  const char *name;
  int family, k, w, a, b, c;
  int scrambler, word_i, word_j;
  uint64_t S;
  int R;
  uint64_t T;
  int n() const { return k * w; }
  // engines sharing the same step matrix (generators.py:58-61 engine_key)
  bool same_engine(const GenDesc &o) const {
    return family == o.family && k == o.k && w == o.w && a == o.a && b == o.b && c == o.c;
  }
};

const GenDesc *gen_desc(int id);  // nullptr if out of range
int engine_id(int id);            // smallest generator id with the same engine
int rt_shape(int family, int k, int w);  // SLP_RT_SHAPES index of an engine shape, or -1

// ---- GF(2) polynomials: little-endian u64 words, bit i = coeff of x^i -----
using Poly = std::vector<uint64_t>;

int poly_degree(const Poly &p);  // -1 for zero
void poly_trim(Poly &p);
Poly poly_mul(const Poly &a, const Poly &b);
Poly poly_mod(Poly a, const Poly &m);
Poly poly_mulmod(const Poly &a, const Poly &b, const Poly &m);
// x^e mod m, e a little-endian multiword integer
Poly poly_x_pow(const uint64_t *e, int ewords, const Poly &m);

// engine step on a flat state of k words (each < 2^w); engines.py:100-140
void engine_step(const GenDesc &g, uint64_t *words);
// characteristic polynomial of the engine (cached per engine); throws on self-check failure
const Poly &engine_char_poly(const GenDesc &g);
const Poly &engine_char_poly(int id);
// host scalar jump of a flat state by polynomial p (Generator.jump semantics)
void host_jump(const GenDesc &g, const Poly &p, uint64_t *flat);

// ---- substream initialisation plan (kernel K1) -----------------------------
// A launch computes dst states [dst0, dst0 + count) of every block from the
// first `m` states: dst0 + t  <-  state (t % m) jumped by poly[poly0 + t / m].
// The first launch (m == 0) starts from the block base state with one poly
// per thread (poly0 + t).
struct InitLaunch {
  uint64_t dst0, count, m;
  uint64_t poly0;
  bool uniform;  // poly index warp-uniform (m % 32 == 0)
};
struct InitPlan {
  int pw;  // words per poly = ceil(n / 64)
  std::vector<uint64_t> polys;  // npolys * pw
  std::vector<InitLaunch> launches;
  uint64_t uid = 0;  // unique per built plan: key of its device copies (slp_api.cu)
};
// cached (bounded LRU); hold the pointer for the duration of a call
std::shared_ptr<const InitPlan> init_plan(int id, const uint64_t *steps, int steps_words, uint64_t n);

void set_last_error(const std::string &s);

}  // namespace slp
