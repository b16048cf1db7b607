// Device building blocks for the scrambled linear generators on sm_100a:
// word operations, the Gen<> template (engine step + scrambler), output
// conversions and PTX helpers.  Kernels: slp_fill.cuh (K2/K3), slp_fused.cuh
// (K4), slp_jump.cuh (K1, K1t), slp_hwd.cuh (K6); slp_device.cuh includes all.
//
// One template instance per registry generator (slp_registry.h): the whole
// state lives in registers in FLAT word order (engines.py:14-18).  The cyclic
// engines (xoroshiro, incl. the 16-word ring of xoroshiro1024, and xorshift)
// are stepped as a register ring whose offset is a compile-time constant
// inside fully unrolled chunks of a multiple of k steps, so the reference's
// ring pointer (generators.py:260-274) costs nothing at run time.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <type_traits>

#include "../../include/slp_b200.h"
#include "slp_ops.h"
#include "slp_registry.h"

namespace slp {
namespace dev {

template <int W>
struct WordOf;
template <>
struct WordOf<64> {
  using type = uint64_t;
};
template <>
struct WordOf<32> {
  using type = uint32_t;
};

// PTX wide multiply-adds: ptxas keeps these on the FMA pipe (IMAD.WIDE.U32 /
// IMAD), even for power-of-two multipliers, which is how shifts and rotations
// are moved off the ALU pipe below.
__device__ __forceinline__ uint64_t mulw(uint32_t a, uint32_t b) {
  uint64_t d;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint64_t madw(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint32_t madlo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Word operations.  64-bit words are manipulated as explicit 32-bit halves.
// The generators are integer-issue bound on the ALU pipe (LOP3/SHF/IADD3,
// profiles/).  Measured on sm_100 (profiles/int_peak.cu): LOP3, SHF and IMAD
// issue at 2 per SM per cycle, IMAD.HI at 1, IMAD.WIDE at 0.5.  Hence:
//   rotl   : two funnel shifts (SHF.L.W)                 -> 2 ALU  (default)
//   rotl_f : three wide multiply-adds by 2^r             -> 3 FMA  (A/B only:
//            Gen::best_mask with SLP_ROT_POLICY=1 loses to IMAD.WIDE's rate)
//   shl    : IMAD.SHL (low half) + SHF.L.U64.HI          -> 1 FMA + 1 ALU
//   mulc   : IMAD.WIDE + IMAD (+ IMAD for a 64-bit constant).
// Pipe-overlap mixes in the same file (round 2): only PLAIN IMADs (IMAD,
// IMAD.SHL, IMAD.IADD, IMAD.X) run beside ALU instructions; IMAD.HI and
// IMAD.WIDE add ~0.5-0.65 / ~1.75 SM cycles per warp instruction to the ALU
// pipe's time.  Hence the *_h forms below (IMAD.HI carries) only pay where
// they replace an IMAD.WIDE (mulc_h), never where they replace one SHF
// (rotl_h, shl_h: A/B knobs only); add_x (IADD3 + IMAD.X) always pays in
// ALU-bound kernels.  See profiles/round2_ab_fused_sites.md.
#ifndef SLP_ROTH_FORM
#define SLP_ROTH_FORM 0  // rotl_h low halves: 1 constant shifts + mad.hi, 0 mul.hi + mad.lo by an opaque 2^r
#endif
#ifndef SLP_MUL_POLICY
#define SLP_MUL_POLICY 1  // 0: shifts via IMAD.WIDE; 1: 64-bit constant shifts as IMAD.SHL + SHF; 2: also x*(2^a+1) as LEA pairs
#endif

template <int W>
struct WOps;

template <>
struct WOps<32> {
  using word = uint32_t;
  template <int R>
  static __device__ __forceinline__ word rotl(word x) {
    return __funnelshift_l(x, x, R);
  }
  template <int R>
  static __device__ __forceinline__ word rotl_f(word x) {
    return __funnelshift_l(x, x, R);  // no cheaper FMA form for one 32-bit word
  }
  template <int R>
  static __device__ __forceinline__ word rotl_h(word x, uint32_t, uint32_t) {
    return __funnelshift_l(x, x, R);
  }
  template <int B>
  static __device__ __forceinline__ word shl(word x) {
    return x << B;
  }
  template <int B>
  static __device__ __forceinline__ word shr(word x) {
    return x >> B;
  }
  template <unsigned long long C>
  static __device__ __forceinline__ word mulc(word x) {
    return x * (uint32_t)C;
  }
  template <int B>
  static __device__ __forceinline__ word shl_h(word x, uint32_t) {
    return x << B;
  }
  static __device__ __forceinline__ word add_x(word a, word b, uint32_t) { return a + b; }
  template <unsigned long long C>
  static __device__ __forceinline__ word mulc_h(word x, uint32_t) {
    return x * (uint32_t)C;
  }
};

template <>
struct WOps<64> {
  using word = uint64_t;
  static __device__ __forceinline__ uint32_t lo(word x) { return (uint32_t)x; }
  static __device__ __forceinline__ uint32_t hi(word x) { return (uint32_t)(x >> 32); }
  static __device__ __forceinline__ word pack(uint32_t l, uint32_t h) { return ((uint64_t)h << 32) | l; }
  template <int R>
  static __device__ __forceinline__ word rotl(word x) {
    uint32_t l = lo(x), h = hi(x);
    if constexpr (R >= 32) {
      const uint32_t t = l;
      l = h;
      h = t;
    }
    constexpr int r = R & 31;
    if constexpr (r == 0) return pack(l, h);
    return pack(__funnelshift_l(h, l, r), __funnelshift_l(l, h, r));
  }
  template <int R>
  static __device__ __forceinline__ word rotl_f(word x) {
    uint32_t l = lo(x), h = hi(x);
    if constexpr (R >= 32) {
      const uint32_t t = l;
      l = h;
      h = t;
    }
    constexpr int r = R & 31;
    if constexpr (r == 0) return pack(l, h);
    constexpr uint32_t m = 1u << r;
    const uint64_t w1 = mulw(l, m);                          // (l << r, l >> (32 - r))
    const uint64_t w2 = madw(h, m, w1 >> 32);                // low: (h << r) | (l >> (32 - r))
    const uint64_t w3 = madw(l, m, w2 >> 32);                // low: (l << r) | (h >> (32 - r))
    return pack((uint32_t)w3, (uint32_t)w2);
  }
  // rotation with its cross-word halves on the FMA pipe: with m = 2^(R mod 32)
  // in a register ptxas cannot see through (Gen::one2), lo' = hi(h*m) +
  // (l << r) and hi' = hi(l*m) + (h << r) (disjoint bits): two IMAD.HI (half
  // the ALU rate, profiles/int_peak.cu) plus two constant shifts (SHF or
  // IMAD.SHL, ptxas's choice) instead of two SHF.L.W on the saturated ALU
  // pipe.  (Low products as mul.lo by an opaque m2, SLP_ROTH_FORM=0, made
  // ptxas fuse lo(l*m) with hi(l*m) into a quarter-rate IMAD.WIDE.)
  template <int R>
  static __device__ __forceinline__ word rotl_h(word x, uint32_t m, uint32_t m2) {
    uint32_t l = lo(x), h = hi(x);
    if constexpr (R >= 32) {
      const uint32_t t = l;
      l = h;
      h = t;
    }
    if constexpr ((R & 31) == 0) return pack(l, h);
    constexpr int r = R & 31;
#if SLP_ROTH_FORM == 1
    // constant shifts (SHF or IMAD.SHL, ptxas's choice) + mad.hi: the SASS
    // IMAD.HI addend is a 64-bit pair, so each mad.hi also costs an IMAD.MOV
    const uint32_t ll = l << r, hl = h << r;
    (void)m2;
    uint32_t nl, nh;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(nl) : "r"(h), "r"(m), "r"(ll));
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(nh) : "r"(l), "r"(m), "r"(hl));
#else
    // FMA pipe only: IMAD.HI (no addend) + IMAD by a second opaque 2^r
    uint32_t ch, cl;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(ch) : "r"(h), "r"(m));
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(cl) : "r"(l), "r"(m));
    const uint32_t nl = madlo(l, m2, ch), nh = madlo(h, m2, cl);
#endif
    return pack(nl, nh);
  }
  template <int B>
  static __device__ __forceinline__ word shl(word x) {
#if SLP_MUL_POLICY >= 1
    // IMAD.SHL (lo) + SHF.L.U64.HI (hi): IMAD.WIDE issues at a quarter of the
    // IMAD rate on sm_100 (profiles/int_peak.cu)
    return x << B;
#else
    if constexpr (B >= 32) return pack(0u, lo(x) << (B - 32));
    const uint64_t w = mulw(lo(x), 1u << B);
    return pack((uint32_t)w, madlo(hi(x), 1u << B, (uint32_t)(w >> 32)));
#endif
  }
  template <int B>
  static __device__ __forceinline__ word shr(word x) {
    if constexpr (B >= 32) return pack(hi(x) >> (B - 32), 0u);
    return pack(__funnelshift_r(lo(x), hi(x), B), hi(x) >> B);
  }
  template <unsigned long long C>
  static __device__ __forceinline__ word mulc(word x) {
#if SLP_MUL_POLICY == 2
    // 2^a + 1 (the ** constants 5 and 9): x + (x << a) = LEA + LEA.HI.X, which
    // issue at up to twice the single-pipe rate, instead of IMAD.WIDE + IMAD
    constexpr int a = (C > 1 && ((C - 1) & (C - 2)) == 0) ? __builtin_ctzll(C - 1) : -1;
    if constexpr (a > 0 && a < 32) return x + (x << a);
#endif
    const uint64_t p = mulw(lo(x), (uint32_t)C);
    uint32_t h = madlo(hi(x), (uint32_t)C, (uint32_t)(p >> 32));
    if constexpr ((C >> 32) != 0) h = madlo(lo(x), (uint32_t)(C >> 32), h);
    return pack((uint32_t)p, h);
  }
  // FMA-pipe forms for kernels whose ALU pipe is the bound (K4).  The carry
  // into the high word is hi32(lo * m) with m in a register ptxas cannot see
  // through: one half-rate IMAD.HI (no addend: SASS IMAD.HI adds a 64-bit
  // register pair, so a PTX mad.hi addend costs a MOV) where shl spends an ALU
  // SHF.L.U64.HI and mulc a quarter-rate IMAD.WIDE.  The halves are split
  // with mov.b64 so that NVVM does not re-combine (x >> 32) << B into a
  // 64-bit shift plus mask.
  static __device__ __forceinline__ void split(word x, uint32_t &l, uint32_t &h) {
    asm("mov.b64 {%0, %1}, %2;" : "=r"(l), "=r"(h) : "l"(x));
  }
  static __device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
  }
  // 64-bit add with the high word on the FMA pipe: IADD3 (carry out) +
  // IMAD.X (hi(a) * one + hi(b) + carry; `one` opaque so it stays an IMAD)
  // instead of IADD3 + IADD3.X.  Plain IMADs run beside ALU instructions
  // (profiles/int_peak.cu mixes), so the add costs one ALU slot, not two.
  static __device__ __forceinline__ word add_x(word a, word b, uint32_t one) {
    uint32_t l, h;
    asm("add.cc.u32 %0, %2, %4;\n\tmadc.lo.u32 %1, %3, %6, %5;"
        : "=r"(l), "=r"(h)
        : "r"(lo(a)), "r"(hi(a)), "r"(lo(b)), "r"(hi(b)), "r"(one));
    return pack(l, h);
  }
  template <int B>
  static __device__ __forceinline__ word shl_h(word x, uint32_t m /* opaque 2^B */) {
    if constexpr (B >= 32) return pack(0u, lo(x) << (B - 32));
    uint32_t l, h;
    split(x, l, h);
    return pack(l << B, madlo(h, m, mulhi(l, m)));
  }
  template <unsigned long long C>
  static __device__ __forceinline__ word mulc_h(word x, uint32_t cq /* opaque (uint32_t)C */) {
    uint32_t l, h;
    split(x, l, h);
    uint32_t nh = madlo(h, (uint32_t)C, mulhi(l, cq));
    if constexpr ((C >> 32) != 0) nh = madlo(l, (uint32_t)(C >> 32), nh);
    return pack(l * (uint32_t)C, nh);
  }
};

// Build-time policy switches (A/B experiments, profiles/): rotation pipe
// balancing and the fused accumulator form.
#ifndef SLP_ROT_POLICY
// what Gen::best_mask proposes for the rotation sites: 0: all rotations on
// the ALU; 1: 3-IMAD.WIDE rotations (rotl_f; A/B: slower); 2: IMAD + IMAD.HI
// rotations (rotl_h; A/B: slower).  A site mask forced by a kernel
// (SLP_FUSED_MASK / SLP_FILL_MASK, fused_site_mask, fill_site_mask) uses
// rotl_h for its rotation bits unless the policy is 1.
#define SLP_ROT_POLICY 0
#endif
#ifndef SLP_SUM_POLICY
#define SLP_SUM_POLICY 3  // 0: 128-bit carry chain per output; 1, 2: IMAD.WIDE accumulators; 3: half sums
#endif

// Pipe cost of one output, in warp instructions per 32 outputs
struct PipeCost {
  int alu, fma;
};

template <int ID, int FAM, int K, int W, int A, int B, int C, int SC, int WI, int WJ, unsigned long long S_, int R_,
          unsigned long long T_>
struct Gen {
  static constexpr int id = ID;  // registry id (slp_registry.h)
  using word = typename WordOf<W>::type;
  using O = WOps<W>;
  static constexpr int k = K;
  static constexpr int w = W;
  static constexpr int n = K * W;
  static constexpr int pw = n / 64;  // u64 words per jump polynomial (degree < n)
  static constexpr bool ring = FAM != SLP_FAM_XOSHIRO;
  static constexpr int sc = SC;
  static constexpr int fam = FAM;
  static constexpr bool runtime = false;
  // kernels call the generator through an object (`eng.step(...)`) so that
  // the same code serves GenR<> below, whose parameters are run-time values;
  // Gen<> only carries the opaque 1 that the FMA-pipe rotations multiply by
  uint32_t one, one2;
  static __device__ __forceinline__ Gen load(const GenRt &rt) {
    Gen g;
    g.one = rt.one;
    g.one2 = rt.one2;
    return g;
  }

  // Rotation sites that may run on either pipe (bit set in a mask = FMA form):
  //   bit 0: engine rotation by A (xoroshiro) / by B (xoshiro)
  //   bit 1: engine rotation by C (xoroshiro)
  //   bit 2: scrambler rotation by R (++ and **)
  //   bit 3: the engine's constant left shift (high word through IMAD.HI)
  //   bit 4: scrambler multiplies (* and **; high word through IMAD.HI)
  //   bit 5: scrambler additions (+ and ++; high word as IMAD.X)
  static constexpr int kSites = (W == 64 ? ((FAM == SLP_FAM_XOROSHIRO ? 3 : (FAM == SLP_FAM_XOSHIRO ? 1 : 0)) |
                                            ((SC == SLP_SC_PLUSPLUS || SC == SLP_SC_STARSTAR) ? 4 : 0) | 8 |
                                            ((SC == SLP_SC_STAR || SC == SLP_SC_STARSTAR) ? 16 : 0) |
                                            ((SC == SLP_SC_PLUS || SC == SLP_SC_PLUSPLUS) ? 32 : 0))
                                         : 0);

  // ALU/FMA instructions per output outside the rotation sites (SASS counts, profiles/)
  static __host__ __device__ constexpr PipeCost fixed() {
    PipeCost c{0, 0};
    const int h = W == 64 ? 2 : 1;  // 32-bit halves per word
    if (FAM == SLP_FAM_XOROSHIRO) {
      c.alu += 2 * h;               // xl = s[l] ^ s0; new = rot ^ xl ^ shl (3-input LOP3)
      c.fma += W == 64 ? 2 : 1;     // xl << B
    } else if (FAM == SLP_FAM_XORSHIFT) {
      c.alu += 5 * h;
      c.fma += 2;
    } else {
      c.alu += (K == 4 ? 4 : 7) * h;  // the xor network (LOP3 fuses pairs)
      c.fma += W == 64 ? 2 : 1;       // t = s1 << A
    }
    if (W == 32) c.alu += FAM == SLP_FAM_XOROSHIRO ? 2 : 1;  // 32-bit rotations always on the ALU
    if (SC == SLP_SC_PLUS) c.alu += h;
    if (SC == SLP_SC_STAR) c.fma += W == 64 ? ((S_ >> 32) ? 3 : 2) : 1;
    if (SC == SLP_SC_PLUSPLUS) c.alu += 2 * h + (W == 32 ? 1 : 0);
    if (SC == SLP_SC_STARSTAR) c.fma += W == 64 ? 4 : 2, c.alu += W == 32 ? 1 : 0;
    return c;
  }
  // best rotation mask given extra per-output work of the calling kernel
  static __host__ __device__ constexpr int best_mask(int extra_alu, int extra_fma) {
    if (SLP_ROT_POLICY == 0) return 0;
    const PipeCost f = fixed();
    int best = 0, best_cost = 1 << 30;
    for (int m = 0; m < 8; ++m) {
      if ((m & ~kSites) != 0) continue;
      int alu = f.alu + extra_alu, fma = f.fma + extra_fma;
      int fma_hi = 0;  // IMAD.HI: half rate on the FMA pipe
      for (int bit = 0; bit < 3; ++bit) {
        if (!(kSites & (1 << bit))) continue;
        if (!(m & (1 << bit)))
          alu += 2;
        else if (SLP_ROT_POLICY == 2)
          fma += 2, fma_hi += 2;  // rotl_h: 2 IMAD + 2 IMAD.HI
        else
          fma += 3;  // rotl_f: 3 IMAD.WIDE (counted as IMAD; measured slower)
      }
      // cycles x 2 per SM: ALU and FMA pipes at 2 warp-inst/clk, dispatch at 4
      const int c_alu = 2 * alu, c_fma = 2 * (fma + 2 * fma_hi), c_disp = alu + fma + fma_hi;
      const int cost = c_alu > c_fma ? (c_alu > c_disp ? c_alu : c_disp) : (c_fma > c_disp ? c_fma : c_disp);
      if (cost < best_cost) {
        best_cost = cost;
        best = m;
      }
    }
    return best;
  }

  template <int M, int RR>
  __device__ __forceinline__ word rot(word x) const {
    if constexpr (M != 0 && SLP_ROT_POLICY == 1)
      return O::template rotl_f<RR>(x);
    else if constexpr (M != 0)
      return O::template rotl_h<RR>(x, one << (RR & 31), one2 << (RR & 31));
    else
      return O::template rotl<RR>(x);
  }
  // constant shift / multiply sites (mask bits 8 and 16 = FMA-pipe form)
  template <int M, int BB>
  __device__ __forceinline__ word shl(word x) const {
    if constexpr (M != 0)
      return O::template shl_h<BB>(x, one << (BB & 31));
    else
      return O::template shl<BB>(x);
  }
  template <int M>
  __device__ __forceinline__ word add(word a, word b) const {
    if constexpr (M != 0)
      return O::add_x(a, b, one);
    else
      return (word)(a + b);
  }
  template <int M, unsigned long long CC>
  __device__ __forceinline__ word mulc(word x) const {
    if constexpr (M != 0)
      return O::template mulc_h<CC>(x, one2 * (uint32_t)CC);
    else
      return O::template mulc<CC>(x);
  }

  // register slot of flat word j when the ring offset is o (constant after unrolling)
  static __device__ __forceinline__ constexpr int slot(int o, int j) { return ring ? (o + j) % K : j; }

  // scramblers.py:84-95, applied to the current (pre-step) state
  template <int M>
  __device__ __forceinline__ word output_m(const word (&s)[K], int o) const {
    const word xi = s[slot(o, WI)];
    if constexpr (SC == SLP_SC_NONE) {
      return xi;
    } else if constexpr (SC == SLP_SC_PLUS) {
      return add<M & 32>(xi, s[slot(o, WJ)]);
    } else if constexpr (SC == SLP_SC_STAR) {
      return mulc<M & 16, S_>(xi);
    } else if constexpr (SC == SLP_SC_PLUSPLUS) {
      return add<M & 32>(rot<M & 4, R_>(add<M & 32>(xi, s[slot(o, WJ)])), xi);
    } else {
      return mulc<M & 16, T_>(rot<M & 4, R_>(mulc<M & 16, S_>(xi)));
    }
  }

  // one engine step in the flat view (engines.py:100-140).  For ring engines
  // the flat view moves by one slot: the caller's next offset is o + 1.
  template <int M>
  __device__ __forceinline__ void step_m(word (&s)[K], int o) const {
    if constexpr (FAM == SLP_FAM_XOROSHIRO) {
      const int i0 = slot(o, 0), il = slot(o, K - 1);
      const word x0 = s[i0];
      const word xl = s[il] ^ x0;
      s[il] = rot<M & 1, A>(x0) ^ xl ^ shl<M & 8, B>(xl);
      s[i0] = rot<M & 2, C>(xl);
    } else if constexpr (FAM == SLP_FAM_XORSHIFT) {
      const int i0 = slot(o, 0), i1 = slot(o, 1);
      const word s0 = s[i0], s1 = s[i1];
      const word t = s0 ^ shl<M & 8, A>(s0);
      s[i0] = t ^ O::template shr<B>(t) ^ s1 ^ O::template shr<C>(s1);
    } else if constexpr (K == 4) {
      const word t = shl<M & 8, A>(s[1]);
      s[2] ^= s[0];
      s[3] ^= s[1];
      s[1] ^= s[2];
      s[0] ^= s[3];
      s[2] ^= t;
      s[3] = rot<M & 1, B>(s[3]);
    } else {
      const word t = shl<M & 8, A>(s[1]);
      s[2] ^= s[0];
      s[5] ^= s[1];
      s[1] ^= s[2];
      s[7] ^= s[3];
      s[3] ^= s[4];
      s[4] ^= s[5];
      s[0] ^= s[6];
      s[6] ^= s[7];
      s[6] ^= t;
      s[7] = rot<M & 1, B>(s[7]);
    }
  }

  // defaults (all-ALU rotations): jump kernel and tails
  __device__ __forceinline__ word output(const word (&s)[K], int o) const { return output_m<0>(s, o); }
  __device__ __forceinline__ void step(word (&s)[K], int o) const { step_m<0>(s, o); }

  // one output + step, registers left in flat order (tails of odd length)
  __device__ __forceinline__ word next_flat(word (&s)[K]) const {
    const word out = output(s, 0);
    step(s, 0);
    if constexpr (ring) {
      const word first = s[0];
#pragma unroll
      for (int j = 0; j + 1 < K; ++j) s[j] = s[j + 1];
      s[K - 1] = first;
    }
    return out;
  }
};

// ---- run-time parameter generators (custom_spec engines) ---------------------
//
// The reference accepts any engine built with custom_spec
// (generators.py:127-135) in LanedStream / output_stream / VecStepper
// (generators.py:426-513, engines.py:276-361).  GenR<FAM, K, W> is one kernel
// instance per engine SHAPE (family, k, w): shift/rotation amounts,
// scrambler kind, word indices and multipliers are loaded once per thread
// from the launch parameters (GenRt) into registers.  Same state layout,
// ring handling and statement order as Gen<>; rotations and shifts take a
// register amount (SHF with a variable shift), word selection is a
// warp-uniform select chain instead of a register index (which would spill
// the state to local memory).
template <int FAM, int K, int W>
struct GenR {
  static constexpr int id = -1;  // no tuned fill configuration: the default one
  using word = typename WordOf<W>::type;
  static constexpr int k = K;
  static constexpr int w = W;
  static constexpr int n = K * W;
  static constexpr int pw = n / 64;
  static constexpr bool ring = FAM != SLP_FAM_XOSHIRO;
  static constexpr int fam = FAM;
  static constexpr bool runtime = true;
  static_assert(n % 64 == 0, "state size must be a whole number of 64-bit words");

  uint32_t a, b, c, r;
  int sc, wi, wj;
  word S, T;

  static __device__ __forceinline__ GenR load(const GenRt &p) {
    GenR g;
    g.a = p.a;
    g.b = p.b;
    g.c = p.c;
    g.r = p.R;
    g.sc = p.sc;
    g.wi = p.wi;
    g.wj = p.wj < 0 ? 0 : p.wj;
    g.S = (word)p.S;
    g.T = (word)p.T;
    return g;
  }
  static constexpr int kSites = 0;  // run-time parameters: every site in its ALU form
  static __host__ __device__ constexpr int best_mask(int, int) { return 0; }
  static __device__ __forceinline__ constexpr int slot(int o, int j) { return ring ? (o + j) % K : j; }

  static __device__ __forceinline__ word rotl(word x, uint32_t s) {
    if constexpr (W == 32) {
      return __funnelshift_l(x, x, s);
    } else {
      uint32_t l = (uint32_t)x, h = (uint32_t)(x >> 32);
      if (s & 32) {
        const uint32_t t = l;
        l = h;
        h = t;
      }
      return ((uint64_t)__funnelshift_l(l, h, s) << 32) | __funnelshift_l(h, l, s);
    }
  }
  // flat word j at ring offset o; j is a run-time value
  __device__ __forceinline__ word pick(const word (&s)[K], int o, int j) const {
    word v = s[slot(o, 0)];
#pragma unroll
    for (int i = 1; i < K; ++i) v = j == i ? s[slot(o, i)] : v;
    return v;
  }

  template <int M>
  __device__ __forceinline__ word output_m(const word (&s)[K], int o) const {
    const word xi = pick(s, o, wi);
    switch (sc) {
      case SLP_SC_PLUS: return (word)(xi + pick(s, o, wj));
      case SLP_SC_STAR: return (word)(xi * S);
      case SLP_SC_PLUSPLUS: return (word)(rotl((word)(xi + pick(s, o, wj)), r) + xi);
      case SLP_SC_STARSTAR: return (word)(rotl((word)(xi * S), r) * T);
      default: return xi;
    }
  }
  template <int M>
  __device__ __forceinline__ void step_m(word (&s)[K], int o) const {
    if constexpr (FAM == SLP_FAM_XOROSHIRO) {
      const int i0 = slot(o, 0), il = slot(o, K - 1);
      const word x0 = s[i0];
      const word xl = s[il] ^ x0;
      s[il] = rotl(x0, a) ^ xl ^ (word)(xl << b);
      s[i0] = rotl(xl, c);
    } else if constexpr (FAM == SLP_FAM_XORSHIFT) {
      const int i0 = slot(o, 0), i1 = slot(o, 1);
      const word s0 = s[i0], s1 = s[i1];
      const word t = s0 ^ (word)(s0 << a);
      s[i0] = t ^ (t >> b) ^ s1 ^ (s1 >> c);
    } else if constexpr (K == 4) {
      const word t = (word)(s[1] << a);
      s[2] ^= s[0];
      s[3] ^= s[1];
      s[1] ^= s[2];
      s[0] ^= s[3];
      s[2] ^= t;
      s[3] = rotl(s[3], b);
    } else {
      const word t = (word)(s[1] << a);
      s[2] ^= s[0];
      s[5] ^= s[1];
      s[1] ^= s[2];
      s[7] ^= s[3];
      s[3] ^= s[4];
      s[4] ^= s[5];
      s[0] ^= s[6];
      s[6] ^= s[7];
      s[6] ^= t;
      s[7] = rotl(s[7], b);
    }
  }
  __device__ __forceinline__ word output(const word (&s)[K], int o) const { return output_m<0>(s, o); }
  __device__ __forceinline__ void step(word (&s)[K], int o) const { step_m<0>(s, o); }
  __device__ __forceinline__ word next_flat(word (&s)[K]) const {
    const word out = output(s, 0);
    step(s, 0);
    if constexpr (ring) {
      const word first = s[0];
#pragma unroll
      for (int j = 0; j + 1 < K; ++j) s[j] = s[j + 1];
      s[K - 1] = first;
    }
    return out;
  }
};

// ---- output conversion (K3) ------------------------------------------------
// bit patterns of the converted element; conversion is exact in both cases:
// x >> 11 < 2^53 and x >> 8 < 2^24 are representable, the scale is a power of 2.

template <int OK, class word>
struct Out;
template <class word>
struct Out<SLP_OUT_NATIVE, word> {
  using bits = word;
  static __device__ __forceinline__ bits conv(word x) { return x; }
};
template <class word>
struct Out<SLP_OUT_U64, word> {
  using bits = uint64_t;
  static __device__ __forceinline__ bits conv(word x) { return (uint64_t)x; }
};
template <class word>
struct Out<SLP_OUT_F64, word> {
  using bits = uint64_t;
  // (x >> 11) * 2^-53 computed as (x with its low 11 bits cleared) * 2^-64:
  // that integer has <= 53 significant bits, so the conversion and the scaling
  // are both exact and the result is bit-identical, and clearing the bits is
  // one LOP3 on the low word where the 64-bit shift was two SHF (the f64 fill
  // is ALU-bound: ncu, profiles/f64_target.py)
  static __device__ __forceinline__ bits conv(word x) {
    return (uint64_t)__double_as_longlong(__ull2double_rn((uint64_t)x & ~0x7FFull) * 0x1.0p-64);
  }
};
template <class word>
struct Out<SLP_OUT_F32, word> {
  using bits = uint32_t;
  static __device__ __forceinline__ bits conv(word x) {
    return (uint32_t)__float_as_uint(__uint2float_rn((uint32_t)x >> 8) * 0x1.0p-24f);
  }
};

// ---- PTX helpers -------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, uint32_t src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
               :
               : "l"(reinterpret_cast<uint64_t>(map)), "r"(src), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// warp index the compiler can prove warp-uniform (result of a shuffle from lane 0)
__device__ __forceinline__ int warp_uniform() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }
// one elected lane of a converged warp (elect.sync picks the same leader every time)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
// store pacing (k_fill): HBM absorbs a stream of row-piece stores at ~6.7 TB/s
// when they are offered at about that rate, but only ~6.1 TB/s when the
// offered rate exceeds it (profiles/wpattern_r3.cu, round2_wpattern_r3*.jsonl);
// a warp therefore issues its tile stores no closer than pace_ns apart on the
// global timer.  A warp that fell behind catches up by at most `burst` periods.
__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void pace_store(uint64_t &next, uint32_t pace_ns, uint32_t burst) {
  uint64_t now = global_ns();
  // sleep through most of the wait: a spinning warp takes issue slots (and
  // power) from the generating ones (~1/3 of the instructions of a paced
  // config-2 fill were this loop)
  while (now < next) {
    const uint64_t d = next - now;
    if (d > 128) __nanosleep((uint32_t)(d < 2048 ? d >> 1 : 1024));
    now = global_ns();
  }
  now = __shfl_sync(0xffffffffu, now, 0);
  // a warp more than `burst` periods behind its schedule restarts it at now
  next = (now > next + (uint64_t)burst * pace_ns ? now : next) + pace_ns;
}
// 128-bit accumulate of a 64-bit value
__device__ __forceinline__ void add128(uint64_t &lo, uint64_t &hi, uint64_t x) {
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, 0;" : "+l"(lo), "+l"(hi) : "l"(x));
}

}  // namespace dev
}  // namespace slp
