// Device templates for the scrambled linear generators on sm_100a.
//
// One template instance per registry generator (slp_registry.h): the whole
// state lives in registers in FLAT word order (engines.py:14-18).  The cyclic
// engines (xoroshiro, incl. the 16-word ring of xoroshiro1024, and xorshift)
// are stepped as a register ring whose offset is a compile-time constant
// inside fully unrolled chunks of a multiple of k steps, so the reference's
// ring pointer (generators.py:260-274) costs nothing at run time.
//
// Kernels (paths relative to /root/reference/pkg/src/slprng/):
//   K1    k_jump   state * p(M) as sum of state*M^d (generators.py:315-334, :493-505)
//   K2/K3 k_fill   scramble + step + convert + store (generators.py:244-311, :465-490)
//   K4    k_fused  scramble + step + in-register reduction (new)
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
};

// Build-time policy switches (A/B experiments, profiles/): rotation pipe
// balancing and the fused accumulator form.
#ifndef SLP_ROT_POLICY
#define SLP_ROT_POLICY 0  // 0: all rotations on the ALU; 1: Gen::best_mask (A/B: no gain, ptxas re-normalises)
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

  // Rotation sites that may run on either pipe (bit set in a mask = FMA form):
  //   bit 0: engine rotation by A (xoroshiro) / by B (xoshiro)
  //   bit 1: engine rotation by C (xoroshiro)
  //   bit 2: scrambler rotation by R (++ and **)
  static constexpr int kSites = (W == 64 ? ((FAM == SLP_FAM_XOROSHIRO ? 3 : (FAM == SLP_FAM_XOSHIRO ? 1 : 0)) |
                                            ((SC == SLP_SC_PLUSPLUS || SC == SLP_SC_STARSTAR) ? 4 : 0))
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
      for (int bit = 0; bit < 3; ++bit) {
        if (!(kSites & (1 << bit))) continue;
        if (m & (1 << bit))
          fma += 3;
        else
          alu += 2;
      }
      const int cost = (2 * alu > 2 * fma ? 2 * alu : 2 * fma) > alu + fma ? (2 * alu > 2 * fma ? 2 * alu : 2 * fma)
                                                                            : alu + fma;
      if (cost < best_cost) {
        best_cost = cost;
        best = m;
      }
    }
    return best;
  }

  template <int M, int RR>
  static __device__ __forceinline__ word rot(word x) {
    if constexpr (M != 0)
      return O::template rotl_f<RR>(x);
    else
      return O::template rotl<RR>(x);
  }

  // register slot of flat word j when the ring offset is o (constant after unrolling)
  static __device__ __forceinline__ constexpr int slot(int o, int j) { return ring ? (o + j) % K : j; }

  // scramblers.py:84-95, applied to the current (pre-step) state
  template <int M>
  static __device__ __forceinline__ word output_m(const word (&s)[K], int o) {
    const word xi = s[slot(o, WI)];
    if constexpr (SC == SLP_SC_NONE) {
      return xi;
    } else if constexpr (SC == SLP_SC_PLUS) {
      return (word)(xi + s[slot(o, WJ)]);
    } else if constexpr (SC == SLP_SC_STAR) {
      return O::template mulc<S_>(xi);
    } else if constexpr (SC == SLP_SC_PLUSPLUS) {
      return (word)(rot<M & 4, R_>((word)(xi + s[slot(o, WJ)])) + xi);
    } else {
      return O::template mulc<T_>(rot<M & 4, R_>(O::template mulc<S_>(xi)));
    }
  }

  // one engine step in the flat view (engines.py:100-140).  For ring engines
  // the flat view moves by one slot: the caller's next offset is o + 1.
  template <int M>
  static __device__ __forceinline__ void step_m(word (&s)[K], int o) {
    if constexpr (FAM == SLP_FAM_XOROSHIRO) {
      const int i0 = slot(o, 0), il = slot(o, K - 1);
      const word x0 = s[i0];
      const word xl = s[il] ^ x0;
      s[il] = rot<M & 1, A>(x0) ^ xl ^ O::template shl<B>(xl);
      s[i0] = rot<M & 2, C>(xl);
    } else if constexpr (FAM == SLP_FAM_XORSHIFT) {
      const int i0 = slot(o, 0), i1 = slot(o, 1);
      const word s0 = s[i0], s1 = s[i1];
      const word t = s0 ^ O::template shl<A>(s0);
      s[i0] = t ^ O::template shr<B>(t) ^ s1 ^ O::template shr<C>(s1);
    } else if constexpr (K == 4) {
      const word t = O::template shl<A>(s[1]);
      s[2] ^= s[0];
      s[3] ^= s[1];
      s[1] ^= s[2];
      s[0] ^= s[3];
      s[2] ^= t;
      s[3] = rot<M & 1, B>(s[3]);
    } else {
      const word t = O::template shl<A>(s[1]);
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
  static __device__ __forceinline__ word output(const word (&s)[K], int o) { return output_m<0>(s, o); }
  static __device__ __forceinline__ void step(word (&s)[K], int o) { step_m<0>(s, o); }

  // one output + step, registers left in flat order (tails of odd length)
  static __device__ __forceinline__ word next_flat(word (&s)[K]) {
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
  static __device__ __forceinline__ bits conv(word x) {
    return (uint64_t)__double_as_longlong(__ull2double_rn((uint64_t)x >> 11) * 0x1.0p-53);
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
// 128-bit accumulate of a 64-bit value
__device__ __forceinline__ void add128(uint64_t &lo, uint64_t &hi, uint64_t x) {
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, 0;" : "+l"(lo), "+l"(hi) : "l"(x));
}

// ---- K2/K3: fill ---------------------------------------------------------------
//
// A warp owns 32 consecutive substreams ("unit"); lane l keeps substream
// u*32+l in registers.  Outputs are produced in tiles of 32 substreams x
// row_bytes (= segs x 128 B, FillShape) per substream; CH = row_bytes / ES
// outputs per substream per tile.  MODE:
//   FILL_TMA     stream-major.  Every output pair goes to the warp's
//                shared-memory tile as it is produced (STS.128,
//                conflict-free under the 128B swizzle), and the full tile
//                leaves with one 3-D TMA bulk tensor store
//                (cp.async.bulk.tensor.3d, SASS UTMASTG) that writes
//                row_bytes contiguous bytes of each of the 32 rows.  The
//                row piece is >= 256 B because HBM absorbs a column sweep of
//                64/128-byte pieces at only ~4.5-4.8 TB/s (profiles/wpattern.cu).
//                With B buffers per warp, store i-B must have finished reading
//                before tile i overwrites its buffer (cp.async.bulk.wait_group.read).
//   FILL_STAGED  stream-major, same staging, element stores (any pitch/alignment);
//   FILL_POS     position-major: each output is one coalesced warp store
//                (any pitch/alignment);
//   FILL_POS_TMA position-major through the same per-warp tile, laid out
//                [position][lane]: one 2-D TMA store writes CH rows of the
//                output x 32 consecutive substreams (256 B for u64).  Direct
//                stores leave 256-byte pieces scattered over CH rows that
//                are 8 MiB apart and ran at 2.5-5.5 TB/s.
// Shared-memory tile layout [seg][row][128 B], chunk q of (seg, row) at
// ((seg*32 + row) * 128) + ((q ^ (row & 7)) << 4)  (CU_TENSOR_MAP_SWIZZLE_128B).

enum { FILL_TMA = 0, FILL_STAGED = 1, FILL_POS = 2, FILL_POS_TMA = 3 };
constexpr int kFillThreads = kFillWarps * 32;

// Fill tile configurations (slp_ops.h):
//   segs x 128 B row pieces per TMA store, bufs tile buffers per warp;
//   pre: with one buffer, the first `pre` 16-byte chunks of tile i are
//     generated into registers while the TMA store of tile i-1 still reads
//     the buffer, so the wait for it overlaps generation;
//   unroll: outputs per sub-block; the tile is generated in a rolled loop
//     of sub-blocks, because fully unrolled 1 KiB tiles of the 8- and 16-word
//     generators overflow the 32 KB L1.5 instruction cache.
struct FillCfg {
  int segs, bufs, pre, unroll;
};
// (a switch, not an array: namespace-scope constexpr arrays are host-only in CUDA)
__host__ __device__ constexpr FillCfg fill_cfg_at(int i) {
  switch (i) {
    case 1: return FillCfg{8, 1, 16, 64};
    case 2: return FillCfg{8, 1, 16, 128};
    case 3: return FillCfg{4, 2, 0, 32};  // 512 B rows, two buffers
    case 4: return FillCfg{4, 2, 0, 64};
    default: return FillCfg{8, 1, 16, 32};  // 0: 1 KiB rows, one buffer
  }
}
constexpr int kNumFillCfgs = 5;
enum { FILL_KIND_NATIVE = 0, FILL_KIND_CONVERT = 1, FILL_KIND_CHECKSUM = 2 };
}  // namespace dev
}  // namespace slp
#include "slp_fill_tuning.h"  // fill_tune(generator id, kind) -> configuration index (measured)
namespace slp {
namespace dev {

// -DSLP_FILL_CFG=i forces configuration i for every kernel (tuning builds,
// profiles/tune_fill.py)
__host__ __device__ constexpr FillCfg fill_cfg(int id, int kind) {
#ifdef SLP_FILL_CFG
  return (void)id, (void)kind, fill_cfg_at(SLP_FILL_CFG);
#else
  return fill_cfg_at(fill_tune(id, kind));
#endif
}

template <class G, int KIND>
struct FillShape {
  static constexpr FillCfg cfg = fill_cfg(G::id, KIND);
  static constexpr int segs = cfg.segs, bufs = cfg.bufs, pre = cfg.pre, unroll = cfg.unroll;
  static constexpr int row_bytes = segs * 128;
  static constexpr int tile_bytes = 32 * row_bytes;
  static constexpr int smem = kFillWarps * bufs * tile_bytes + 1024;
  static_assert(smem <= 227 * 1024, "fill tiles exceed shared memory");
};

template <int OK, bool CSUM>
__host__ __device__ constexpr int fill_kind() {
  return CSUM ? FILL_KIND_CHECKSUM : (OK == SLP_OUT_NATIVE ? FILL_KIND_NATIVE : FILL_KIND_CONVERT);
}

__host__ __device__ constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }

__device__ __forceinline__ uint32_t swz(int seg, int r, int q) { return ((seg * 32 + r) << 7) + ((q ^ (r & 7)) << 4); }

__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, uint32_t src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
               :
               : "l"(reinterpret_cast<uint64_t>(map)), "r"(src), "r"(x), "r"(y), "r"(z)
               : "memory");
}

// CSUM: also reduce the integer outputs while storing them (wrapping sum,
// xor, exact sum and low-bit sum, as k_fused) -- "store mode plus fused
// checksum" of BASELINE config 3 in one pass; partials go to p.partials.
// exact per-CTA reduction of checksum accumulators into partials[blockIdx.x]
template <int WPB>
__device__ __forceinline__ void reduce_checksum_block(uint64_t slo, uint64_t shi, uint64_t sx, uint64_t slow,
                                                      double fs, void *partials) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const uint64_t olo = __shfl_xor_sync(0xffffffffu, slo, off);
    const uint64_t ohi = __shfl_xor_sync(0xffffffffu, shi, off);
    const uint64_t nlo = slo + olo;
    shi = shi + ohi + (nlo < slo ? 1 : 0);
    slo = nlo;
    sx ^= __shfl_xor_sync(0xffffffffu, sx, off);
    slow += __shfl_xor_sync(0xffffffffu, slow, off);
    fs += __shfl_xor_sync(0xffffffffu, fs, off);
  }
  __shared__ uint64_t r_lo[WPB], r_hi[WPB], r_x[WPB], r_low[WPB];
  __shared__ double r_fs[WPB];
  if (lane == 0) {
    r_lo[warp] = slo;
    r_hi[warp] = shi;
    r_x[warp] = sx;
    r_low[warp] = slow;
    r_fs[warp] = fs;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t lo = 0, hi = 0, x = 0, low = 0;
    double f = 0.0;
    for (int i = 0; i < WPB; ++i) {
      const uint64_t nlo = lo + r_lo[i];
      hi += r_hi[i] + (nlo < lo ? 1 : 0);
      lo = nlo;
      x ^= r_x[i];
      low += r_low[i];
      f += r_fs[i];
    }
    slp_checksum *part = static_cast<slp_checksum *>(partials) + blockIdx.x;
    part->sum_lo = lo;
    part->sum_hi = hi;
    part->xor_all = x;
    part->low_sum = low;
    part->count = 0;
    part->fsum = f;
  }
}

template <class G, int OK, int MODE, bool CSUM = false>
__global__ void __launch_bounds__(kFillThreads) k_fill(FillParams p, const __grid_constant__ CUtensorMap tmap) {
  using word = typename G::word;
  using Cv = Out<OK, word>;
  using bits = typename Cv::bits;
  constexpr int K = G::k;
  constexpr int ES = sizeof(bits);
  using Shape = FillShape<G, fill_kind<OK, CSUM>()>;
  constexpr int kFillBufs = Shape::bufs, kSegs = Shape::segs, kTileBytes = Shape::tile_bytes;
  constexpr int CH = Shape::row_bytes / ES;                       // outputs per substream per tile
  constexpr int EPC = 16 / ES;                                    // elements per 16-byte chunk
  constexpr int U = Shape::unroll < CH ? Shape::unroll : CH;       // outputs per sub-block
  static_assert(CH % U == 0 && U % EPC == 0 && (U * ES) % 128 == 0, "sub-blocks must be whole 128-byte segments");
  static_assert(!G::ring || U % K == 0, "sub-blocks must cover whole ring periods");
  // 16-byte chunks produced before the buffer wait (at most one sub-block)
  constexpr int PRE = MODE == FILL_POS ? 0 : (Shape::pre * EPC <= U ? Shape::pre : U / EPC);
  constexpr int MSK = G::best_mask(0, 0);  // rotation pipe mix (ALU vs FMA), see Gen::best_mask
  const int lane = threadIdx.x & 31;
  const int warp = warp_uniform();  // keeps TMA coordinates in uniform registers

  extern __shared__ uint8_t smem_raw[];
  uint32_t tiles = 0;
  if constexpr (MODE != FILL_POS)
    tiles = ((smem_u32(smem_raw) + 1023u) & ~1023u) + warp * kFillBufs * kTileBytes;  // 128B-swizzle atoms: 1 KiB

  const word *__restrict__ sin = static_cast<const word *>(p.sin);
  word *sout = static_cast<word *>(p.sout);
  bits *__restrict__ out = static_cast<bits *>(p.out);
  const uint64_t ntiles = p.T / CH;
  const uint64_t rem = p.T - ntiles * CH;
  uint32_t issued = 0;  // tiles produced by this warp
  uint64_t cs_lo = 0, cs_hi = 0, cs_x = 0, cs_low = 0;  // CSUM accumulators (zero states emit zeros)

  // the next unit's start states are loaded while this unit is generated
  // (the load latency otherwise stalls every warp at each unit start)
  const uint64_t ustride = (uint64_t)gridDim.x * kFillWarps;
  auto load_states = [&](uint64_t unit, word(&dst)[K]) {
    const uint64_t st = unit * 32 + lane;
    const bool ok = unit < p.nunits && st < p.nstreams;
#pragma unroll
    for (int j = 0; j < K; ++j) dst[j] = ok ? sin[j * p.ld + st] : (word)0;
  };
  word nxt[K];
  load_states((uint64_t)blockIdx.x * kFillWarps + warp, nxt);
  for (uint64_t u = (uint64_t)blockIdx.x * kFillWarps + warp; u < p.nunits; u += ustride) {
    const uint64_t row0 = u * 32;
    const uint64_t stream = row0 + lane;
    const bool valid = stream < p.nstreams;
    word s[K];
#pragma unroll
    for (int j = 0; j < K; ++j) s[j] = nxt[j];
    load_states(u + ustride, nxt);

    for (uint64_t c = 0; c < ntiles; ++c) {
      const uint64_t pos0 = c * CH;
      uint32_t tile = 0;
      auto wait_buffer = [&] {
        if constexpr (MODE == FILL_TMA || MODE == FILL_POS_TMA) {
          if (issued >= kFillBufs && elect_one()) bulk_wait_read<kFillBufs - 1>();
        }
        __syncwarp();
      };
      // one 16-byte chunk (outputs b+e .. b+e+EPC-1 of this lane's row) into the
      // tile; b (runtime) is a sub-block start, e (compile time) the offset in it
      auto put = [&](uint32_t b, int e, const bits(&v)[EPC]) {
        if constexpr (MODE == FILL_POS_TMA) {  // tile [position][lane]
          const uint32_t row = tile + (b * 32 + lane) * ES;
#pragma unroll
          for (int i = 0; i < EPC; ++i) {
            const uint32_t addr = row + (e + i) * 32 * ES;
            if constexpr (ES == 8)
              asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"((uint64_t)v[i]) : "memory");
            else
              asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"((uint32_t)v[i]) : "memory");
          }
          return;
        }
        const int byte = e * ES;
        const uint32_t addr = tile + ((b * ES / 128) << 12) + swz(byte >> 7, lane, (byte & 127) >> 4);
        if constexpr (ES == 8) {
          asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(addr), "l"((uint64_t)v[0]), "l"((uint64_t)v[1])
                       : "memory");
        } else {
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"((uint32_t)v[0]),
                       "r"((uint32_t)v[1]), "r"((uint32_t)v[2]), "r"((uint32_t)v[3])
                       : "memory");
        }
      };
      // EPC outputs at sub-block offset e (ring offset (e + i) % K is static since U % K == 0)
      // CSUM, per tile: sums of the 32-bit halves (exact in 64 bits), xor and
      // low-bit sum, one chunk at a time (3-input adds / LOP3 over the chunk)
      uint64_t t_lo = 0, t_hi = 0;
      word t_x = 0;
      uint32_t t_low = 0;
      auto gen = [&](int e, bits(&v)[EPC]) {
        word rr[EPC];
#pragma unroll
        for (int i = 0; i < EPC; ++i) {
          const int o = (e + i) % K;
          rr[i] = G::template output_m<MSK>(s, o);
          v[i] = Cv::conv(rr[i]);
          G::template step_m<MSK>(s, o);
        }
        if constexpr (CSUM) {
          constexpr uint32_t LOWM = G::w == 64 ? 0x7FFu : 0xFFu;
          word x = rr[0];
          uint32_t lw = (uint32_t)rr[0] & LOWM;
          uint64_t slo = (uint32_t)rr[0], shi = (uint64_t)rr[0] >> 32;
#pragma unroll
          for (int i = 1; i < EPC; ++i) {
            x ^= rr[i];
            lw += (uint32_t)rr[i] & LOWM;
            slo += (uint32_t)rr[i];
            shi += (uint64_t)rr[i] >> 32;
          }
          t_x ^= x;
          t_low += lw;
          t_lo += slo;
          if constexpr (G::w == 64) t_hi += shi;
        }
      };
      auto emit = [&](uint32_t b, int e, const bits(&v)[EPC]) {
        if constexpr (MODE == FILL_POS) {
          if (valid) {
#pragma unroll
            for (int i = 0; i < EPC; ++i) out[(pos0 + b + e + i) * p.ld_out + stream] = v[i];
          }
        } else {
          put(b, e, v);
        }
      };
      if constexpr (MODE != FILL_POS) {
        tile = tiles + (issued % kFillBufs) * kTileBytes;
        if constexpr (PRE == 0) wait_buffer();
      }
      // sub-block 0, peeled: its first PRE chunks are produced while the
      // buffer's previous TMA store is still reading it
      bits hold[PRE > 0 ? PRE : 1][EPC];
#pragma unroll
      for (int e = 0; e < U; e += EPC) {
        bits v[EPC];
        gen(e, v);
        if (e < PRE * EPC) {
#pragma unroll
          for (int i = 0; i < EPC; ++i) hold[e / EPC][i] = v[i];
          if (e == (PRE - 1) * EPC) {
            wait_buffer();
#pragma unroll
            for (int q = 0; q < PRE; ++q) put(0, q * EPC, hold[q]);
          }
        } else {
          emit(0, e, v);
        }
      }
      // remaining sub-blocks: a rolled loop keeps the body within the
      // instruction cache (a fully unrolled 1 KiB-row tile of an 8-word
      // generator is ~60 KB of SASS, twice the 32 KB L1.5 I-cache)
#pragma unroll 1
      for (uint32_t b = U; b < (uint32_t)CH; b += U) {
#pragma unroll
        for (int e = 0; e < U; e += EPC) {
          bits v[EPC];
          gen(e, v);
          emit(b, e, v);
        }
      }
      if constexpr (CSUM) {
        add128(cs_lo, cs_hi, t_lo);
        add128(cs_lo, cs_hi, t_hi << 32);
        cs_hi += t_hi >> 32;
        cs_x ^= (uint64_t)t_x;
        cs_low += t_low;
      }
      if constexpr (MODE == FILL_TMA) {
        fence_proxy_async_smem();
        __syncwarp();
        if (elect_one()) {
          tma_store_3d(&tmap, tile, 0, (int)row0, (int)(pos0 * ES / 128));
          bulk_commit();
        }
        ++issued;
      } else if constexpr (MODE == FILL_POS_TMA) {
        fence_proxy_async_smem();
        __syncwarp();
        if (elect_one()) {
          tma_store_2d(&tmap, tile, (int)row0, (int)pos0);
          bulk_commit();
        }
        ++issued;
      } else if constexpr (MODE == FILL_STAGED) {
        __syncwarp();
        // element stores; CPR lanes cover one 128-byte segment of a row
        constexpr int CPR = 128 / ES;  // elements per segment
        constexpr int RPP = 32 / CPR;  // rows per pass (1 for u32, 2 for u64)
#pragma unroll 4
        for (int r0 = 0; r0 < 32 * kSegs; r0 += RPP) {
          const int rs = r0 + lane / CPR;  // (seg, row) flattened seg-major
          const int seg = rs / 32, r = rs % 32;
          const int e = lane % CPR;
          const uint64_t srow = row0 + r;
          bits v;
          const uint32_t addr = tile + swz(seg, r, (e * ES) >> 4) + (e * ES & 15);
          if constexpr (ES == 8) {
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
          } else {
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
          }
          if (srow < p.nstreams) out[srow * p.ld_out + pos0 + seg * CPR + e] = v;
        }
        __syncwarp();
        ++issued;
      }
    }
    for (uint64_t t = 0; t < rem; ++t) {
      const word r = G::next_flat(s);
      const bits x = Cv::conv(r);
      if constexpr (CSUM) {
        add128(cs_lo, cs_hi, (uint64_t)r);
        cs_x ^= (uint64_t)r;
        cs_low += (uint32_t)r & (G::w == 64 ? 0x7FFu : 0xFFu);
      }
      if (valid) {
        const uint64_t pos = ntiles * CH + t;
        if constexpr (MODE == FILL_POS || MODE == FILL_POS_TMA)
          out[pos * p.ld_out + stream] = x;
        else
          out[stream * p.ld_out + pos] = x;
      }
    }
    if (valid && sout) {
#pragma unroll
      for (int j = 0; j < K; ++j) sout[j * p.ld + stream] = s[j];
    }
  }
  if constexpr (MODE == FILL_TMA || MODE == FILL_POS_TMA) {
    if (elect_one()) bulk_wait_all<0>();
  }
  if constexpr (CSUM) reduce_checksum_block<kFillWarps>(cs_lo, cs_hi, cs_x, cs_low, 0.0, p.partials);
}

// ---- K4: fused consumer ---------------------------------------------------------
//
// Per output: wrapping sum (IADD3 + IADD3.X) and xor (one LOP3 per two
// outputs).  MANT adds the exact 128-bit sum (one more IADD3.X with carry) and
// the sum of the low 11 (w=64) / 8 (w=32) bits, from which the exact sum of
// the converted doubles / floats follows: mant = (sum - low) >> shift.
// F64 adds a genuine float64 accumulation of the converted values.

constexpr int kFusedThreads = 256;

template <class G, bool MANT, bool F64>
#ifndef SLP_FUSED_MINB
#define SLP_FUSED_MINB 1
#endif
__global__ void __launch_bounds__(kFusedThreads, SLP_FUSED_MINB) k_fused(FusedParams p) {
  using word = typename G::word;
  constexpr int K = G::k;
  constexpr int CH = 16;  // multiple of every ring size
  constexpr uint32_t LOWMASK = G::w == 64 ? 0x7FFu : 0xFFu;
  constexpr int SH = G::w == 64 ? 11 : 8;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  constexpr int WPB = kFusedThreads / 32;
  const word *__restrict__ sin = static_cast<const word *>(p.sin);
  word *sout = static_cast<word *>(p.sout);
  const uint64_t nfull = p.T / CH;
  const uint64_t rem = p.T - nfull * CH;

  // Per-output accumulation runs mostly on the FMA pipe (the generator
  // itself saturates the ALU pipe): sum of the low and of the high 32-bit
  // halves in two 64-bit IMAD.WIDE accumulators (x_half * one + acc, `one`
  // is an opaque 1 from the parameters so ptxas cannot turn it into IADD3);
  // together they give the EXACT sum.  xor: one 3-input LOP3 per output pair
  // and half.  MANT: low-bit sum = LOP3 + IMAD.
  constexpr int MSK = G::best_mask(G::w == 64 ? 1 : 1, (G::w == 64 ? 2 : 1) + (MANT ? 1 : 0));
  const uint32_t one = p.one;
  uint64_t slo = 0, shi = 0, sx = 0, slow = 0;
  double fs = 0.0, fs2 = 0.0;
  for (uint64_t u = (uint64_t)blockIdx.x * WPB + warp; u < p.nunits; u += (uint64_t)gridDim.x * WPB) {
    const uint64_t stream = u * 32 + lane;
    if (stream >= p.nstreams) continue;
    word s[K];
#pragma unroll
    for (int j = 0; j < K; ++j) s[j] = sin[j * p.ld + stream];
    uint64_t acc_lo = 0, acc_hi = 0;  // sums of 32-bit halves (< 2^32 terms per substream)
    uint64_t acc_lo2 = 0, acc_hi2 = 0;
    for (uint64_t c = 0; c < nfull; ++c) {
      uint32_t lw = 0, lw2 = 0;
      word xx = 0;
#pragma unroll
      for (int t = 0; t < CH; t += 2) {
        const word o0 = G::template output_m<MSK>(s, t % K);
        G::template step_m<MSK>(s, t % K);
        const word o1 = G::template output_m<MSK>(s, (t + 1) % K);
        G::template step_m<MSK>(s, (t + 1) % K);
#if SLP_SUM_POLICY == 2
        // separate even/odd accumulators: one IMAD.WIDE per chain per pair,
        // nothing for ptxas to re-associate into IADD3
        acc_lo = madw((uint32_t)o0, one, acc_lo);
        acc_lo2 = madw((uint32_t)o1, one, acc_lo2);
        if constexpr (G::w == 64) {
          acc_hi = madw((uint32_t)((uint64_t)o0 >> 32), one, acc_hi);
          acc_hi2 = madw((uint32_t)((uint64_t)o1 >> 32), one, acc_hi2);
        }
        if constexpr (MANT) {
          lw = madlo((uint32_t)o0 & LOWMASK, one, lw);
          lw2 = madlo((uint32_t)o1 & LOWMASK, one, lw2);
        }
#elif SLP_SUM_POLICY == 1
        acc_lo = madw((uint32_t)o0, one, acc_lo);
        acc_lo = madw((uint32_t)o1, one, acc_lo);
        if constexpr (G::w == 64) {
          acc_hi = madw((uint32_t)((uint64_t)o0 >> 32), one, acc_hi);
          acc_hi = madw((uint32_t)((uint64_t)o1 >> 32), one, acc_hi);
        }
        if constexpr (MANT) {
          lw = madlo((uint32_t)o0 & LOWMASK, one, lw);
          lw = madlo((uint32_t)o1 & LOWMASK, one, lw);
        }
#elif SLP_SUM_POLICY == 3
        // exact sum as two 64-bit sums of 32-bit halves, one output pair per
        // 3-input add (IADD3 + IADD3.X per half): 2 ALU ops per output
        // instead of a 128-bit carry chain per output (4)
        if constexpr (MANT) {
          acc_lo += (uint64_t)(uint32_t)o0 + (uint32_t)o1;
          if constexpr (G::w == 64) acc_hi += ((uint64_t)o0 >> 32) + ((uint64_t)o1 >> 32);
          lw += ((uint32_t)o0 & LOWMASK) + ((uint32_t)o1 & LOWMASK);
        } else {
          slo += (uint64_t)o0 + (uint64_t)o1;
        }
#else
        if constexpr (MANT) {
          add128(slo, shi, (uint64_t)o0);
          add128(slo, shi, (uint64_t)o1);
          lw += ((uint32_t)o0 & LOWMASK) + ((uint32_t)o1 & LOWMASK);
        } else {
          slo += (uint64_t)o0 + (uint64_t)o1;
        }
#endif
        xx ^= o0 ^ o1;
        if constexpr (F64) {  // two independent chains: the DADD latency, not the pipe, bounds one chain
          fs += __ull2double_rn((uint64_t)o0 >> SH);
          fs2 += __ull2double_rn((uint64_t)o1 >> SH);
        }
      }
      sx ^= (uint64_t)xx;
      slow += (uint64_t)lw + lw2;
#if SLP_SUM_POLICY == 3
      if constexpr (MANT) {
        if ((c & ((1ull << 26) - 1)) == ((1ull << 26) - 1)) {  // every 2^30 outputs: keep the half sums < 2^64
          add128(slo, shi, acc_lo);
          add128(slo, shi, acc_hi << 32);
          shi += acc_hi >> 32;
          acc_lo = acc_hi = 0;
        }
      }
#endif
    }
    for (uint64_t t = 0; t < rem; ++t) {
      const word x = G::next_flat(s);
      acc_lo += (uint32_t)x;
      if constexpr (G::w == 64) acc_hi += (uint32_t)((uint64_t)x >> 32);
      sx ^= (uint64_t)x;
      slow += (uint32_t)x & LOWMASK;
      if constexpr (F64) fs += __ull2double_rn((uint64_t)x >> SH);
    }
    // fold this substream's exact sum acc_lo + acc_hi * 2^32 into the 128-bit total
    add128(slo, shi, acc_lo2);
    add128(slo, shi, acc_hi2 << 32);
    shi += acc_hi2 >> 32;
    add128(slo, shi, acc_lo);
    add128(slo, shi, acc_hi << 32);
    shi += acc_hi >> 32;
    if (sout) {
#pragma unroll
      for (int j = 0; j < K; ++j) sout[j * p.ld + stream] = s[j];
    }
  }
  fs += fs2;
  // warp reduction (exact: 128-bit sums, xor; fixed shuffle order for fs)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const uint64_t olo = __shfl_xor_sync(0xffffffffu, slo, off);
    const uint64_t ohi = __shfl_xor_sync(0xffffffffu, shi, off);
    const uint64_t nlo = slo + olo;
    shi = shi + ohi + (nlo < slo ? 1 : 0);
    slo = nlo;
    sx ^= __shfl_xor_sync(0xffffffffu, sx, off);
    slow += __shfl_xor_sync(0xffffffffu, slow, off);
    fs += __shfl_xor_sync(0xffffffffu, fs, off);
  }
  __shared__ uint64_t r_lo[WPB], r_hi[WPB], r_x[WPB], r_low[WPB];
  __shared__ double r_fs[WPB];
  if (lane == 0) {
    r_lo[warp] = slo;
    r_hi[warp] = shi;
    r_x[warp] = sx;
    r_low[warp] = slow;
    r_fs[warp] = fs;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t lo = 0, hi = 0, x = 0, low = 0;
    double f = 0.0;
    for (int i = 0; i < WPB; ++i) {
      const uint64_t nlo = lo + r_lo[i];
      hi += r_hi[i] + (nlo < lo ? 1 : 0);
      lo = nlo;
      x ^= r_x[i];
      low += r_low[i];
      f += r_fs[i];
    }
    slp_checksum *part = static_cast<slp_checksum *>(p.partials) + blockIdx.x;
    part->sum_lo = lo;
    part->sum_hi = hi;
    part->xor_all = x;
    part->low_sum = low;
    part->count = 0;
    part->fsum = f;
  }
}

// deterministic final reduction of the per-CTA partials (one CTA, fixed order)
__global__ void k_fused_final(const slp_checksum *parts, int nparts, slp_checksum *result, uint64_t count,
                              double fscale);

// ---- K1: jump --------------------------------------------------------------------
//
// dst = src * p(M) = XOR over set coefficients d of src * M^d, stepping a copy
// of the state through d = 0..n-1 (the reference's Generator.jump / _vec_jump).
// UNIFORM: the polynomial is the same for the whole warp -> plain branch;
// otherwise each lane has its own polynomial -> masked xor (one LOP3 per word).

constexpr int kJumpThreads = 128;

template <class G, bool UNIFORM>
__global__ void __launch_bounds__(kJumpThreads) k_jump(JumpParams p, const __grid_constant__ BaseStates base) {
  using word = typename G::word;
  constexpr int K = G::k;
  const uint64_t t = (uint64_t)blockIdx.x * kJumpThreads + threadIdx.x;
  if (t >= p.count) return;
  const uint64_t b = blockIdx.y;
  word cur[K], acc[K];
  if (p.use_base) {
#pragma unroll
    for (int j = 0; j < K; ++j) cur[j] = (word)base.w[b * K + j];
  } else {
    const word *src = static_cast<const word *>(p.src);
    const uint64_t si = b * p.batch_stride + p.src_off + (p.pmode == 3 ? t / p.m : (p.m ? t % p.m : t));
#pragma unroll
    for (int j = 0; j < K; ++j) cur[j] = src[j * p.ld_src + si];
  }
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = 0;
  const uint64_t pidx =
      p.poly0 + (p.pmode == 1 ? t / p.m : (p.pmode == 2 ? t : (p.pmode == 3 ? t % p.m : 0)));
  const uint64_t *poly = p.polys ? p.polys + pidx * G::pw : base.w;  // slp_jump_states: poly in params
  const int pw_used = p.pw_used > 0 && p.pw_used < G::pw ? p.pw_used : G::pw;
#pragma unroll 1
  for (int wi = 0; wi < pw_used; ++wi) {
    const uint64_t cb = poly[wi];
#pragma unroll
    for (int bb = 0; bb < 64; ++bb) {
      const int o = bb % K;
      if constexpr (UNIFORM) {
        if ((cb >> bb) & 1ull) {
#pragma unroll
          for (int j = 0; j < K; ++j) acc[j] ^= cur[G::slot(o, j)];
        }
      } else {
        const word msk = (word)0 - (word)((cb >> bb) & 1ull);
#pragma unroll
        for (int j = 0; j < K; ++j) acc[j] ^= cur[G::slot(o, j)] & msk;
      }
      G::step(cur, o);
    }
  }
  word *dst = static_cast<word *>(p.dst);
  const uint64_t di = b * p.batch_stride + p.dst_off + t;
#pragma unroll
  for (int j = 0; j < K; ++j) dst[j * p.ld_dst + di] = acc[j];
}

// ---- K1t: table-driven uniform jump (method of four Russians) -------------------
//
// A jump by a fixed polynomial p is the GF(2)-linear map state -> state * p(M)
// (the reference's Generator.jump, generators.py:315-334).  Its n x n matrix
// has rows r_i = e_i * p(M) (K1 on the n unit vectors, once per polynomial).
// Grouping the input bits in nibbles, state * p(M) = XOR over nibble groups g
// of T_g[nibble_g(state)] with T_g[v] = XOR of the rows 4g+b for the bits b
// of v: n/4 table lookups and n^2/128 word xors per state instead of n engine
// steps plus ~n/2 k-word xors.  Bits are numbered in the state's 32-bit
// words (flat word order, low half first for w = 64).  A CTA holds one
// table slice (<= 8 output words, <= 128 KB) in shared memory.  A lookup is
// S/2 LDS.64: the 16 entries of one (group, word pair) are 16 consecutive
// 8-byte vectors = exactly the 32 banks, so the lanes of a half-warp never
// conflict (distinct entries hit distinct banks, equal entries broadcast).
// (LDS.128 over 256-byte rows conflicts: entries v and v+8 share banks;
// ncu counted ~3 extra wavefronts per load.)

template <class G>
struct JumpTable {
  static constexpr int NB = G::n;              // state bits
  static constexpr int NW = NB / 32;           // 32-bit words per state
  static constexpr int S = NW < 8 ? NW : 8;    // output words per slice
  static constexpr int Z = NW / S;             // slices
  static constexpr int VW = 2;                 // words per vector load (LDS.64: see below)
  static constexpr int Q = S / VW;             // vector loads per lookup
  static constexpr int NG = NB / 4;            // nibble groups
  static constexpr int slice_words = NG * 16 * S;
  static constexpr uint64_t table_words = (uint64_t)Z * slice_words;  // n^2 / 8
  static_assert(NW * 32 == NB && NW % S == 0 && S % VW == 0, "table geometry");
};
constexpr int kTableThreads = 256;

// 32-bit word j of state i in SoA [k][ld] storage of w-bit words
template <class G>
__device__ __forceinline__ uint32_t state_w32(const void *base, uint64_t ld, uint64_t i, int j) {
  if constexpr (G::w == 64)
    return static_cast<const uint32_t *>(base)[2 * ((uint64_t)(j >> 1) * ld + i) + (j & 1)];
  else
    return static_cast<const uint32_t *>(base)[(uint64_t)j * ld + i];
}

// thread (g, v): entry v of nibble group g, all output words
template <class G>
__global__ void k_build_table(const void *rows, uint32_t *table) {
  using JT = JumpTable<G>;
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= JT::NG * 16) return;
  const int g = id >> 4, v = id & 15;
  for (int w = 0; w < JT::NW; ++w) {
    uint32_t x = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if ((v >> b) & 1) x ^= state_w32<G>(rows, JT::NB, (uint64_t)(4 * g + b), w);
    const int z = w / JT::S, ws = w % JT::S, q = ws / JT::VW, e = ws % JT::VW;
    table[(uint64_t)z * JT::slice_words + ((uint64_t)(g * JT::Q + q) * 16 + v) * JT::VW + e] = x;
  }
}

template <class G>
__global__ void __launch_bounds__(kTableThreads) k_jump_table(TableJumpParams p, uint32_t cpc) {
  using JT = JumpTable<G>;
  using word = typename G::word;
  using vec = uint2;
  extern __shared__ __align__(16) uint8_t tsm_raw[];
  vec *tsm = reinterpret_cast<vec *>(tsm_raw);
  const uint64_t c = blockIdx.x / cpc, part = blockIdx.x % cpc;
  const int z = blockIdx.z;
  const uint64_t b = blockIdx.y;
  {
    const uint4 *tg = reinterpret_cast<const uint4 *>(p.tables + ((p.table0 + c) * JT::Z + z) * JT::slice_words);
    uint4 *d = reinterpret_cast<uint4 *>(tsm_raw);
    for (int i = threadIdx.x; i < JT::slice_words / 4; i += kTableThreads) d[i] = tg[i];
  }
  __syncthreads();
  const uint64_t t0 = c * p.m;
  const uint64_t t1 = t0 + p.m < p.count ? t0 + p.m : p.count;
  for (uint64_t t = t0 + part * kTableThreads + threadIdx.x; t < t1; t += (uint64_t)cpc * kTableThreads) {
    const uint64_t si = b * p.batch_stride + p.src_off + (t - t0);
    uint32_t acc[JT::S];
#pragma unroll
    for (int e = 0; e < JT::S; ++e) acc[e] = 0;
    uint32_t x = state_w32<G>(p.src, p.ld_src, si, 0);
#pragma unroll(JT::NW <= 8 ? JT::NW : 4)
    for (int j = 0; j < JT::NW; ++j) {
      const uint32_t xn = j + 1 < JT::NW ? state_w32<G>(p.src, p.ld_src, si, j + 1) : 0u;  // prefetch
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const int v = (x >> (4 * h)) & 15;
        const int g = j * 8 + h;
#pragma unroll
        for (int q = 0; q < JT::Q; ++q) {
          const vec tv = tsm[(g * JT::Q + q) * 16 + v];
          acc[q * JT::VW + 0] ^= tv.x;
          acc[q * JT::VW + 1] ^= tv.y;
        }
      }
      x = xn;
    }
    const uint64_t di = b * p.batch_stride + p.dst_off + t;
    word *dst = static_cast<word *>(p.dst);
    if constexpr (G::w == 64) {
#pragma unroll
      for (int e = 0; e < JT::S; e += 2)
        dst[(uint64_t)((z * JT::S + e) >> 1) * p.ld_dst + di] = ((uint64_t)acc[e + 1] << 32) | acc[e];
    } else {
#pragma unroll
      for (int e = 0; e < JT::S; ++e) dst[(uint64_t)(z * JT::S + e) * p.ld_dst + di] = acc[e];
    }
  }
}

// ---- host launchers ----------------------------------------------------------------

template <class G, int OK, int MODE, bool CSUM = false>
int launch_fill(const FillParams &p0, cudaStream_t st, int *grid_out = nullptr) {
  using bits = typename Out<OK, typename G::word>::bits;
  constexpr int ES = sizeof(bits);
  FillParams p = p0;
  if (grid_out) *grid_out = 0;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof tmap);
  if constexpr (MODE == FILL_TMA) {
    int rc = make_store_tmap(&tmap, p.out, ES, p.T, p.nstreams, p.ld_out, FillShape<G, fill_kind<OK, CSUM>()>::segs);
    if (rc != SLP_OK) return rc;
  } else if constexpr (MODE == FILL_POS_TMA) {
    int rc = make_store_tmap_pm(&tmap, p.out, ES, p.T, p.nstreams, p.ld_out,
                                FillShape<G, fill_kind<OK, CSUM>()>::row_bytes / ES);
    if (rc != SLP_OK) return rc;
  }
  auto kern = k_fill<G, OK, MODE, CSUM>;
  const int smem = MODE == FILL_POS ? 0 : FillShape<G, fill_kind<OK, CSUM>()>::smem;
  p.nunits = (p.nstreams + 31) / 32;
  const int dev = current_device();
  static std::atomic<int> per_sm[64];  // occupancy per device, computed once (benign race: same value)
  if (dev < 0 || dev >= 64) return SLP_ERR_CUDA;
  if (!per_sm[dev]) {
    if (smem > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return cuda_fail("cudaFuncSetAttribute");
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kFillThreads, smem) != cudaSuccess || b < 1)
      return cuda_fail("occupancy");
    per_sm[dev] = b;
  }
  if (p.nunits == 0 || p.T == 0) return SLP_OK;
  uint64_t want = (p.nunits + kFillWarps - 1) / kFillWarps;
  uint64_t cap = (uint64_t)sm_count(dev) * per_sm[dev] * fill_grid_mult();
  const unsigned grid = (unsigned)(want < cap ? want : cap);
  if constexpr (CSUM) {
    if ((uint64_t)grid * sizeof(slp_checksum) > p.workspace_bytes) return SLP_ERR_BUFFER;
  }
  if (grid_out) *grid_out = (int)grid;
  kern<<<grid, kFillThreads, smem, st>>>(p, tmap);
  return check_launch("k_fill");
}

// store + checksum in one pass: stream-major TMA path only (else UNSUPPORTED;
// callers fall back to a fill followed by a fused pass over the same states)
template <class G>
int fill_csum_impl(const FillParams &p, int out_kind, cudaStream_t st, int *grid_out) {
  constexpr int W = G::w;
  if (grid_out) *grid_out = 0;
  int ok;
  if (out_kind == SLP_OUT_NATIVE || (out_kind == SLP_OUT_U64 && W == 64))
    ok = SLP_OUT_NATIVE;
  else if (out_kind == SLP_OUT_F64 && W == 64)
    ok = SLP_OUT_F64;
  else if (out_kind == SLP_OUT_F32 && W == 32)
    ok = SLP_OUT_F32;
  else
    return SLP_ERR_UNSUPPORTED;
  const int es = ok == SLP_OUT_NATIVE ? W / 8 : (ok == SLP_OUT_F32 ? 4 : 8);
  if (!tma_ok(p.out, es, p.T, p.nstreams, p.ld_out, fill_cfg(G::id, FILL_KIND_CHECKSUM).segs))
    return SLP_ERR_UNSUPPORTED;
  if constexpr (W == 64) {
    if (ok == SLP_OUT_F64) return launch_fill<G, SLP_OUT_F64, FILL_TMA, true>(p, st, grid_out);
  } else {
    if (ok == SLP_OUT_F32) return launch_fill<G, SLP_OUT_F32, FILL_TMA, true>(p, st, grid_out);
  }
  return launch_fill<G, SLP_OUT_NATIVE, FILL_TMA, true>(p, st, grid_out);
}

template <class G>
int fill_impl(const FillParams &p, int out_kind, int layout, cudaStream_t st) {
  constexpr int W = G::w;
  int ok;
  if (out_kind == SLP_OUT_NATIVE || (out_kind == SLP_OUT_U64 && W == 64))
    ok = SLP_OUT_NATIVE;
  else if (out_kind == SLP_OUT_U64)
    ok = SLP_OUT_U64;
  else if (out_kind == SLP_OUT_F64 && W == 64)
    ok = SLP_OUT_F64;
  else if (out_kind == SLP_OUT_F32 && W == 32)
    ok = SLP_OUT_F32;
  else
    return SLP_ERR_UNSUPPORTED;
  const int es = (ok == SLP_OUT_NATIVE) ? W / 8 : (ok == SLP_OUT_F32 ? 4 : 8);
  int mode;
  if (layout == SLP_POSITION_MAJOR)
    mode = tma_ok_pm(p.out, es, p.T, p.nstreams, p.ld_out,
                     fill_cfg(G::id, ok == SLP_OUT_NATIVE ? FILL_KIND_NATIVE : FILL_KIND_CONVERT).segs * 128 / es)
               ? FILL_POS_TMA
               : FILL_POS;
  else if (layout == SLP_STREAM_MAJOR)
    mode = tma_ok(p.out, es, p.T, p.nstreams, p.ld_out,
                  fill_cfg(G::id, ok == SLP_OUT_NATIVE ? FILL_KIND_NATIVE : FILL_KIND_CONVERT).segs)
               ? FILL_TMA
               : FILL_STAGED;
  else
    return SLP_ERR_INVALID;
#define SLP_FILL_CASE(OKV)                                                     \
  if (ok == OKV) {                                                             \
    if (mode == FILL_TMA) return launch_fill<G, OKV, FILL_TMA>(p, st);         \
    if (mode == FILL_STAGED) return launch_fill<G, OKV, FILL_STAGED>(p, st);   \
    if (mode == FILL_POS_TMA) return launch_fill<G, OKV, FILL_POS_TMA>(p, st); \
    return launch_fill<G, OKV, FILL_POS>(p, st);                               \
  }
  if constexpr (W == 64) {
    SLP_FILL_CASE(SLP_OUT_NATIVE)
    SLP_FILL_CASE(SLP_OUT_F64)
  } else {
    SLP_FILL_CASE(SLP_OUT_NATIVE)
    SLP_FILL_CASE(SLP_OUT_U64)
    SLP_FILL_CASE(SLP_OUT_F32)
  }
#undef SLP_FILL_CASE
  return SLP_ERR_UNSUPPORTED;
}

template <class G, bool MANT, bool F64>
int launch_fused_t(const FusedParams &p0, cudaStream_t st, int *grid_out) {
  FusedParams p = p0;
  p.nunits = (p.nstreams + 31) / 32;
  auto kern = k_fused<G, MANT, F64>;
  const int dev = current_device();
  static std::atomic<int> per_sm[64];  // occupancy per device, computed once (benign race: same value)
  if (dev < 0 || dev >= 64) return SLP_ERR_CUDA;
  if (!per_sm[dev]) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kFusedThreads, 0) != cudaSuccess || b < 1)
      return cuda_fail("occupancy");
    per_sm[dev] = b;
  }
  constexpr int WPB = kFusedThreads / 32;
  uint64_t want = (p.nunits + WPB - 1) / WPB;
  if (want == 0) want = 1;
  const uint64_t cap = (uint64_t)sm_count(dev) * per_sm[dev];
  const unsigned grid = (unsigned)(want < cap ? want : cap);
  if (grid_out) *grid_out = (int)grid;
  if ((uint64_t)grid * sizeof(slp_checksum) > p.workspace_bytes) return SLP_ERR_BUFFER;
  kern<<<grid, kFusedThreads, 0, st>>>(p);
  return check_launch("k_fused");
}

template <class G>
int fused_impl(const FusedParams &p, int flags, cudaStream_t st, int *grid_out) {
  if (flags & SLP_FUSE_F64) return launch_fused_t<G, true, true>(p, st, grid_out);
  if (flags & SLP_FUSE_EXACT) return launch_fused_t<G, true, false>(p, st, grid_out);
  return launch_fused_t<G, false, false>(p, st, grid_out);
}

template <class G>
int fused_grid_cap(int dev) {
  int best = 1;
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_fused<G, true, true>, kFusedThreads, 0) == cudaSuccess)
    best = b > best ? b : best;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_fused<G, true, false>, kFusedThreads, 0) == cudaSuccess)
    best = b > best ? b : best;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_fused<G, false, false>, kFusedThreads, 0) == cudaSuccess)
    best = b > best ? b : best;
  return sm_count(dev) * best;
}

template <class G>
int jump_impl(const JumpParams &p, const BaseStates *base, bool uniform, uint64_t nbatch, cudaStream_t st) {
  if (p.count == 0 || nbatch == 0) return SLP_OK;
  const uint64_t gx = (p.count + kJumpThreads - 1) / kJumpThreads;
  if (gx > 0x7fffffffull || nbatch > 65535) return SLP_ERR_INVALID;
  dim3 grid((unsigned)gx, (unsigned)nbatch);
  static BaseStates zero_base;  // unused when p.use_base == 0
  const BaseStates &bs = base ? *base : zero_base;
  if (uniform)
    k_jump<G, true><<<grid, kJumpThreads, 0, st>>>(p, bs);
  else
    k_jump<G, false><<<grid, kJumpThreads, 0, st>>>(p, bs);
  return check_launch("k_jump");
}

template <class G>
uint64_t table_words_impl() {
  return JumpTable<G>::table_words;
}

template <class G>
int build_table_impl(const void *rows, uint32_t *table, cudaStream_t st) {
  constexpr int nthr = JumpTable<G>::NG * 16;
  k_build_table<G><<<(nthr + 127) / 128, 128, 0, st>>>(rows, table);
  return check_launch("k_build_table");
}

template <class G>
int jump_table_impl(const TableJumpParams &p, uint64_t nbatch, cudaStream_t st) {
  using JT = JumpTable<G>;
  if (p.count == 0 || nbatch == 0) return SLP_OK;
  if (nbatch > 65535 || p.m == 0) return SLP_ERR_INVALID;
  constexpr int smem = JT::slice_words * 4;
  auto kern = k_jump_table<G>;
  const int dev = current_device();
  static std::atomic<int> per_sm[64];  // occupancy per device (benign race: same value)
  if (dev < 0 || dev >= 64) return SLP_ERR_CUDA;
  if (!per_sm[dev]) {
    if (smem > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return cuda_fail("cudaFuncSetAttribute");
    int bl = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bl, kern, kTableThreads, smem) != cudaSuccess || bl < 1)
      return cuda_fail("occupancy");
    per_sm[dev] = bl;
  }
  const uint64_t ntab = (p.count + p.m - 1) / p.m;
  // CTAs per table: fill ~2 waves, but give each CTA >= 4 states per thread
  // so the table load is amortised
  const uint64_t slots = (uint64_t)sm_count(dev) * per_sm[dev] * 2;
  uint64_t cpc = slots / (ntab * nbatch * JT::Z);
  const uint64_t cap = (p.m + 4 * kTableThreads - 1) / (4 * kTableThreads);
  if (cpc > cap) cpc = cap;
  if (cpc < 1) cpc = 1;
  if (ntab * cpc > 0x7fffffffull) return SLP_ERR_INVALID;
  dim3 grid((unsigned)(ntab * cpc), (unsigned)nbatch, (unsigned)JT::Z);
  kern<<<grid, kTableThreads, smem, st>>>(p, (uint32_t)cpc);
  return check_launch("k_jump_table");
}

// ---- K6: Hamming-weight-dependency counting consumer ---------------------------
//
// Fused "generate -> test value -> popcount -> trit -> signature -> count"
// for the HWD test (hwd.py:206-233 HwdCounters._add, :446-470 transitional,
// :473-476 split).  Thread i owns one contiguous segment of the generator's
// single output stream: it starts `warm` test values early (its state comes
// from K1) only to rebuild the signature of the k preceding trits, then
// counts `cnt` values.
// Counters follow the reference's packed small-counter scheme (hwd.py:167-247):
// one 32-bit shared-memory cell per signature, count in the high 13 bits and
// weight sum in the low 19, bumped with one 32-bit shared atomic per value
// (the shared-atomic rate is this kernel's limit).  The host sizes segments
// so the busiest cell expects <= 4096 counts per CTA; at the end the CTA
// checks conservation (sum of counts == values counted, as HwdCounters.flush)
// and drains into exact 64-bit global counters.  If a cell overflowed, the
// CTA recounts its segments exactly with 64-bit global atomics instead, so
// the result is always exact (the reference would report a forced failure).

constexpr int kHwdThreads = 256;
constexpr uint32_t kHwdRecip = 0x55555556u;  // ceil(2^32 / 3), hwd.py:44

// counts one thread's segment; GLOBAL: 64-bit global atomics, else packed smem
// cells.  SLICED: only signatures in [cell_lo, cell_lo + p.slice_cells) are
// counted (3^k cells split over the CTAs of blockIdx.y); returns the number
// of values counted.
template <class G, bool TRANS, bool SPLIT, bool GLOBAL, bool SLICED = false>
__device__ __forceinline__ uint32_t hwd_segment(const HwdParams &p, uint64_t i, uint32_t *cells,
                                                uint32_t cell_lo = 0) {
  using word = typename G::word;
  constexpr int K = G::k;
  constexpr int TW = SPLIT ? 32 : G::w;  // test-value width
  const word *sin = static_cast<const word *>(p.sin);
  word s[K];
#pragma unroll
  for (int j = 0; j < K; ++j) s[j] = sin[j * p.ld + i];
  // cnt <= tseg < 2^16 and warm <= k + 2: 32-bit counters
  uint32_t cnt = (uint32_t)((i + 1) * p.tseg <= p.total ? p.tseg : p.total - i * p.tseg);
  uint32_t counted = SLICED ? 0u : cnt;
  uint32_t warm = (uint32_t)(i == 0 ? p.warm0 : p.warm);
  uint32_t sig = 0;
  uint64_t prev = 0;
  const int lo = p.lo, hi = p.hi;
  const uint32_t pow3 = p.pow3k1;
  auto consume = [&](uint64_t x, bool count) {
    if constexpr (TRANS) {
      const uint64_t y = x ^ (((x << 1) | (prev >> (TW - 1))) & (TW == 64 ? ~0ull : ((1ull << TW) - 1)));
      prev = x;
      x = y;
    }
    const int nu = TW == 64 ? __popcll(x) : __popc((uint32_t)x);
    const uint32_t t = (uint32_t)(nu >= lo) + (uint32_t)(nu > hi);
    if (count) {
      if constexpr (SLICED) {
        const uint32_t rel = sig - cell_lo;
        if (rel < p.slice_cells) {
          ++counted;
          if constexpr (GLOBAL) {
            atomicAdd(p.g_counts + sig, 1ull);
            atomicAdd(p.g_sums + sig, (unsigned long long)nu);
          } else {
            atomicAdd(cells + rel, (1u << 19) | (uint32_t)nu);
          }
        }
      } else if constexpr (GLOBAL) {
        atomicAdd(p.g_counts + sig, 1ull);
        atomicAdd(p.g_sums + sig, (unsigned long long)nu);
      } else {
        atomicAdd(cells + sig, (1u << 19) | (uint32_t)nu);
      }
    }
    sig = __umulhi(sig, kHwdRecip) + t * pow3;
  };
  // phase A: warm-up, only rebuilds the signature (scalar steps keep flat order)
  bool pending = false;
  uint64_t pend = 0;
  while (warm > 0) {
    const word x = G::next_flat(s);
    if constexpr (SPLIT) {
      consume((uint64_t)x & 0xFFFFFFFFull, false);
      if (--warm > 0) {
        consume((uint64_t)x >> 32, false);
        --warm;
      } else {
        pending = true;  // the high half is the first counted value
        pend = (uint64_t)x >> 32;
      }
    } else {
      consume((uint64_t)x, false);
      --warm;
    }
  }
  if (pending && cnt > 0) {
    consume(pend, true);
    --cnt;
  }
  // phase B: counting in unrolled chunks of CH words (ring offsets static)
  constexpr int CH = 16;
  constexpr uint32_t VPW = SPLIT ? 2 : 1;  // test values per generator word
  for (uint32_t c = cnt / (CH * VPW); c > 0; --c) {
#pragma unroll
    for (int t = 0; t < CH; ++t) {
      const word x = G::output(s, t % K);
      G::step(s, t % K);
      if constexpr (SPLIT) {
        consume((uint64_t)x & 0xFFFFFFFFull, true);
        consume((uint64_t)x >> 32, true);
      } else {
        consume((uint64_t)x, true);
      }
    }
  }
  cnt %= CH * VPW;
  // phase C: tail
  while (cnt > 0) {
    const word x = G::next_flat(s);
    if constexpr (SPLIT) {
      consume((uint64_t)x & 0xFFFFFFFFull, true);
      if (--cnt > 0) {
        consume((uint64_t)x >> 32, true);
        --cnt;
      }
    } else {
      consume((uint64_t)x, true);
      --cnt;
    }
  }
  return counted;
}

// SLICED (k >= 10): 3^k packed cells exceed shared memory, so the cells are
// split into gridDim.y slices; CTA (x, y) regenerates the segments of CTA
// column x and counts only the signatures of slice y.  Generation is repeated
// per slice, but every count stays a shared-memory atomic (global 64-bit
// atomics are 8-20x slower per value).
template <class G, bool TRANS, bool SPLIT, bool SLICED>
__global__ void __launch_bounds__(kHwdThreads) k_hwd(HwdParams p) {
  extern __shared__ uint32_t cells[];
  __shared__ unsigned long long s_counted, s_cellsum;
  const int tid = threadIdx.x;
  const uint64_t i = (uint64_t)blockIdx.x * kHwdThreads + tid;
  if (p.global_cells) {  // 3^k cells do not fit in shared memory even when sliced
    if (i < p.nthreads) hwd_segment<G, TRANS, SPLIT, true>(p, i, nullptr);
    return;
  }
  const uint32_t cell_lo = SLICED ? blockIdx.y * p.slice_cells : 0u;
  const uint32_t nc = SLICED ? (p.ncells - cell_lo < p.slice_cells ? p.ncells - cell_lo : p.slice_cells) : p.ncells;
  for (uint32_t c = tid; c < nc; c += kHwdThreads) cells[c] = 0u;
  if (tid == 0) s_counted = s_cellsum = 0ull;
  __syncthreads();
  uint32_t mine = 0;
  if (i < p.nthreads) mine = hwd_segment<G, TRANS, SPLIT, false, SLICED>(p, i, cells, cell_lo);
  atomicAdd(&s_counted, (unsigned long long)mine);
  __syncthreads();
  unsigned long long part = 0;
  for (uint32_t c = tid; c < nc; c += kHwdThreads) part += cells[c] >> 19;
  atomicAdd(&s_cellsum, part);
  __syncthreads();
  if (s_cellsum == s_counted) {  // conservation holds: no packed cell overflowed
    for (uint32_t c = tid; c < nc; c += kHwdThreads) {
      const uint32_t cell = cells[c];
      if (cell) {
        atomicAdd(p.g_counts + cell_lo + c, (unsigned long long)(cell >> 19));
        atomicAdd(p.g_sums + cell_lo + c, (unsigned long long)(cell & 0x7FFFFu));
      }
    }
  } else {  // recount this CTA's segments (its slice) exactly (rare: heavily skewed streams)
    if (tid == 0 && p.overflow_ctas) atomicAdd(p.overflow_ctas, 1ull);
    if (i < p.nthreads) hwd_segment<G, TRANS, SPLIT, true, SLICED>(p, i, nullptr, cell_lo);
  }
}

template <class G, bool TRANS, bool SPLIT, bool SLICED>
int launch_hwd_t(const HwdParams &p, cudaStream_t st) {
  auto kern = k_hwd<G, TRANS, SPLIT, SLICED>;
  const uint32_t cells = SLICED ? p.slice_cells : p.ncells;
  const size_t smem = p.global_cells ? 0 : (size_t)cells * sizeof(uint32_t);
  if (smem > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
                              cudaSuccess)
    return cuda_fail("cudaFuncSetAttribute(hwd)");
  const uint64_t grid = (p.nthreads + kHwdThreads - 1) / kHwdThreads;
  if (grid == 0) return SLP_OK;
  const uint64_t slices = SLICED ? (p.ncells + p.slice_cells - 1) / p.slice_cells : 1;
  if (grid > 0x7fffffffull || slices > 65535) return SLP_ERR_INVALID;
  kern<<<dim3((unsigned)grid, (unsigned)slices), kHwdThreads, smem, st>>>(p);
  return check_launch("k_hwd");
}

template <class G>
int hwd_impl(const HwdParams &p, int transitional, int split, cudaStream_t st) {
  const bool sliced = !p.global_cells && p.slice_cells < p.ncells;
#define SLP_HWD_LAUNCH(TR, SP)                                                              \
  return sliced ? launch_hwd_t<G, TR, SP, true>(p, st) : launch_hwd_t<G, TR, SP, false>(p, st)
  if (split) {
    if constexpr (G::w == 64) {
      if (transitional) SLP_HWD_LAUNCH(true, true);
      SLP_HWD_LAUNCH(false, true);
    } else {
      return SLP_ERR_INVALID;  // split needs 64-bit source words
    }
  }
  if (transitional) SLP_HWD_LAUNCH(true, false);
  SLP_HWD_LAUNCH(false, false);
#undef SLP_HWD_LAUNCH
}

template <class G>
GenOps make_ops() {
  GenOps o;
  o.fill = &fill_impl<G>;
  o.fill_csum = &fill_csum_impl<G>;
  o.fused = &fused_impl<G>;
  o.fused_grid_cap = &fused_grid_cap<G>;
  o.jump = &jump_impl<G>;
  o.hwd = &hwd_impl<G>;
  o.table_words = &table_words_impl<G>;
  o.build_table = &build_table_impl<G>;
  o.jump_table = &jump_table_impl<G>;
  return o;
}

}  // namespace dev
}  // namespace slp

// Gen<> type of registry entry `id`
#define SLP_GEN_TYPE(id, name, fam, k, w, a, b, c, sc, wi, wj, S, R, T) \
  ::slp::dev::Gen<id, fam, k, w, a, b, c, sc, wi, wj, S, R, T>
