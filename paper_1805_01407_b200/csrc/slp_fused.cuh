// Kernel K4: fused consumer (k_fused) and its launchers.
#pragma once

#include "slp_gen.cuh"

namespace slp {
namespace dev {

// ---- K4: fused consumer ---------------------------------------------------------
//
// Per output: wrapping sum (IADD3 + IADD3.X) and xor (one LOP3 per two
// outputs).  MANT adds the exact 128-bit sum (one more IADD3.X with carry) and
// the sum of the low 11 (w=64) / 8 (w=32) bits, from which the exact sum of
// the converted doubles / floats follows: mant = (sum - low) >> shift.
// F64 adds a genuine float64 accumulation of the converted values.

constexpr int kFusedThreads = 256;

// FMA-form sites of the generator inside K4 (Gen::kSites).  Measured
// (profiles/round2_ab_fused_sites.md): only plain IMAD overlaps with the ALU
// pipe -- IMAD.HI and IMAD.WIDE add to its time (profiles/int_peak.cu mixes)
// -- so rotations and shifts stay ALU forms (every FMA form lost 1-25%).  The
// scrambler multiplies do better as IMAD + IMAD + IMAD.HI (site 16) than as
// IMAD.WIDE + IMAD: +1..4%, except the two cases below (-1%); and the
// scrambler additions' high words as IMAD.X (site 32), which is a plain IMAD
// with a carry-in and runs beside the ALU pipe.
template <class G, bool MANT, bool F64>
__host__ __device__ constexpr int fused_site_mask() {
  if constexpr (G::runtime) {
    return 0;
  } else if constexpr ((G::kSites & 32) != 0) {
    // + / ++: the additions' high words as IMAD.X (site 32): ++ gains 4-6%
    // (sum + xor) and 9-12% (exact, + f64); + gains 2-3% in the exact modes
    return (G::sc == SLP_SC_PLUSPLUS || MANT) ? 32 : 0;
  } else if constexpr (!(G::kSites & 16)) {
    return G::best_mask(1, (G::w == 64 ? 2 : 1) + (MANT ? 1 : 0));
  } else {
    if (G::fam == SLP_FAM_XOSHIRO && G::k == 8 && !MANT) return 0;                                // xoshiro512**, sum + xor
    if (G::fam == SLP_FAM_XOROSHIRO && G::k == 16 && G::sc == SLP_SC_STARSTAR && !F64) return 0;  // xoroshiro1024**
    return 16;
  }
}

template <class G, bool MANT, bool F64>
#ifndef SLP_FUSED_MINB
#define SLP_FUSED_MINB 1
#endif
__global__ void __launch_bounds__(kFusedThreads, SLP_FUSED_MINB) k_fused(FusedParams p) {
  const G eng = G::load(p.rt);
  using word = typename G::word;
  constexpr int K = G::k;
  constexpr int CH = 16;  // multiple of every ring size
  constexpr uint32_t LOWMASK = G::w == 64 ? 0x7FFu : 0xFFu;
  constexpr int SH = G::w == 64 ? 11 : 8;
  // float64 term of an output, before the final power-of-2 scale
  // (kFusedF64Scale): for w = 64 the output with its low 11 bits cleared
  // (2^11 times x >> 11, so every partial sum is exactly 2^11 times the
  // shifted one and the scaled result is bit-identical) -- one LOP3 on the
  // low word instead of a two-SHF 64-bit shift
  auto fterm = [](uint64_t x) -> double {
    if constexpr (G::w == 64)
      return __ull2double_rn(x & ~0x7FFull);
    else
      return __ull2double_rn(x >> SH);
  };
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
#ifdef SLP_FUSED_MASK  // A/B: force the FMA-form sites (masked to the generator's sites); MASK2: odd outputs
  constexpr int MSK = SLP_FUSED_MASK & G::kSites;
#ifdef SLP_FUSED_MASK2
  constexpr int MSK2 = SLP_FUSED_MASK2 & G::kSites;
#else
  constexpr int MSK2 = MSK;
#endif
#else
  constexpr int MSK = fused_site_mask<G, MANT, F64>();
  constexpr int MSK2 = MSK;
#endif
  const uint32_t one = p.one;
  (void)one;  // only the IMAD.WIDE accumulator policies (SLP_SUM_POLICY 1, 2) read it
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
        const word o0 = eng.template output_m<MSK>(s, t % K);
        eng.template step_m<MSK>(s, t % K);
        const word o1 = eng.template output_m<MSK2>(s, (t + 1) % K);
        eng.template step_m<MSK2>(s, (t + 1) % K);
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
          fs += fterm((uint64_t)o0);
          fs2 += fterm((uint64_t)o1);
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
      const word x = eng.next_flat(s);
      acc_lo += (uint32_t)x;
      if constexpr (G::w == 64) acc_hi += (uint32_t)((uint64_t)x >> 32);
      sx ^= (uint64_t)x;
      slow += (uint32_t)x & LOWMASK;
      if constexpr (F64) fs += fterm((uint64_t)x);
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

}  // namespace dev
}  // namespace slp
