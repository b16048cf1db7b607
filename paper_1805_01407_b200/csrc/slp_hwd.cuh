// Kernel K6: Hamming-weight-dependency counting consumer (k_hwd) and its launchers.
#pragma once

#include "slp_gen.cuh"

namespace slp {
namespace dev {

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

template <class G>
__host__ __device__ constexpr int hwd_site_mask() {
  if constexpr (G::runtime) {
    return 0;
  } else {
    // measured (profiles/round2_ab_hwd_sites.jsonl): ++ +2.7..3.2%; ** +0.7% (xoshiro256),
    // +1.9% (xoshiro512), -1.8% (xoroshiro128: keeps IMAD.WIDE)
    if ((G::kSites & 32) && G::sc == SLP_SC_PLUSPLUS) return 32;
    return ((G::kSites & 16) && G::fam == SLP_FAM_XOSHIRO) ? 16 : 0;
  }
}

// counts one thread's segment; GLOBAL: 64-bit global atomics, else packed smem
// cells.  SLICED: only signatures in [cell_lo, cell_lo + p.slice_cells) are
// counted (3^k cells split over the CTAs of blockIdx.y); returns the number
// of values counted.
template <class G, bool TRANS, bool SPLIT, bool GLOBAL, bool SLICED = false>
__device__ __forceinline__ uint32_t hwd_segment(const HwdParams &p, uint64_t i, uint32_t *cells,
                                                uint32_t cell_lo = 0) {
  const G eng = G::load(p.rt);
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
    const word x = eng.next_flat(s);
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
  // phase B: counting in unrolled chunks of CH words (ring offsets static).
  // The kernel is ALU-bound like K4, so the scrambler takes the same FMA-pipe
  // forms (Gen::kSites: multiplies with IMAD.HI carries, ++ additions with
  // IMAD.X high words; profiles/round2_ab_fused_sites.md).  SLP_HWD_MASK: A/B.
  constexpr int CH = 16;
#ifdef SLP_HWD_MASK
  constexpr int MSK = SLP_HWD_MASK & G::kSites;
#else
  constexpr int MSK = hwd_site_mask<G>();
#endif
  constexpr uint32_t VPW = SPLIT ? 2 : 1;  // test values per generator word
  for (uint32_t c = cnt / (CH * VPW); c > 0; --c) {
#pragma unroll
    for (int t = 0; t < CH; ++t) {
      const word x = eng.template output_m<MSK>(s, t % K);
      eng.template step_m<MSK>(s, t % K);
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
    const word x = eng.next_flat(s);
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

}  // namespace dev
}  // namespace slp
