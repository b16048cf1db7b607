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

template <int FAM, int K, int W, int A, int B, int C, int SC, int WI, int WJ, unsigned long long S_, int R_,
          unsigned long long T_>
struct Gen {
  using word = typename WordOf<W>::type;
  static constexpr int k = K;
  static constexpr int w = W;
  static constexpr int n = K * W;
  static constexpr int pw = n / 64;  // u64 words per jump polynomial (degree < n)
  static constexpr bool ring = FAM != SLP_FAM_XOSHIRO;

  static __device__ __forceinline__ word rotl(word x, int r) { return (word)((x << r) | (x >> (W - r))); }

  // register slot of flat word j when the ring offset is o (constant after unrolling)
  static __device__ __forceinline__ constexpr int slot(int o, int j) { return ring ? (o + j) % K : j; }

  // scramblers.py:84-95, applied to the current (pre-step) state
  static __device__ __forceinline__ word output(const word (&s)[K], int o) {
    const word xi = s[slot(o, WI)];
    if constexpr (SC == SLP_SC_NONE) {
      return xi;
    } else if constexpr (SC == SLP_SC_PLUS) {
      return (word)(xi + s[slot(o, WJ)]);
    } else if constexpr (SC == SLP_SC_STAR) {
      return (word)(xi * (word)S_);
    } else if constexpr (SC == SLP_SC_PLUSPLUS) {
      return (word)(rotl((word)(xi + s[slot(o, WJ)]), R_) + xi);
    } else {
      return (word)(rotl((word)(xi * (word)S_), R_) * (word)T_);
    }
  }

  // one engine step in the flat view (engines.py:100-140).  For ring engines
  // the flat view moves by one slot: the caller's next offset is o + 1.
  static __device__ __forceinline__ void step(word (&s)[K], int o) {
    if constexpr (FAM == SLP_FAM_XOROSHIRO) {
      const int i0 = slot(o, 0), il = slot(o, K - 1);
      const word x0 = s[i0];
      const word xl = s[il] ^ x0;
      s[il] = rotl(x0, A) ^ xl ^ (word)(xl << B);
      s[i0] = rotl(xl, C);
    } else if constexpr (FAM == SLP_FAM_XORSHIFT) {
      const int i0 = slot(o, 0), i1 = slot(o, 1);
      const word s0 = s[i0], s1 = s[i1];
      const word t = s0 ^ (word)(s0 << A);
      s[i0] = t ^ (t >> B) ^ s1 ^ (s1 >> C);
    } else if constexpr (K == 4) {
      const word t = (word)(s[1] << A);
      s[2] ^= s[0];
      s[3] ^= s[1];
      s[1] ^= s[2];
      s[0] ^= s[3];
      s[2] ^= t;
      s[3] = rotl(s[3], B);
    } else {
      const word t = (word)(s[1] << A);
      s[2] ^= s[0];
      s[5] ^= s[1];
      s[1] ^= s[2];
      s[7] ^= s[3];
      s[3] ^= s[4];
      s[4] ^= s[5];
      s[0] ^= s[6];
      s[6] ^= s[7];
      s[6] ^= t;
      s[7] = rotl(s[7], B);
    }
  }

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

// CH outputs; CH % K == 0 for ring engines so the ring offset returns to 0
template <class G, int CH>
__device__ __forceinline__ void gen_chunk(typename G::word (&s)[G::k], typename G::word (&o)[CH]) {
  static_assert(!G::ring || CH % G::k == 0, "chunk must be a multiple of the ring size");
#pragma unroll
  for (int t = 0; t < CH; ++t) {
    o[t] = G::output(s, t % G::k);
    G::step(s, t % G::k);
  }
}

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
// 128-bit accumulate of a 64-bit value
__device__ __forceinline__ void add128(uint64_t &lo, uint64_t &hi, uint64_t x) {
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, 0;" : "+l"(lo), "+l"(hi) : "l"(x));
}

// ---- K2/K3: fill ---------------------------------------------------------------
//
// A warp owns 32 consecutive substreams ("unit"); lane l keeps substream
// u*32+l in registers and emits 128 B (CH outputs) per chunk.  MODE:
//   FILL_TMA     stream-major; the warp's 32 x 128 B tile is staged in shared
//                memory with the 128B swizzle (conflict-free STS.128) and
//                written by one TMA bulk tensor store (cp.async.bulk.tensor),
//                double-buffered so generation overlaps the store;
//   FILL_STAGED  stream-major, same staging, element stores (any alignment);
//   FILL_POS     position-major: each step is one coalesced warp store.

enum { FILL_TMA = 0, FILL_STAGED = 1, FILL_POS = 2 };
constexpr int kFillWarps = 4;
constexpr int kFillBufs = 2;
constexpr int kTileBytes = 32 * 128;
constexpr int kFillSmem = kFillWarps * kFillBufs * kTileBytes + 1024;

template <class G, int OK, int MODE>
__global__ void __launch_bounds__(kFillWarps * 32) k_fill(FillParams p, const __grid_constant__ CUtensorMap tmap) {
  using word = typename G::word;
  using O = Out<OK, word>;
  using bits = typename O::bits;
  constexpr int K = G::k;
  constexpr int ES = sizeof(bits);
  constexpr int CH = 128 / ES;   // outputs per 128-byte row
  constexpr int EPC = 16 / ES;   // elements per 16-byte chunk
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;

  extern __shared__ uint8_t smem_raw[];
  uint8_t *wtiles = nullptr;
  if constexpr (MODE != FILL_POS) {
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t aligned = (raw + 1023u) & ~1023u;  // 128B swizzle atoms are 1 KiB
    wtiles = smem_raw + (aligned - raw) + warp * kFillBufs * kTileBytes;
  }

  const word *__restrict__ sin = static_cast<const word *>(p.sin);
  word *sout = static_cast<word *>(p.sout);
  bits *__restrict__ out = static_cast<bits *>(p.out);
  const uint64_t nfull = p.T / CH;
  const uint64_t rem = p.T - nfull * CH;
  uint32_t issued = 0;

  for (uint64_t u = (uint64_t)blockIdx.x * kFillWarps + warp; u < p.nunits; u += (uint64_t)gridDim.x * kFillWarps) {
    const uint64_t stream = u * 32 + lane;
    const bool valid = stream < p.nstreams;
    word s[K];
#pragma unroll
    for (int j = 0; j < K; ++j) s[j] = valid ? sin[j * p.ld + stream] : (word)0;

    for (uint64_t c = 0; c < nfull; ++c) {
      word o[CH];
      gen_chunk<G, CH>(s, o);
      if constexpr (MODE == FILL_POS) {
        if (valid) {
          bits *dst = out + (c * CH) * p.ld_out + stream;
#pragma unroll
          for (int t = 0; t < CH; ++t) dst[(uint64_t)t * p.ld_out] = O::conv(o[t]);
        }
      } else {
        uint8_t *tile = wtiles + (issued & (kFillBufs - 1)) * kTileBytes;
        if constexpr (MODE == FILL_TMA) {
          if (lane == 0 && issued >= kFillBufs) bulk_wait_read<kFillBufs - 1>();
        }
        __syncwarp();
        // row `lane`, 16-byte chunk q stored at chunk q ^ (lane & 7)  (CU_TENSOR_MAP_SWIZZLE_128B)
        uint8_t *row = tile + lane * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          uint8_t *dst = row + ((q ^ (lane & 7)) << 4);
          if constexpr (ES == 8) {
            *reinterpret_cast<ulonglong2 *>(dst) =
                make_ulonglong2((unsigned long long)O::conv(o[2 * q]), (unsigned long long)O::conv(o[2 * q + 1]));
          } else {
            *reinterpret_cast<uint4 *>(dst) = make_uint4((uint32_t)O::conv(o[4 * q]), (uint32_t)O::conv(o[4 * q + 1]),
                                                         (uint32_t)O::conv(o[4 * q + 2]), (uint32_t)O::conv(o[4 * q + 3]));
          }
        }
        if constexpr (MODE == FILL_TMA) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&tmap, smem_u32(tile), (int)(c * CH), (int)(u * 32));
            bulk_commit();
          }
        } else {
          __syncwarp();
          // element stores, lanes sweep rows: ES=8 -> 2 rows per pass, ES=4 -> 1 row
          constexpr int LPR = CH;  // lanes per row
          constexpr int RPP = 32 / LPR;
#pragma unroll 4
          for (int r0 = 0; r0 < 32; r0 += RPP) {
            const int r = r0 + lane / LPR;
            const int e = lane % LPR;
            const uint64_t srow = u * 32 + r;
            const bits v = *reinterpret_cast<const bits *>(tile + r * 128 + (((e / EPC) ^ (r & 7)) << 4) + (e % EPC) * ES);
            if (srow < p.nstreams) out[srow * p.ld_out + c * CH + e] = v;
          }
          __syncwarp();
        }
        ++issued;
      }
    }
    for (uint64_t t = 0; t < rem; ++t) {
      const word x = G::next_flat(s);
      if (valid) {
        const uint64_t pos = nfull * CH + t;
        if constexpr (MODE == FILL_POS)
          out[pos * p.ld_out + stream] = O::conv(x);
        else
          out[stream * p.ld_out + pos] = O::conv(x);
      }
    }
    if (valid && sout) {
#pragma unroll
      for (int j = 0; j < K; ++j) sout[j * p.ld + stream] = s[j];
    }
  }
  if constexpr (MODE == FILL_TMA) {
    if (lane == 0) bulk_wait_all<0>();
  }
}

// ---- K4: fused consumer ---------------------------------------------------------

constexpr int kFusedThreads = 256;

template <class G, bool F64>
__global__ void __launch_bounds__(kFusedThreads) k_fused(FusedParams p) {
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

  uint64_t slo = 0, shi = 0, sx = 0, slow = 0;
  double fs = 0.0;
  for (uint64_t u = (uint64_t)blockIdx.x * WPB + warp; u < p.nunits; u += (uint64_t)gridDim.x * WPB) {
    const uint64_t stream = u * 32 + lane;
    if (stream >= p.nstreams) continue;
    word s[K];
#pragma unroll
    for (int j = 0; j < K; ++j) s[j] = sin[j * p.ld + stream];
    for (uint64_t c = 0; c < nfull; ++c) {
      word o[CH];
      gen_chunk<G, CH>(s, o);
      uint32_t lw = 0;
      word xx = 0;
#pragma unroll
      for (int t = 0; t < CH; t += 2) {
        add128(slo, shi, (uint64_t)o[t]);
        add128(slo, shi, (uint64_t)o[t + 1]);
        xx ^= o[t] ^ o[t + 1];
        lw += ((uint32_t)o[t] & LOWMASK) + ((uint32_t)o[t + 1] & LOWMASK);
        if constexpr (F64) {
          fs += __ull2double_rn((uint64_t)o[t] >> SH);
          fs += __ull2double_rn((uint64_t)o[t + 1] >> SH);
        }
      }
      sx ^= (uint64_t)xx;
      slow += lw;
    }
    for (uint64_t t = 0; t < rem; ++t) {
      const word x = G::next_flat(s);
      add128(slo, shi, (uint64_t)x);
      sx ^= (uint64_t)x;
      slow += (uint32_t)x & LOWMASK;
      if constexpr (F64) fs += __ull2double_rn((uint64_t)x >> SH);
    }
    if (sout) {
#pragma unroll
      for (int j = 0; j < K; ++j) sout[j * p.ld + stream] = s[j];
    }
  }
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
    const uint64_t si = b * p.batch_stride + p.src_off + (p.m ? t % p.m : t);
#pragma unroll
    for (int j = 0; j < K; ++j) cur[j] = src[j * p.ld_src + si];
  }
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = 0;
  const uint64_t pidx = p.poly0 + (p.pmode == 1 ? t / p.m : (p.pmode == 2 ? t : 0));
  const uint64_t *poly = p.polys ? p.polys + pidx * G::pw : base.w;  // slp_jump_states: poly in params
#pragma unroll 1
  for (int wi = 0; wi < G::pw; ++wi) {
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

// ---- host launchers ----------------------------------------------------------------

template <class G, int OK, int MODE>
int launch_fill(const FillParams &p0, cudaStream_t st) {
  using bits = typename Out<OK, typename G::word>::bits;
  constexpr int ES = sizeof(bits);
  FillParams p = p0;
  p.nunits = (p.nstreams + 31) / 32;
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof tmap);
  if constexpr (MODE == FILL_TMA) {
    int rc = make_store_tmap(&tmap, p.out, ES, p.T, p.nstreams, p.ld_out);
    if (rc != SLP_OK) return rc;
  }
  auto kern = k_fill<G, OK, MODE>;
  const int smem = MODE == FILL_POS ? 0 : kFillSmem;
  const int dev = current_device();
  static int per_sm[64] = {0};
  if (dev < 0 || dev >= 64) return SLP_ERR_CUDA;
  if (!per_sm[dev]) {
    if (smem > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return cuda_fail("cudaFuncSetAttribute");
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kFillWarps * 32, smem) != cudaSuccess || b < 1)
      return cuda_fail("occupancy");
    per_sm[dev] = b;
  }
  if (p.nunits == 0 || p.T == 0) return SLP_OK;
  uint64_t want = (p.nunits + kFillWarps - 1) / kFillWarps;
  uint64_t cap = (uint64_t)sm_count(dev) * per_sm[dev] * fill_grid_mult();
  const unsigned grid = (unsigned)(want < cap ? want : cap);
  kern<<<grid, kFillWarps * 32, smem, st>>>(p, tmap);
  return check_launch("k_fill");
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
    mode = FILL_POS;
  else if (layout == SLP_STREAM_MAJOR)
    mode = tma_ok(p.out, es, p.T, p.nstreams, p.ld_out) ? FILL_TMA : FILL_STAGED;
  else
    return SLP_ERR_INVALID;
#define SLP_FILL_CASE(OKV)                                                     \
  if (ok == OKV) {                                                             \
    if (mode == FILL_TMA) return launch_fill<G, OKV, FILL_TMA>(p, st);         \
    if (mode == FILL_STAGED) return launch_fill<G, OKV, FILL_STAGED>(p, st);   \
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

template <class G, bool F64>
int launch_fused_t(const FusedParams &p0, cudaStream_t st, int *grid_out) {
  FusedParams p = p0;
  p.nunits = (p.nstreams + 31) / 32;
  auto kern = k_fused<G, F64>;
  const int dev = current_device();
  static int per_sm[64] = {0};
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
  if (flags & SLP_FUSE_F64) return launch_fused_t<G, true>(p, st, grid_out);
  return launch_fused_t<G, false>(p, st, grid_out);
}

template <class G>
int fused_grid_cap(int dev) {
  auto kern = k_fused<G, true>;
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kFusedThreads, 0) != cudaSuccess) b = 8;
  auto kern2 = k_fused<G, false>;
  int b2 = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b2, kern2, kFusedThreads, 0) != cudaSuccess) b2 = 8;
  return sm_count(dev) * (b > b2 ? b : b2);
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
GenOps make_ops() {
  GenOps o;
  o.fill = &fill_impl<G>;
  o.fused = &fused_impl<G>;
  o.fused_grid_cap = &fused_grid_cap<G>;
  o.jump = &jump_impl<G>;
  return o;
}

}  // namespace dev
}  // namespace slp

// Gen<> type of registry entry `id`
#define SLP_GEN_TYPE(id, name, fam, k, w, a, b, c, sc, wi, wj, S, R, T) \
  ::slp::dev::Gen<fam, k, w, a, b, c, sc, wi, wj, S, R, T>
