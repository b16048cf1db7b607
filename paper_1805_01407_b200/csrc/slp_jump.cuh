// Kernels K1 (polynomial jump, k_jump) and K1t (table-driven jump, k_jump_table) and their launchers.
#pragma once

#include <cstdlib>

#include "slp_gen.cuh"

namespace slp {
namespace dev {

// ---- K1: jump --------------------------------------------------------------------
//
// dst = src * p(M) = XOR over set coefficients d of src * M^d, stepping a copy
// of the state through d = 0..n-1 (the reference's Generator.jump / _vec_jump).
// UNIFORM: the polynomial is the same for the whole warp -> plain branch;
// otherwise each lane has its own polynomial -> masked xor (one LOP3 per word).

constexpr int kJumpThreads = 128;

inline int env_int_jump(const char *name, int dflt) {
  const char *v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Wide engines (k >= 8) with few states are bound by the latency of one
// thread's n dependent steps (2^15 xoroshiro1024 jumps: 52-59 us per launch,
// profiles/round2_init1024_launches.csv).  p.parts > 1 splits one jump over
// `parts` adjacent lanes: lane q first steps its copy q * n / parts times
// without accumulating (~10 instructions per step instead of ~45), then
// handles coefficients [q * n / parts, (q + 1) * n / parts); the partial sums
// are xor-ed with shuffles.  More total work, a 2-3x shorter critical path.
template <class G, bool UNIFORM>
__global__ void __launch_bounds__(kJumpThreads) k_jump(JumpParams p, const __grid_constant__ BaseStates base) {
  const G eng = G::load(p.rt);
  using word = typename G::word;
  constexpr int K = G::k;
  constexpr bool SPLIT = K >= 8;  // p.parts is honoured (jump_impl only sets it for these)
  const uint32_t parts = SPLIT ? (p.parts ? p.parts : 1u) : 1u;
  const uint64_t gt = (uint64_t)blockIdx.x * kJumpThreads + threadIdx.x;
  uint64_t t = SPLIT ? gt / parts : gt;
  const uint32_t part = SPLIT ? (uint32_t)(gt - t * parts) : 0u;
  const bool live = t < p.count;
  if (!SPLIT && !live) return;
  if (!live) t = 0;  // split: the lanes of a warp stay together for the shuffles (results discarded)
  uint64_t b = blockIdx.y;
  if (p.fold) {  // few states per batch: fold the batches into x so the warps are full
    b = t / p.fold;
    t -= b * p.fold;
  }
  word cur[K], acc[K];
  if (p.use_base) {
#pragma unroll
    for (int j = 0; j < K; ++j) cur[j] = (word)base.w[b * K + j];
  } else {
    const word *src = static_cast<const word *>(p.src);
    const uint64_t sbs = p.src_batch_stride ? p.src_batch_stride : p.batch_stride;
    const uint64_t si = b * sbs + p.src_off + (p.m ? t % p.m : t);
#pragma unroll
    for (int j = 0; j < K; ++j) cur[j] = src[j * p.ld_src + si];
  }
#pragma unroll
  for (int j = 0; j < K; ++j) acc[j] = 0;
  const uint64_t pidx =
      p.poly0 + (p.pmode == 1 ? t / p.m : (p.pmode == 2 ? t : 0));
  const uint64_t *poly = p.polys ? p.polys + pidx * G::pw : base.w;  // slp_jump_states: poly in params
  const int pw_used = p.pw_used > 0 && p.pw_used < G::pw ? p.pw_used : G::pw;
  // bits per unrolled chunk: the whole word for small states; 16 for k >= 8,
  // whose 64-bit body (~27-61 KB of SASS) thrashes the instruction cache when
  // few warps run (segment split, direct launches).  16 is a multiple of the
  // ring length, so the register rotation stays static.
  constexpr int UB = K >= 8 ? 16 : 64;
  int w0 = 0, w1 = pw_used;
  if constexpr (SPLIT) {
    if (parts > 1) {
      const int wpp = G::pw / (int)parts;  // polynomial words per part (parts divides pw)
      w0 = (int)part * wpp;
      w1 = w0 + wpp < pw_used ? w0 + wpp : pw_used;
      if (w0 < w1) {  // advance to x^(64 * w0) without accumulating
#pragma unroll 1
        for (int c = 0; c < w0 * (64 / UB); ++c) {
#pragma unroll
          for (int bb = 0; bb < UB; ++bb) eng.step(cur, bb % K);
        }
      }
    }
  }
#pragma unroll 1
  for (int wi = w0; wi < w1; ++wi) {
    uint64_t cb = poly[wi];
#pragma unroll 1
    for (int c = 0; c < 64; c += UB, cb >>= (UB & 63)) {
#pragma unroll
      for (int bb = 0; bb < UB; ++bb) {
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
        eng.step(cur, o);
      }
    }
  }
  if constexpr (SPLIT) {
    for (uint32_t off = 1; off < parts; off <<= 1) {
#pragma unroll
      for (int j = 0; j < K; ++j) acc[j] ^= __shfl_xor_sync(0xffffffffu, acc[j], off);
    }
    if (!live || part != 0) return;
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

// Threads per K1t CTA.  A 1024-bit engine's table slice (128 KB) allows one
// CTA per SM, and 8 warps do not cover the shared-memory latency: 512 threads
// take 2^20 xoroshiro1024 states from 1.26 to 1.14 ms and 2^21 from 2.69 to
// 2.18 ms; 1024 threads and the smaller engines (several CTAs per SM) lose
// 3-10% (profiles/round2_k1t_threads.jsonl).
#ifndef SLP_K1T_THREADS
#define SLP_K1T_THREADS 256
#endif
#ifndef SLP_K1T_THREADS_WIDE
#define SLP_K1T_THREADS_WIDE 512
#endif

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
  static constexpr int threads = NB >= 1024 ? SLP_K1T_THREADS_WIDE : SLP_K1T_THREADS;  // per CTA
  static constexpr uint64_t table_words = (uint64_t)Z * slice_words;  // n^2 / 8
  static_assert(NW * 32 == NB && NW % S == 0 && S % VW == 0, "table geometry");
};

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
__global__ void __launch_bounds__(JumpTable<G>::threads) k_jump_table(TableJumpParams p, uint32_t cpc) {
  using JT = JumpTable<G>;
  constexpr int kTableThreads = JT::threads;
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


template <class G>
int jump_impl(const JumpParams &p, const BaseStates *base, bool uniform, uint64_t nbatch, cudaStream_t st) {
  if (p.count == 0 || nbatch == 0) return SLP_OK;
  JumpParams q = p;
  q.parts = 1;
  if constexpr (G::k >= 8) {
    // split each jump over lanes while the launch is far from filling the GPU
    // (SLP_JUMP_PARTS: 0 auto, 1 off, 2/4/8 forced; A/B and tests -- read on every call)
    const int forced = env_int_jump("SLP_JUMP_PARTS", 0);
    const uint64_t total = p.count * nbatch;
    uint32_t parts = 1;
    if (forced == 2 || forced == 4 || forced == 8)
      parts = (uint32_t)forced;
    else if (forced == 0) {
      // measured (profiles/round2_jump_parts.md): the 16-word ring engine, whose
      // step is ~4x cheaper than the accumulate, wants 4 lanes up to 2^17
      // jumps; xoshiro512's step costs as much as half an accumulate: 2 lanes
      if (G::k >= 16)
        parts = total <= (1ull << 13) ? 8u : (total <= (1ull << 17) ? 4u : (total <= (1ull << 18) ? 2u : 1u));
      else
        parts = total <= (1ull << 12) ? 8u : (total <= (1ull << 13) ? 4u : (total <= (1ull << 17) ? 2u : 1u));
    }
    while (parts > 1 && (G::pw % (int)parts) != 0) parts >>= 1;
    q.parts = parts;
  }
  const uint64_t gx = (p.count * q.parts + kJumpThreads - 1) / kJumpThreads;
  if (gx > 0x7fffffffull || nbatch > 65535) return SLP_ERR_INVALID;
  dim3 grid((unsigned)gx, (unsigned)nbatch);
  static BaseStates zero_base;  // unused when p.use_base == 0
  const BaseStates &bs = base ? *base : zero_base;
  if (uniform)
    k_jump<G, true><<<grid, kJumpThreads, 0, st>>>(q, bs);
  else
    k_jump<G, false><<<grid, kJumpThreads, 0, st>>>(q, bs);
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
  constexpr int kTableThreads = JT::threads;
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
#ifndef SLP_K1T_STATES_PER_THREAD
#define SLP_K1T_STATES_PER_THREAD 2  // A/B 1, 2, 4: 2 is 8% faster for xoshiro256, equal elsewhere
#endif
  constexpr uint64_t spt = SLP_K1T_STATES_PER_THREAD;
  const uint64_t cap = (p.m + spt * kTableThreads - 1) / (spt * kTableThreads);
  if (cpc > cap) cpc = cap;
  if (cpc < 1) cpc = 1;
  if (ntab * cpc > 0x7fffffffull) return SLP_ERR_INVALID;
  dim3 grid((unsigned)(ntab * cpc), (unsigned)nbatch, (unsigned)JT::Z);
  kern<<<grid, kTableThreads, smem, st>>>(p, (uint32_t)cpc);
  return check_launch("k_jump_table");
}

}  // namespace dev
}  // namespace slp
