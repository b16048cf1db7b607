// Kernels K2/K3: step + scramble + convert + store (k_fill) and its launchers.
#pragma once

#include <cstdlib>

#include "slp_gen.cuh"

namespace slp {
namespace dev {

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
//   FILL_TMA_G   stream-major rows that do not start 16-byte aligned (odd
//                pitch, unaligned base; TmapGroup in slp_ops.h): row r first
//                emits lead[r % g] outputs with element stores, so its tiles
//                start aligned (32 B for u64); the tile keeps the rows of
//                one parity together ([parity][seg][row / g][128 B], same
//                swizzle) and leaves with g 3-D TMA stores (one per parity);
//                the tail's common sub-blocks run through the tile loop, the
//                rest one output at a time into the same tile;
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

enum { FILL_TMA = 0, FILL_STAGED = 1, FILL_POS = 2, FILL_POS_TMA = 3, FILL_TMA_G = 4 };
template <int MODE>
struct FillTmap {
  using type = CUtensorMap;
};
template <>
struct FillTmap<FILL_TMA_G> {
  using type = TmapGroup;
};
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
    case 5: return FillCfg{4, 1, 16, 32};  // 512 B rows, one buffer (A/B builds only)
    case 6: return FillCfg{6, 1, 16, 32};  // 768 B rows, one buffer (A/B builds with 9 warps)
    case 7: return FillCfg{5, 1, 8, 16};   // 640 B rows, one buffer (A/B builds with 11 warps)
    default: return FillCfg{8, 1, 16, 32};  // 0: 1 KiB rows, one buffer
  }
}
constexpr int kNumFillCfgs = 5;
enum { FILL_KIND_NATIVE = 0, FILL_KIND_CONVERT = 1, FILL_KIND_CHECKSUM = 2, FILL_KIND_SHORT = 3, FILL_KIND_GROUP = 4 };
// row-group TMA (FILL_TMA_G, rows not 16-byte aligned): -DSLP_GROUP_CFG=i
// gives that mode its own tile configuration (A/B); -1 = the tuned one
#ifndef SLP_GROUP_CFG
#define SLP_GROUP_CFG -1
#endif
}  // namespace dev
}  // namespace slp
#include "slp_fill_tuning.h"  // fill_tune(generator id, kind) -> configuration index (measured)
namespace slp {
namespace dev {

// -DSLP_FILL_CFG=i forces configuration i for every kernel (tuning builds,
// profiles/tune_fill.py)
__host__ __device__ constexpr FillCfg fill_cfg(int id, int kind) {
  // short rows (T below one tuned tile): 256-byte pieces, two buffers
  if (kind == FILL_KIND_SHORT) return FillCfg{2, 2, 0, 32};
  if (kind == FILL_KIND_GROUP) return fill_cfg_at(SLP_GROUP_CFG >= 0 ? SLP_GROUP_CFG : 0);
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
__device__ __forceinline__ void tma_store_4d(const CUtensorMap *map, uint32_t src, int x, int y, int z, int w) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];"
               :
               : "l"(reinterpret_cast<uint64_t>(map)), "r"(src), "r"(x), "r"(y), "r"(z), "r"(w)
               : "memory");
}

// element offset of stream-major row (segment) v: (v >> jsh) * ld_out + (v mod J) * T
__device__ __forceinline__ uint64_t sm_row(const FillParams &p, uint64_t v) {
  return (v >> p.jsh) * p.ld_out + (v & ((1ull << p.jsh) - 1)) * p.T;
}
// position-major segment v = j * pm_n + i: (row offset j * T, column i); no split: (0, v)
__device__ __forceinline__ void pm_seg(const FillParams &p, uint64_t v, uint64_t &row_off, uint64_t &col) {
  if (p.pm_n) {
    const uint64_t j = v / p.pm_n;
    row_off = j * p.T;
    col = v - j * p.pm_n;
  } else {
    row_off = 0;
    col = v;
  }
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

// FMA-form site mask of the generator inside k_fill (even / odd outputs).
// Build knobs for A/B: SLP_FILL_MASK[2] (every kind), SLP_FILLC_MASK[2]
// (converted and store + checksum kinds only: the generation-bound ones).
// Default (measured, profiles/round2_ab_fused_sites.md): the ++ scrambler's
// additions with IMAD.X high words (site 32) where generation bounds the fill
// -- store + checksum (+6-7%) and the 8- and 16-word engines (xoshiro512++
// store +3%, converted +5%); everything else keeps the all-ALU forms (the
// HBM-bound native store loses 9% with IMAD.HI multiplies).
template <class G, int OK, bool CSUM>
__host__ __device__ constexpr int fill_site_mask(int odd) {
  int m = G::best_mask(0, 0), m2 = m;
  if constexpr (!G::runtime) {
    if (G::w == 64 && G::sc == SLP_SC_PLUSPLUS && (CSUM || G::k >= 8)) m = m2 = 32;
  }
#ifdef SLP_FILL_MASK
  m = m2 = SLP_FILL_MASK;
#ifdef SLP_FILL_MASK2
  m2 = SLP_FILL_MASK2;
#endif
#endif
#ifdef SLP_FILLC_MASK
  if (CSUM || OK != SLP_OUT_NATIVE) {
    m = m2 = SLP_FILLC_MASK;
#ifdef SLP_FILLC_MASK2
    m2 = SLP_FILLC_MASK2;
#endif
  }
#endif
  return (odd ? m2 : m) & G::kSites;
}

template <class G, int OK, int MODE, bool CSUM = false, bool SHORT = false, bool TAIL = false>
__global__ void __launch_bounds__(kFillThreads)
    k_fill(FillParams p, const __grid_constant__ typename FillTmap<MODE>::type tmap) {
  const G eng = G::load(p.rt);  // run-time parameters (GenR); empty for registry generators
  using word = typename G::word;
  using Cv = Out<OK, word>;
  using bits = typename Cv::bits;
  constexpr int K = G::k;
  constexpr int ES = sizeof(bits);
  using Shape = FillShape<G, SHORT ? (int)FILL_KIND_SHORT
                                   : (MODE == FILL_TMA_G && SLP_GROUP_CFG >= 0 ? (int)FILL_KIND_GROUP
                                                                               : fill_kind<OK, CSUM>())>;
  constexpr int kFillBufs = Shape::bufs, kSegs = Shape::segs, kTileBytes = Shape::tile_bytes;
  constexpr int CH = Shape::row_bytes / ES;                       // outputs per substream per tile
  constexpr int EPC = 16 / ES;                                    // elements per 16-byte chunk
  constexpr int U = Shape::unroll < CH ? Shape::unroll : CH;       // outputs per sub-block
  static_assert(CH % U == 0 && U % EPC == 0 && (U * ES) % 128 == 0, "sub-blocks must be whole 128-byte segments");
  static_assert(!G::ring || U % K == 0, "sub-blocks must cover whole ring periods");
  // 16-byte chunks produced before the buffer wait (at most one sub-block)
  constexpr int PRE = MODE == FILL_POS ? 0 : (Shape::pre * EPC <= U ? Shape::pre : U / EPC);
  // pipe mix of the generator's sites (ALU vs FMA forms, Gen::kSites); MSK2 = odd outputs
  constexpr int MSK = fill_site_mask<G, OK, CSUM>(0), MSK2 = fill_site_mask<G, OK, CSUM>(1);
  const int lane = threadIdx.x & 31;
  const int warp = warp_uniform();  // keeps TMA coordinates in uniform registers
  // shared-tile address of chunk q of piece seg of unit row r: [seg][row] or,
  // for FILL_TMA_G, [parity][seg][row / g] (each parity is one TMA box)
  auto taddr = [&](int seg, int r, int q) -> uint32_t {
    if constexpr (MODE == FILL_TMA_G) {
      const int row = ((r & (tmap.g - 1)) * kSegs + seg) * (32 >> tmap.gsh) + (r >> tmap.gsh);
      return (row << 7) + ((q ^ (row & 7)) << 4);
    } else {
      return swz(seg, r, q);
    }
  };
  // the unit row (substream) this lane generates.  FILL_TMA_G permutes it:
  // lanes 8q..8q+7 (one shared-memory wavefront of STS.128) take eight rows
  // of one parity, whose swizzle keys row / g differ; with lane = row the
  // g rows sharing a key (one per parity) hit the same banks (4-way conflicts
  // for g = 4, profiles/round2 odd32 ncu capture)
  int lrow = lane;
  if constexpr (MODE == FILL_TMA_G) lrow = ((lane & ((32 >> tmap.gsh) - 1)) << tmap.gsh) | (lane >> (5 - tmap.gsh));
  int lead = 0;  // FILL_TMA_G: outputs of this lane's row before its first tile
  if constexpr (MODE == FILL_TMA_G) lead = tmap.lead[lrow & (tmap.g - 1)];
  // FILL_TMA_G, this lane's row: row = lane_row0 + seg * R with R = 32 / g a
  // multiple of 8 (g <= 4, tma_group_ok), so the swizzle key row & 7 is the
  // same for every piece: one multiply-add per chunk instead of recomputing
  // the row and its key (the generic taddr) for every 16-byte store
  uint32_t g_lane_row0 = 0, g_rows_per_seg = 0, g_key = 0;
  if constexpr (MODE == FILL_TMA_G) {
    g_rows_per_seg = 32u >> tmap.gsh;
    g_lane_row0 = (uint32_t)(lrow & (tmap.g - 1)) * kSegs * g_rows_per_seg + (uint32_t)(lrow >> tmap.gsh);
    g_key = g_lane_row0 & 7u;
  }

  extern __shared__ uint8_t smem_raw[];
  uint32_t tiles = 0;
  if constexpr (MODE != FILL_POS)
    tiles = ((smem_u32(smem_raw) + 1023u) & ~1023u) + warp * kFillBufs * kTileBytes;  // 128B-swizzle atoms: 1 KiB

  const word *__restrict__ sin = static_cast<const word *>(p.sin);
  word *sout = static_cast<word *>(p.sout);
  bits *__restrict__ out = static_cast<bits *>(p.out);
  uint64_t ntiles = p.T / CH;
  if constexpr (MODE == FILL_TMA_G) ntiles = (p.T - tmap.lead_max) / CH;  // tiles every row has after its lead
  const uint64_t rem = p.T - ntiles * CH;
  uint32_t issued = 0;  // tiles produced by this warp
  uint64_t pace_next = 0;  // store pacing: earliest issue time (global ns) of this warp's next tile store
  uint64_t cs_lo = 0, cs_hi = 0, cs_x = 0, cs_low = 0;  // CSUM accumulators (zero states emit zeros)

  // the next unit's start states are loaded while this unit is generated
  // (the load latency otherwise stalls every warp at each unit start)
  const uint64_t ustride = (uint64_t)gridDim.x * kFillWarps;
  auto load_states = [&](uint64_t unit, word(&dst)[K]) {
    const uint64_t st = unit * 32 + lrow;
    const bool ok = unit < p.nunits && st < p.nstreams;
#pragma unroll
    for (int j = 0; j < K; ++j) dst[j] = ok ? sin[j * p.ld + st] : (word)0;
  };
  // FILL_TMA_G: one 3-D store per row parity g (skipped where npieces[g] == 0)
  // of the tile whose first piece is piece0 (counted after each row's lead)
  auto store_groups = [&](uint32_t tile, uint64_t row0, uint64_t piece0, const int *npieces) {
    if constexpr (MODE == FILL_TMA_G) {
      // unrolled to the maximum g (4): each store gets its own uniform
      // registers, so no store waits for the previous one to read its operands
#pragma unroll
      for (int g = 0; g < 4; ++g)
        if (g < tmap.g && (!npieces || npieces[g] > 0))
          tma_store_3d(&tmap.m[g], tile + ((g * kSegs * (32 >> tmap.gsh)) << 7), 0, (int)(row0 >> tmap.gsh),
                       (int)piece0);
    }
  };
  word nxt[K];
  load_states((uint64_t)blockIdx.x * kFillWarps + warp, nxt);
  for (uint64_t u = (uint64_t)blockIdx.x * kFillWarps + warp; u < p.nunits; u += ustride) {
    const uint64_t row0 = u * 32;
    const uint64_t stream = row0 + lrow;
    const bool valid = stream < p.nstreams;
    uint64_t pm_roff = 0, pm_col = stream;  // position-major: this lane's segment (row offset, column)
    if constexpr (MODE == FILL_POS || MODE == FILL_POS_TMA) pm_seg(p, stream, pm_roff, pm_col);
    word s[K];
#pragma unroll
    for (int j = 0; j < K; ++j) s[j] = nxt[j];
    load_states(u + ustride, nxt);
    if constexpr (MODE == FILL_TMA_G) {  // the lead: this row's outputs before its 16-byte boundary
      for (int t = 0; t < lead; ++t) {
        const bits x = Cv::conv(eng.next_flat(s));
        if (valid) out[stream * p.ld_out + t] = x;
      }
    }

    // TAIL: a ragged row's last rem < CH outputs form one more tile; its
    // whole sub-blocks run through the same (rolled) code as a full tile
    // (FILL_TMA_G: the same for the tail every row of the warp has after its lead)
    constexpr bool TAIL_LOOP = TAIL || MODE == FILL_TMA_G;
    uint64_t rem_loop = rem;
    if constexpr (MODE == FILL_TMA_G) rem_loop = p.T - tmap.lead_max - ntiles * CH;
    const uint64_t nloop = ntiles + (TAIL_LOOP && rem_loop >= (uint64_t)U ? 1 : 0);
    uint32_t tail_tile = 0;
    for (uint64_t c = 0; c < nloop; ++c) {
      const uint64_t pos0 = c * CH;
      const uint32_t sub_end = (!TAIL_LOOP || c < ntiles) ? (uint32_t)CH : (uint32_t)(rem_loop / U) * U;
      bits *const pos_row = out + (pm_roff + pos0) * p.ld_out + pm_col;  // FILL_POS: row pos0, this lane's column
      uint32_t tile = 0;
      auto wait_buffer = [&] {
        if constexpr (MODE == FILL_TMA || MODE == FILL_POS_TMA || MODE == FILL_TMA_G) {
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
        uint32_t addr;
        if constexpr (MODE == FILL_TMA_G)
          addr = tile + ((g_lane_row0 + ((uint32_t)(b * ES / 128) + (uint32_t)(byte >> 7)) * g_rows_per_seg) << 7) +
                 ((((uint32_t)(byte & 127) >> 4) ^ g_key) << 4);
        else
          addr = tile + ((b * ES / 128) << 12) + swz(byte >> 7, lane, (byte & 127) >> 4);
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
          if ((i & 1) == 0) {  // folded after unrolling
            rr[i] = eng.template output_m<MSK>(s, o);
            eng.template step_m<MSK>(s, o);
          } else {
            rr[i] = eng.template output_m<MSK2>(s, o);
            eng.template step_m<MSK2>(s, o);
          }
          v[i] = Cv::conv(rr[i]);
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
          // predicated stores (no branch per chunk): a branch per chunk let
          // the compiler hoard a sub-block of outputs (255 registers + spills)
          bits *ptr = pos_row + (uint64_t)(b + e) * p.ld_out;
#pragma unroll
          for (int i = 0; i < EPC; ++i) {
            bits *q = ptr + (uint64_t)i * p.ld_out;
            if constexpr (ES == 8)
              asm volatile("{\n\t.reg .pred pv;\n\tsetp.ne.u32 pv, %2, 0;\n\t@pv st.global.b64 [%0], %1;\n\t}" ::"l"(q),
                           "l"((uint64_t)v[i]), "r"((uint32_t)valid)
                           : "memory");
            else
              asm volatile("{\n\t.reg .pred pv;\n\tsetp.ne.u32 pv, %2, 0;\n\t@pv st.global.b32 [%0], %1;\n\t}" ::"l"(q),
                           "r"((uint32_t)v[i]), "r"((uint32_t)valid)
                           : "memory");
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
      for (uint32_t b = U; b < sub_end; b += U) {
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
      if constexpr (TAIL_LOOP) {
        if (c == ntiles) {  // the tail tile: completed and stored below
          tail_tile = tile;
          break;
        }
      }
      if constexpr (MODE == FILL_TMA) {
        fence_proxy_async_smem();
        if (p.pace_ns) pace_store(pace_next, p.pace_ns, p.pace_burst);
        __syncwarp();
        if (elect_one()) {
#ifndef SLP_MEASURE_NO_STORE  // variant builds only: generation without the stores (profiles/nostore_probe.py)
          tma_store_4d(&tmap, tile, 0, (int)(row0 & ((1ull << p.jsh) - 1)), (int)(row0 >> p.jsh),
                       (int)(pos0 * ES / 128));
#endif
          bulk_commit();
        }
        ++issued;
      } else if constexpr (MODE == FILL_POS_TMA) {
        fence_proxy_async_smem();
        if (p.pace_ns) pace_store(pace_next, p.pace_ns, p.pace_burst);
        __syncwarp();
        if (elect_one()) {
          uint64_t roff, col0;
          pm_seg(p, row0, roff, col0);  // a warp's 32 segments share one row block (pm_n % 32 == 0)
          tma_store_2d(&tmap, tile, (int)col0, (int)(roff + pos0));
          bulk_commit();
        }
        ++issued;
      } else if constexpr (MODE == FILL_TMA_G) {
        fence_proxy_async_smem();
        if (p.pace_ns) pace_store(pace_next, p.pace_ns, p.pace_burst);
        __syncwarp();
        if (elect_one()) {
          store_groups(tile, row0, pos0 * ES / 128, nullptr);
          bulk_commit();
        }
        ++issued;

      } else if constexpr (MODE == FILL_STAGED) {
        __syncwarp();
        // element stores.  8-byte outputs go row by row: each warp store is
        // 32 consecutive outputs (256 B) of one row, 3.2 -> 4.7 TB/s for u64
        // against segment-major order.  4-byte outputs keep segment-major
        // order (one 128-byte segment of a row per store), which measured
        // faster for them (2.46 vs 2.20 TB/s, profiles/ragged_bench.py).
        constexpr int CPR = 128 / ES;  // elements per segment
        constexpr int RL = kSegs * CPR;  // outputs per row in the tile
#pragma unroll 4
        for (int f0 = 0; f0 < 32 * RL; f0 += 32) {
          int r, seg, e;
          if constexpr (ES == 8) {
            const int f = f0 + lane;  // (row, column) flattened row-major
            r = f / RL;
            seg = (f % RL) / CPR;
            e = f % CPR;
          } else {
            const int rs = f0 / CPR;  // (segment, row) flattened segment-major, CPR = 32
            seg = rs / 32;
            r = rs % 32;
            e = lane;
          }
          const uint64_t grow = row0 + r;
          bits v;
          const uint32_t addr = tile + swz(seg, r, (e * ES) >> 4) + (e * ES & 15);
          if constexpr (ES == 8) {
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
          } else {
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
          }
          if (grow < p.nstreams) out[grow * p.ld_out + pos0 + seg * CPR + e] = v;
        }
        __syncwarp();
        ++issued;
      }
    }
    if constexpr (MODE == FILL_POS || MODE == FILL_POS_TMA) {
      // tail positions: each store is one coalesced warp row already
      for (uint64_t t = 0; t < rem; ++t) {
        const word r = eng.next_flat(s);
        const bits x = Cv::conv(r);
        if constexpr (CSUM) {
          add128(cs_lo, cs_hi, (uint64_t)r);
          cs_x ^= (uint64_t)r;
          cs_low += (uint32_t)r & (G::w == 64 ? 0x7FFu : 0xFFu);
        }
        if (valid) out[(pm_roff + ntiles * CH + t) * p.ld_out + pm_col] = x;
      }
    } else if constexpr (MODE == FILL_TMA_G) {
      // this row's last T - lead - ntiles*CH outputs (0 .. CH - 1 + lead_max):
      // whole sub-blocks through the tile loop, the rest one at a time into
      // the tile (past CH: element stores); per parity, whole pieces leave by
      // TMA, the partial piece with element stores
      const uint64_t done = ntiles * CH;
      const uint32_t remr = (uint32_t)(p.T - lead - done);
      const uint32_t rem_w = (uint32_t)(p.T - done);  // the largest (lead 0) in the warp
      if (rem_w > 0) {
        // whole sub-blocks common to every row already ran in the tile loop
        const uint32_t rb = rem_loop >= (uint64_t)U ? (uint32_t)(rem_loop / U) * U : 0u;
        uint32_t tile = tail_tile;
        if (rb == 0) {
          tile = tiles + (issued % kFillBufs) * kTileBytes;
          if (issued >= kFillBufs && elect_one()) bulk_wait_read<kFillBufs - 1>();
          __syncwarp();
        }
        for (uint32_t t = rb; t < remr; ++t) {
          const bits x = Cv::conv(eng.next_flat(s));
          if (t < (uint32_t)CH) {
            const uint32_t byte = t * ES;
            const uint32_t addr = tile + taddr(byte >> 7, lrow, (byte & 127) >> 4) + (byte & 15);
            if constexpr (ES == 8)
              asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"((uint64_t)x) : "memory");
            else
              asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"((uint32_t)x) : "memory");
          } else if (valid) {
            out[stream * p.ld_out + lead + done + t] = x;
          }
        }
        constexpr int CPR = 128 / ES;  // elements per 128-byte piece
        int npieces[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        bool any = false;
        for (int g = 0; g < tmap.g; ++g) {
          const uint64_t rg = p.T - tmap.lead[g] - done;
          npieces[g] = (int)((rg < (uint64_t)CH ? rg : (uint64_t)CH) / CPR);
          any |= npieces[g] > 0;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (any) {
          if (elect_one()) {
            store_groups(tile, row0, done * ES / 128, npieces);
            bulk_commit();
          }
          ++issued;
        }
        // partial pieces: columns [npieces * CPR, min(rem, CH)) of each row;
        // pieces below every parity's npieces went out whole by TMA
        const uint32_t lim_w = rem_w < (uint32_t)CH ? rem_w : (uint32_t)CH;
        constexpr int RPP = 32 / CPR;
        const int nseg = (int)((lim_w + CPR - 1) / CPR);
        int seg_lo = npieces[0];
        for (int g = 1; g < tmap.g; ++g) seg_lo = npieces[g] < seg_lo ? npieces[g] : seg_lo;
        for (int r0 = 32 * seg_lo; r0 < 32 * nseg; r0 += RPP) {
          const int rs = r0 + lane / CPR;  // (piece, row) flattened piece-major
          const int seg = rs / 32, r = rs % 32;
          const int e = lane % CPR;
          const int rl = tmap.lead[r & (tmap.g - 1)];
          const uint64_t rr = p.T - rl - done;
          const uint64_t lim = rr < (uint64_t)CH ? rr : (uint64_t)CH;
          const uint64_t col = (uint64_t)seg * CPR + e;
          const uint64_t grow = row0 + r;
          if (col >= (lim / CPR) * CPR && col < lim && grow < p.nstreams) {
            bits v;
            const uint32_t addr = tile + taddr(seg, r, (e * ES) >> 4) + (e * ES & 15);
            if constexpr (ES == 8) {
              asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
            } else {
              asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
            }
            out[grow * p.ld_out + rl + done + col] = v;
          }
        }
        __syncwarp();
      }
    } else if constexpr (TAIL) {
      if (rem > 0) {
        // the tail tile: whole sub-blocks came from the loop above; the last
        // rem % U outputs are generated one at a time into the same tile.  Its
        // whole 128-byte pieces leave with the TMA store (the tensor map ends
        // at the last whole piece of a row and clips the box); the final
        // partial piece leaves with element stores.
        const uint32_t rb = rem >= (uint64_t)U ? (uint32_t)(rem / U) * U : 0u;
        uint32_t tile = tail_tile;
        if (rb == 0) {
          tile = tiles + (issued % kFillBufs) * kTileBytes;
          if constexpr (MODE == FILL_TMA) {
            if (issued >= kFillBufs && elect_one()) bulk_wait_read<kFillBufs - 1>();
          }
          __syncwarp();
        }
        for (uint32_t t = rb; t < (uint32_t)rem; ++t) {
          const bits x = Cv::conv(eng.next_flat(s));
          const uint32_t byte = t * ES;
          const uint32_t addr = tile + swz(byte >> 7, lane, (byte & 127) >> 4) + (byte & 15);
          if constexpr (ES == 8)
            asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"((uint64_t)x) : "memory");
          else
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"((uint32_t)x) : "memory");
        }
        constexpr int CPR = 128 / ES;  // elements per 128-byte piece
        constexpr int RPP = 32 / CPR;  // rows per pass
        int seg0 = 0;
        if constexpr (MODE == FILL_TMA) {
          seg0 = (int)(rem / CPR);
          if (seg0 > 0) {
            fence_proxy_async_smem();
            __syncwarp();
            if (elect_one()) {
              tma_store_4d(&tmap, tile, 0, (int)(row0 & ((1ull << p.jsh) - 1)), (int)(row0 >> p.jsh),
                           (int)(ntiles * CH * ES / 128));
              bulk_commit();
            }
            ++issued;  // only a committed store owns its buffer (bulk_wait_read counts groups)
          }
        }
        __syncwarp();
        const int nseg = (int)((rem + CPR - 1) / CPR);
        for (int r0 = 32 * seg0; r0 < 32 * nseg; r0 += RPP) {
          const int rs = r0 + lane / CPR;  // (piece, row) flattened piece-major
          const int seg = rs / 32, r = rs % 32;
          const int e = lane % CPR;
          const uint64_t col = (uint64_t)seg * CPR + e;
          const uint64_t grow = row0 + r;
          if (col < rem && grow < p.nstreams) {
            bits v;
            const uint32_t addr = tile + swz(seg, r, (e * ES) >> 4) + (e * ES & 15);
            if constexpr (ES == 8) {
              asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
            } else {
              asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
            }
            out[sm_row(p, grow) + ntiles * CH + col] = v;
          }
        }
        __syncwarp();
      }
    } else if constexpr (CSUM) {
      if (rem > 0) {
      // stream-major tail (T not a multiple of the tile): the last rem < CH
      // outputs of each row go through the warp's tile right after its last
      // tile and leave with coalesced element stores (the store + checksum
      // instance; the fill's TAIL instance above reuses the tile loop).
      const uint32_t tile = tiles + (issued % kFillBufs) * kTileBytes;
      if constexpr (MODE == FILL_TMA) {
        if (issued >= kFillBufs && elect_one()) bulk_wait_read<kFillBufs - 1>();
      }
      __syncwarp();
      for (uint32_t t = 0; t < (uint32_t)rem; ++t) {
        const word r = eng.next_flat(s);
        const bits x = Cv::conv(r);
        if constexpr (CSUM) {
          add128(cs_lo, cs_hi, (uint64_t)r);
          cs_x ^= (uint64_t)r;
          cs_low += (uint32_t)r & (G::w == 64 ? 0x7FFu : 0xFFu);
        }
        const uint32_t byte = t * ES;
        const uint32_t addr = tile + swz(byte >> 7, lane, (byte & 127) >> 4) + (byte & 15);
        if constexpr (ES == 8)
          asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"((uint64_t)x) : "memory");
        else
          asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"((uint32_t)x) : "memory");
      }
      __syncwarp();
      constexpr int CPR = 128 / ES;  // elements per 128-byte segment
      constexpr int RPP = 32 / CPR;  // rows per pass
      const int nseg = (int)((rem + CPR - 1) / CPR);
      for (int r0 = 0; r0 < 32 * nseg; r0 += RPP) {
        const int rs = r0 + lane / CPR;  // (segment, row) flattened segment-major
        const int seg = rs / 32, r = rs % 32;
        const int e = lane % CPR;
        const uint64_t col = (uint64_t)seg * CPR + e;
        const uint64_t grow = row0 + r;
        if (col < rem && grow < p.nstreams) {
          bits v;
          const uint32_t addr = tile + swz(seg, r, (e * ES) >> 4) + (e * ES & 15);
          if constexpr (ES == 8) {
            asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
          } else {
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
          }
          out[sm_row(p, grow) + ntiles * CH + col] = v;
        }
      }
      __syncwarp();
      }
    }
    if (valid && sout) {
#pragma unroll
      for (int j = 0; j < K; ++j) sout[j * p.ld + stream] = s[j];
    }
  }
  if constexpr (MODE == FILL_TMA || MODE == FILL_POS_TMA || MODE == FILL_TMA_G) {
    if (elect_one()) bulk_wait_all<0>();
  }
  if constexpr (CSUM) reduce_checksum_block<kFillWarps>(cs_lo, cs_hi, cs_x, cs_low, 0.0, p.partials);
}


// ---- host launchers ----------------------------------------------------------------

// Position-major, 4-byte outputs (32-bit generators, native or f32): with one
// substream per lane a warp's row piece is only 128 bytes (4.2 TB/s).  Here
// each lane runs TWO substreams (row0 + lane and row0 + 32 + lane), so a
// warp's tile is [64 positions][64 substreams] (256-byte rows) and leaves with
// one 2-D TMA store of 64 x 64; two 16 KB buffers per warp.
constexpr int kPm2Pos = 64;
constexpr int kPm2TileBytes = kPm2Pos * 64 * 4;

// store pacing period (pace_store): `units` units of work spread over `agents`
// (warps) that each store `tiles_per_unit` tiles of `tile_bytes` per unit and
// read / write `state_bytes` of substream states per unit.  The target rate
// (fill_pace_gbps) is in bytes of output + 1.5 x bytes of state traffic per
// ns: state reads mixed into the write stream cost about 1.5x their bytes
// (best paced rates measured for rows of 64, 128 and 1024 outputs and the
// 16-word xoroshiro1024 states all fit that, profiles/round2_pace_short.jsonl,
// round2_pace_x.jsonl).  Position-major tiles (8 MiB-apart rows of 256 B)
// congest earlier and are paced at 95% of it.  The busiest agent stores
// ceil(units / agents) x tiles_per_unit tiles in the target time.  0 = unpaced.
inline uint32_t pace_period_ns(uint64_t units, uint64_t agents, uint64_t tiles_per_unit, uint64_t tile_bytes,
                               uint64_t state_bytes, bool position_major = false) {
  int gbps = fill_pace_gbps();
  if (position_major) gbps = gbps * 95 / 100;
  if (gbps <= 0 || !units || !agents || !tiles_per_unit) return 0;
  const uint64_t tiles_max = (units + agents - 1) / agents * tiles_per_unit;
  const double ns = (double)units * ((double)tiles_per_unit * tile_bytes + 1.5 * (double)state_bytes) / gbps;
  return (uint32_t)(ns / (double)tiles_max);
}
constexpr int kPm2Smem = kFillWarps * 2 * kPm2TileBytes + 1024;

template <class G, int OK>
__global__ void __launch_bounds__(kFillThreads) k_fill_pm2(FillParams p, const __grid_constant__ CUtensorMap tmap) {
  const G eng = G::load(p.rt);
  using word = typename G::word;
  using Cv = Out<OK, word>;
  using bits = typename Cv::bits;
  constexpr int K = G::k;
  static_assert(sizeof(bits) == 4 && kPm2Pos % K == 0, "4-byte outputs, whole ring periods");
  constexpr int MSK = G::best_mask(0, 0);
  const int lane = threadIdx.x & 31;
  const int warp = warp_uniform();
  extern __shared__ uint8_t smem_raw[];
  const uint32_t tiles = ((smem_u32(smem_raw) + 1023u) & ~1023u) + warp * 2 * kPm2TileBytes;
  const word *__restrict__ sin = static_cast<const word *>(p.sin);
  word *sout = static_cast<word *>(p.sout);
  bits *__restrict__ out = static_cast<bits *>(p.out);
  const uint64_t ntiles = p.T / kPm2Pos, rem = p.T - ntiles * kPm2Pos;
  const uint64_t nunits = (p.nstreams + 63) / 64;
  uint32_t issued = 0;
  uint64_t pace_next = 0;  // store pacing (pace_store)
  for (uint64_t u = (uint64_t)blockIdx.x * kFillWarps + warp; u < nunits; u += (uint64_t)gridDim.x * kFillWarps) {
    const uint64_t row0 = u * 64;
    const uint64_t stA = row0 + lane, stB = row0 + 32 + lane;
    const bool vA = stA < p.nstreams, vB = stB < p.nstreams;
    word a[K], b[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      a[j] = vA ? sin[j * p.ld + stA] : (word)0;
      b[j] = vB ? sin[j * p.ld + stB] : (word)0;
    }
    for (uint64_t c = 0; c < ntiles; ++c) {
      const uint32_t tile = tiles + (issued & 1) * kPm2TileBytes;
      if (issued >= 2 && elect_one()) bulk_wait_read<1>();
      __syncwarp();
#pragma unroll
      for (int t = 0; t < kPm2Pos; ++t) {
        const int o = t % K;
        const bits xa = Cv::conv(eng.template output_m<MSK>(a, o));
        eng.template step_m<MSK>(a, o);
        const bits xb = Cv::conv(eng.template output_m<MSK>(b, o));
        eng.template step_m<MSK>(b, o);
        const uint32_t row = tile + t * 256 + lane * 4;
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(row), "r"((uint32_t)xa) : "memory");
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(row + 128), "r"((uint32_t)xb) : "memory");
      }
      fence_proxy_async_smem();
      if (p.pace_ns) pace_store(pace_next, p.pace_ns, p.pace_burst);
      __syncwarp();
      if (elect_one()) {
        uint64_t roff, col0;
        pm_seg(p, row0, roff, col0);  // a warp's 64 segments share one row block (pm_n % 64 == 0)
        tma_store_2d(&tmap, tile, (int)col0, (int)(roff + c * kPm2Pos));
        bulk_commit();
      }
      ++issued;
    }
    for (uint64_t t = 0; t < rem; ++t) {  // tail positions: coalesced warp rows
      const bits xa = Cv::conv(eng.next_flat(a));
      const bits xb = Cv::conv(eng.next_flat(b));
      const uint64_t pos = ntiles * kPm2Pos + t;
      uint64_t ra, ca, rb, cb;
      pm_seg(p, stA, ra, ca);
      pm_seg(p, stB, rb, cb);
      if (vA) out[(ra + pos) * p.ld_out + ca] = xa;
      if (vB) out[(rb + pos) * p.ld_out + cb] = xb;
    }
    if (sout) {
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (vA) sout[j * p.ld + stA] = a[j];
        if (vB) sout[j * p.ld + stB] = b[j];
      }
    }
  }
  if (elect_one()) bulk_wait_all<0>();
}

template <class G, int OK>
int launch_fill_pm2(const FillParams &p, cudaStream_t st) {
  CUtensorMap tmap;
  memset(&tmap, 0, sizeof tmap);
  const uint64_t rows = p.pm_n ? p.T * (p.nstreams / p.pm_n) : p.T, cols = p.pm_n ? p.pm_n : p.nstreams;
  int rc = make_store_tmap_pm(&tmap, p.out, 4, rows, cols, p.ld_out, kPm2Pos, 64);
  if (rc != SLP_OK) return rc;
  auto kern = k_fill_pm2<G, OK>;
  const int dev = current_device();
  static std::atomic<int> attr_set[64];
  if (dev < 0 || dev >= 64) return SLP_ERR_CUDA;
  if (!attr_set[dev]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kPm2Smem) != cudaSuccess)
      return cuda_fail("cudaFuncSetAttribute(pm2)");
    attr_set[dev] = 1;
  }
  const uint64_t nunits = (p.nstreams + 63) / 64;
  if (nunits == 0 || p.T == 0) return SLP_OK;
  const uint64_t want = (nunits + kFillWarps - 1) / kFillWarps;
  const uint64_t cap = (uint64_t)sm_count(dev) * fill_grid_mult();
  const unsigned grid = (unsigned)(want < cap ? want : cap);
  FillParams q = p;
  q.pace_ns = pace_period_ns(nunits, (uint64_t)grid * kFillWarps, p.T / kPm2Pos, kPm2TileBytes,
                             64ull * G::k * sizeof(typename G::word) * (p.sout ? 2 : 1), true);
  q.pace_burst = (uint32_t)fill_pace_burst();
  kern<<<grid, kFillThreads, kPm2Smem, st>>>(q, tmap);
  return check_launch("k_fill_pm2");
}

// Position-major rows that no TMA tensor map can address (odd pitch for
// 8-byte outputs, pitch % 4 != 0 for 4-byte outputs, unaligned base): with
// one coalesced warp store per output, every warp's 32-element row piece
// starts and ends inside a 32-byte sector, and each such partial-sector write
// costs a DRAM read-modify-write (ncu: 0.90 GB of DRAM reads per 8 GiB
// fill, 2.4 TB/s; profiles/round2_pm_odd_ncu.csv).  Here the CTA's 7 warps
// (224 consecutive substreams) stage CH positions in shared memory, each
// row laid out at the same offset modulo 16 as in global memory; then one
// thread writes the 32-byte-aligned interior of every row with a 1-D bulk
// copy (cp.async.bulk.global.shared::cta: whole sectors only) and a few
// threads store the 0-3 edge elements at each end.  Partial sectors remain
// only at CTA boundaries (2 per 224 outputs instead of 2 per 32).
constexpr int kPosCtaCH = 16;  // positions per tile (2 x 30 KB buffers: 3 CTAs per SM overlap their phases)

template <int ES>
struct PosCta {
  static constexpr int W = kFillWarps * 32;                  // substreams per CTA
  static constexpr int ROW = ((W * ES + 32 + 127) / 128) * 128;  // smem bytes per row (+ offset room)
  static constexpr int TILE = kPosCtaCH * ROW;
  static constexpr int SMEM = 2 * TILE + 128;
};

template <class G, int OK>
__global__ void __launch_bounds__(kFillThreads) k_fill_pos_cta(FillParams p) {
  const G eng = G::load(p.rt);
  using word = typename G::word;
  using Cv = Out<OK, word>;
  using bits = typename Cv::bits;
  constexpr int K = G::k;
  constexpr int ES = sizeof(bits);
  using PC = PosCta<ES>;
  constexpr int CH = kPosCtaCH;
  static_assert(CH % K == 0, "tiles must cover whole ring periods");
  extern __shared__ uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 127u) & ~127u;
  uint8_t *sgen = smem_raw + (sbase - smem_u32(smem_raw));  // generic pointer of sbase
  const int tid = threadIdx.x;
  const word *__restrict__ sin = static_cast<const word *>(p.sin);
  word *sout = static_cast<word *>(p.sout);
  bits *__restrict__ out = static_cast<bits *>(p.out);
  const uint64_t nblk = (p.nstreams + PC::W - 1) / PC::W;
  const uint64_t ntiles = (p.T + CH - 1) / CH;
  uint32_t issued = 0;
  for (uint64_t cb = blockIdx.x; cb < nblk; cb += gridDim.x) {
    const uint64_t c0 = cb * PC::W;
    const uint64_t stream = c0 + tid;
    const bool valid = stream < p.nstreams;
    const int wcols = (int)(p.nstreams - c0 < (uint64_t)PC::W ? p.nstreams - c0 : PC::W);
    word s[K];
#pragma unroll
    for (int j = 0; j < K; ++j) s[j] = valid ? sin[j * p.ld + stream] : (word)0;
    for (uint64_t c = 0; c < ntiles; ++c) {
      const uint64_t pos0 = c * CH;
      const int rows = (int)(p.T - pos0 < (uint64_t)CH ? p.T - pos0 : CH);
      const uint32_t buf = (issued & 1) * PC::TILE;
      // the bulk stores of the tile two back (issued by lane 0 of every warp)
      // must have read this buffer
      if (issued >= 2 && (tid & 31) == 0) bulk_wait_read<1>();
      __syncthreads();
      // row t of the tile starts at global byte g_row0 + t * pitch; in shared
      // memory at the same offset modulo 16
      const uint64_t pitch = p.ld_out * ES;
      const uint64_t g_row0 = (uint64_t)(out + pos0 * p.ld_out + c0);
      if (rows == CH) {
#pragma unroll
        for (int t = 0; t < CH; ++t) {
          const bits x = Cv::conv(eng.output(s, t % K));
          eng.step(s, t % K);
          const uint32_t a = buf + t * PC::ROW + (uint32_t)((g_row0 + t * pitch) & 15) + tid * ES;
          if constexpr (ES == 8)
            asm volatile("st.shared.b64 [%0], %1;" ::"r"(sbase + a), "l"((uint64_t)x) : "memory");
          else
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(sbase + a), "r"((uint32_t)x) : "memory");
        }
      } else {
        for (int t = 0; t < rows; ++t) {  // last, partial tile: scalar steps keep flat order
          const bits x = Cv::conv(eng.next_flat(s));
          const uint32_t a = buf + t * PC::ROW + (uint32_t)((g_row0 + t * pitch) & 15) + tid * ES;
          if constexpr (ES == 8)
            asm volatile("st.shared.b64 [%0], %1;" ::"r"(sbase + a), "l"((uint64_t)x) : "memory");
          else
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(sbase + a), "r"((uint32_t)x) : "memory");
        }
      }
      fence_proxy_async_smem();
      __syncthreads();
      // row t: global bytes [g0, g1); interior [A, B) = whole 32-byte sectors;
      // lane 0 of warp w issues the rows t = w mod kFillWarps
      if ((tid & 31) == 0) {
        for (int t = tid >> 5; t < rows; t += kFillWarps) {
          const uint64_t g0 = g_row0 + t * pitch, g1 = g0 + (uint64_t)wcols * ES;
          const uint64_t A = (g0 + 31) & ~31ull, B = g1 & ~31ull;
          if (B > A) {
            const uint32_t src = sbase + buf + t * PC::ROW + (uint32_t)(g0 & 15) + (uint32_t)(A - g0);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(A), "r"(src),
                         "r"((uint32_t)(B - A))
                         : "memory");
          }
        }
        bulk_commit();
      }
      // edges: elements outside [A, B), at most 3 (7 for 4-byte outputs) per end and row
      constexpr int EPS = 32 / ES;  // elements per sector
      for (int q = tid; q < rows * 2 * EPS; q += kFillThreads) {
        const int t = q / (2 * EPS), r = q % (2 * EPS);
        const uint64_t g0 = g_row0 + t * pitch, g1 = g0 + (uint64_t)wcols * ES;
        const uint64_t A = (g0 + 31) & ~31ull, B = g1 & ~31ull;
        // head: elements before A; tail: elements from B on (without an
        // interior, B <= A, the piece is shorter than 64 bytes: head and tail
        // together cover its < 2 * EPS elements)
        int e;
        if (r < EPS) {
          e = r;
          if (B > A && g0 + (uint64_t)e * ES >= A) continue;
        } else {
          e = (B > A ? (int)((B - g0) / ES) : EPS) + (r - EPS);
        }
        if (e >= wcols) continue;
        const uint32_t a = sbase + buf + t * PC::ROW + (uint32_t)(g0 & 15) + e * ES;
        bits v;
        if constexpr (ES == 8)
          asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
        else
          asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
        out[(pos0 + t) * p.ld_out + c0 + e] = v;
      }
      ++issued;
    }
    if (valid && sout) {
#pragma unroll
      for (int j = 0; j < K; ++j) sout[j * p.ld + stream] = s[j];
    }
  }
  if ((tid & 31) == 0) bulk_wait_all<0>();
}

template <class G, int OK>
int launch_fill_pos_cta(const FillParams &p, cudaStream_t st) {
  using bits = typename Out<OK, typename G::word>::bits;
  using PC = PosCta<(int)sizeof(bits)>;
  auto kern = k_fill_pos_cta<G, OK>;
  const int dev = current_device();
  static std::atomic<int> per_sm[64];
  if (dev < 0 || dev >= 64) return SLP_ERR_CUDA;
  if (!per_sm[dev]) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PC::SMEM) != cudaSuccess)
      return cuda_fail("cudaFuncSetAttribute(pos_cta)");
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, kFillThreads, PC::SMEM) != cudaSuccess || b < 1)
      return cuda_fail("occupancy(pos_cta)");
    per_sm[dev] = b;
  }
  const uint64_t nblk = (p.nstreams + PC::W - 1) / PC::W;
  if (nblk == 0 || p.T == 0) return SLP_OK;
  const uint64_t cap = (uint64_t)sm_count(dev) * per_sm[dev] * fill_grid_mult();
  const unsigned grid = (unsigned)(nblk < cap ? nblk : cap);
  // (not paced: measured 8-18% slower paced; the kernel is generation-bound)
  FillParams q = p;
  q.pace_ns = 0;
  kern<<<grid, kFillThreads, PC::SMEM, st>>>(q);
  return check_launch("k_fill_pos_cta");
}

template <class G, int OK, int MODE, bool CSUM = false, bool SHORT = false, bool TAIL = false>
int launch_fill(const FillParams &p0, cudaStream_t st, int *grid_out = nullptr) {
  using Shape = FillShape<G, SHORT ? (int)FILL_KIND_SHORT
                                   : (MODE == FILL_TMA_G && SLP_GROUP_CFG >= 0 ? (int)FILL_KIND_GROUP
                                                                               : fill_kind<OK, CSUM>())>;
  using bits = typename Out<OK, typename G::word>::bits;
  constexpr int ES = sizeof(bits);
  FillParams p = p0;
  if (grid_out) *grid_out = 0;
  if constexpr ((MODE == FILL_TMA || MODE == FILL_STAGED) && !CSUM && !TAIL) {
    if (p.T % (Shape::row_bytes / ES) != 0) return launch_fill<G, OK, MODE, false, SHORT, true>(p, st, grid_out);
  }
  typename FillTmap<MODE>::type tmap;
  memset(&tmap, 0, sizeof tmap);
  if constexpr (MODE == FILL_TMA) {
    int rc = make_store_tmap(&tmap, p.out, ES, p.T, p.nstreams, p.ld_out, Shape::segs, (int)p.jsh);
    if (rc != SLP_OK) return rc;
  } else if constexpr (MODE == FILL_TMA_G) {
    int rc = make_store_tmap_group(&tmap, p.out, ES, p.T, p.nstreams, p.ld_out, Shape::segs);
    if (rc != SLP_OK) return rc;
  } else if constexpr (MODE == FILL_POS_TMA) {
    const uint64_t rows = p.pm_n ? p.T * (p.nstreams / p.pm_n) : p.T, cols = p.pm_n ? p.pm_n : p.nstreams;
    int rc = make_store_tmap_pm(&tmap, p.out, ES, rows, cols, p.ld_out,
                                Shape::row_bytes / ES);
    if (rc != SLP_OK) return rc;
  }
  auto kern = k_fill<G, OK, MODE, CSUM, SHORT, TAIL>;
  const int smem = MODE == FILL_POS ? 0 : Shape::smem;
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
  p.pace_ns = 0;
  // (not paced, measured slower paced: row-group rows of 4-byte outputs (3-6%)
  // and store + checksum, which is generation-bound (up to 8%))
  if constexpr (!CSUM && (MODE == FILL_TMA || MODE == FILL_POS_TMA || (MODE == FILL_TMA_G && ES == 8))) {
    const uint64_t tiles_per_unit = (p.T + Shape::row_bytes / ES - 1) / (Shape::row_bytes / ES);
    p.pace_ns = pace_period_ns(p.nunits, (uint64_t)grid * kFillWarps, tiles_per_unit, Shape::tile_bytes,
                               32ull * G::k * sizeof(typename G::word) * (p.sout ? 2 : 1), MODE == FILL_POS_TMA);
    p.pace_burst = (uint32_t)fill_pace_burst();
  }
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
  // position-major segment split (pm_n > 0): the output is [pm_rows][ld_out];
  // a TMA box covers one row block only when a warp's segments share it
  const uint64_t pm_rows = p.pm_n ? p.T * (p.nstreams / p.pm_n) : p.T;
  const uint64_t pm_cols = p.pm_n ? p.pm_n : p.nstreams;
  if constexpr (W == 32) {
    // position-major 4-byte outputs: two substreams per lane, 256-byte rows
    if (layout == SLP_POSITION_MAJOR && es == 4 && (!p.pm_n || p.pm_n % 64 == 0) &&
        tma_ok_pm(p.out, 4, pm_rows, pm_cols, p.ld_out, kPm2Pos)) {
      if (ok == SLP_OUT_F32) return launch_fill_pm2<G, SLP_OUT_F32>(p, st);
      return launch_fill_pm2<G, SLP_OUT_NATIVE>(p, st);
    }
  }
  int mode;
  if (layout == SLP_POSITION_MAJOR)
    mode = (!p.pm_n || p.pm_n % 32 == 0) &&
                   tma_ok_pm(p.out, es, pm_rows, pm_cols, p.ld_out,
                             fill_cfg(G::id, ok == SLP_OUT_NATIVE ? FILL_KIND_NATIVE : FILL_KIND_CONVERT).segs * 128 / es)
               ? FILL_POS_TMA
               : FILL_POS;
  else if (layout != SLP_STREAM_MAJOR)
    return SLP_ERR_INVALID;
  // stream-major rows shorter than one tuned tile take the short shape
  // (256-byte pieces): otherwise every output would go through the tail path
  const int segs = fill_cfg(G::id, ok == SLP_OUT_NATIVE ? FILL_KIND_NATIVE : FILL_KIND_CONVERT).segs;
  const bool short_rows = layout == SLP_STREAM_MAJOR && p.T < (uint64_t)segs * 128 / es;
  if (layout == SLP_STREAM_MAJOR) {
    const int ssegs = short_rows ? fill_cfg(0, FILL_KIND_SHORT).segs : segs;
    const int gsegs = short_rows || SLP_GROUP_CFG < 0 ? ssegs : fill_cfg(0, FILL_KIND_GROUP).segs;
    mode = tma_ok(p.out, es, p.T, p.nstreams, p.ld_out, ssegs)
               ? FILL_TMA
               : (tma_group_ok(p.out, es, p.T, p.nstreams, p.ld_out, gsegs) ? FILL_TMA_G : FILL_STAGED);
    // stream-major segment rows (jsh > 0) are addressed through the 4-D store map only
    if (p.jsh && (mode != FILL_TMA || short_rows)) return SLP_ERR_UNSUPPORTED;
  }
  // rows no TMA map can address: the CTA-staged sector-aligned path (no split)
  static const bool pos_cta_off = std::getenv("SLP_POS_CTA_OFF") != nullptr;  // A/B: element stores
  if (mode == FILL_POS && !p.pm_n && ((uintptr_t)p.out % es) == 0 && !pos_cta_off) {
    if constexpr (W == 64) {
      if (ok == SLP_OUT_F64) return launch_fill_pos_cta<G, SLP_OUT_F64>(p, st);
      return launch_fill_pos_cta<G, SLP_OUT_NATIVE>(p, st);
    } else {
      if (ok == SLP_OUT_F32) return launch_fill_pos_cta<G, SLP_OUT_F32>(p, st);
      if (ok == SLP_OUT_U64) return launch_fill_pos_cta<G, SLP_OUT_U64>(p, st);
      return launch_fill_pos_cta<G, SLP_OUT_NATIVE>(p, st);
    }
  }
#define SLP_FILL_CASE(OKV)                                                                              \
  if (ok == OKV) {                                                                                      \
    if (mode == FILL_TMA)                                                                               \
      return short_rows ? launch_fill<G, OKV, FILL_TMA, false, true>(p, st)                             \
                        : launch_fill<G, OKV, FILL_TMA>(p, st);                                         \
    if (mode == FILL_TMA_G)                                                                             \
      return short_rows ? launch_fill<G, OKV, FILL_TMA_G, false, true>(p, st)                           \
                        : launch_fill<G, OKV, FILL_TMA_G>(p, st);                                       \
    if (mode == FILL_STAGED)                                                                            \
      return short_rows ? launch_fill<G, OKV, FILL_STAGED, false, true>(p, st)                          \
                        : launch_fill<G, OKV, FILL_STAGED>(p, st);                                      \
    if (mode == FILL_POS_TMA) return launch_fill<G, OKV, FILL_POS_TMA>(p, st);                          \
    return launch_fill<G, OKV, FILL_POS>(p, st);                                                        \
  }  /* ragged T: launch_fill redirects to its TAIL instance */
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

}  // namespace dev
}  // namespace slp
