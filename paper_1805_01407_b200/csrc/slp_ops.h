// Launch-parameter structs and the per-generator dispatch table shared by the
// kernel instantiation units (slp_inst_*.cu) and the C ABI (slp_api.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace slp {

// Run-time generator parameters (custom_spec engines, generators.py:127-135):
// read by the GenR<> kernel instances (slp_gen.cuh), ignored by the
// registry instances, whose parameters are template constants.
struct GenRt {
  uint32_t a, b, c;     // engine shift/rotation amounts (engines.py:100-140)
  int32_t sc, wi, wj;   // scrambler kind (SLP_SC_*) and flat word indices (wj < 0: unused)
  uint32_t R;           // scrambler rotation (++ and **)
  uint64_t S, T;        // scrambler multipliers (* and **)
  uint32_t one, one2;   // = 1, opaque to ptxas: multipliers 2^r for FMA-pipe rotations (Gen::rot)
};

struct FillParams {
  const void *sin;   // SoA states [k][ld]
  void *sout;        // may alias sin; nullptr = no write-back
  uint64_t ld;
  uint64_t nstreams;
  uint64_t T;
  void *out;
  uint64_t ld_out;
  uint64_t nunits;   // filled by the launcher
  void *partials;           // store+checksum mode: slp_checksum[grid]
  size_t workspace_bytes;
  GenRt rt;                // run-time generator parameters (custom engines)
  // segment split (slp_fill for few, long substreams): the nstreams rows are
  // segments of n = nstreams >> jsh real substreams, T outputs each.
  // Stream-major: segment v = i * J + j (J = 1 << jsh) is row i, columns
  // [j * T, (j + 1) * T): element offset (v >> jsh) * ld_out + (v & (J - 1)) * T.
  // Position-major (pm_n = n > 0): segment v = j * n + i is column i, rows
  // [j * T, (j + 1) * T).  jsh = 0 and pm_n = 0: no split.
  uint32_t jsh;
  uint64_t pm_n;
  // store pacing (TMA modes of k_fill): minimum ns between one warp's tile
  // stores, set by the launcher from the target rate (0 = unpaced)
  uint32_t pace_ns;
  uint32_t pace_burst;  // periods a late warp may catch up (pace_store)
};

struct FusedParams {
  const void *sin;
  void *sout;
  uint64_t ld;
  uint64_t nstreams;
  uint64_t T;
  void *partials;          // slp_checksum[grid]
  size_t workspace_bytes;  // bytes available at partials
  uint64_t nunits;
  uint32_t one;            // = 1, opaque to ptxas (keeps accumulations on IMAD)
  GenRt rt;                // run-time generator parameters (custom engines)
};

struct JumpParams {
  const void *src;
  uint64_t ld_src;
  void *dst;
  uint64_t ld_dst;
  const uint64_t *polys;  // device, G::pw words per polynomial
  uint64_t poly0;
  int pmode;              // 0: poly0 for all, 1: poly0 + t / m, 2: poly0 + t
  int use_base;           // source state = BaseStates entry of the batch
  uint64_t count;         // states per batch
  uint64_t m;             // source index t % m (0: t)
  uint64_t src_off, dst_off, batch_stride;
  uint64_t src_batch_stride;  // source states per batch (0: batch_stride)
  uint64_t fold;              // > 0: batches folded into t (batch t / fold, index t % fold), grid.y = 1
  int pw_used;            // polynomial words actually used (0 = all); trims the loop for low-degree polys
  uint32_t parts;         // lanes per jump (k_jump's latency split; set by jump_impl, 0 = 1)
  GenRt rt;                // run-time generator parameters (custom engines)
};

// table-driven uniform jump (kernel K1t): dst[dst_off + t] = src[src_off + t % m]
// jumped by table (table0 + t / m), t < count; tables from build_table
struct TableJumpParams {
  const void *src;
  uint64_t ld_src;
  void *dst;
  uint64_t ld_dst;
  const uint32_t *tables;  // device, table_words() uint32 per table
  uint64_t table0;
  uint64_t count, m;
  uint64_t src_off, dst_off, batch_stride;
  GenRt rt;                // run-time generator parameters (custom engines)
};

// fill tile geometry (kernel K2): each warp emits tiles of 32 substreams x
// segs x 128 bytes, one TMA store each, one CTA of 7 warps per SM.  The tile
// configuration (segs, buffers, pre-wait chunks, sub-block unroll) is chosen
// per (generator, kind) from a measured table (FillCfg / fill_cfg in
// slp_fill.cuh, slp_fill_tuning.h, profiles/tune_fill.py); -DSLP_FILL_CFG=i
// forces one configuration for every kernel (A/B builds).
#ifndef SLP_FILL_WARPS
#define SLP_FILL_WARPS 7
#endif
constexpr int kFillWarps = SLP_FILL_WARPS;
// default store-pacing target of the TMA fill modes in GB/s of output + 1.5 x
// state traffic (0 = unpaced; pace_period_ns in slp_fill.cuh)
#ifndef SLP_DEFAULT_PACE_GBPS
#define SLP_DEFAULT_PACE_GBPS 6600
#endif
constexpr int kDefaultPaceGbps = SLP_DEFAULT_PACE_GBPS;

// up to 16 batches (long-jump blocks) x 16 words, passed by value
constexpr int kMaxBaseBatches = 16;
struct BaseStates {
  uint64_t w[kMaxBaseBatches * 16];
};

// HWD counting consumer (kernel K6)
struct HwdParams {
  const void *sin;           // SoA start states, one per thread
  uint64_t ld;
  uint64_t nthreads;
  uint64_t tseg;             // counted test values per thread (last thread: the rest)
  uint64_t total;            // counted test values in this launch
  uint64_t warm, warm0;      // warm-up test values (thread 0 may differ)
  int lo, hi;                // trit thresholds: nu < lo -> 0, nu <= hi -> 1, else 2
  uint32_t pow3k1;           // 3^(k-1)
  uint32_t ncells;           // 3^k
  int global_cells;          // 1: count straight into global memory (3^k too large even when sliced)
  uint32_t slice_cells;      // shared-memory cells per CTA; CTA (x, y) counts signatures in
                             // [y * slice_cells, (y + 1) * slice_cells) (gridDim.y slices)
  unsigned long long *g_counts, *g_sums;  // 3^k each, accumulated
  unsigned long long *overflow_ctas;      // nullable: CTAs that fell back to the exact recount
  GenRt rt;                // run-time generator parameters (custom engines)
};

struct GenOps {
  int (*fill)(const FillParams &, int out_kind, int layout, cudaStream_t);
  int (*fill_csum)(const FillParams &, int out_kind, cudaStream_t, int *grid_out);
  int (*fused)(const FusedParams &, int flags, cudaStream_t, int *grid_out);
  int (*fused_grid_cap)(int dev);
  int (*jump)(const JumpParams &, const BaseStates *, bool uniform, uint64_t nbatch, cudaStream_t);
  int (*hwd)(const HwdParams &, int transitional, int split, cudaStream_t);
  // K1t: uint32 words per jump table; expand the n rows of a jump matrix
  // (SoA [k][n] states: row i = unit vector i jumped) into one table
  uint64_t (*table_words)();
  int (*build_table)(const void *rows, uint32_t *table, cudaStream_t);
  int (*jump_table)(const TableJumpParams &, uint64_t nbatch, cudaStream_t);
};

const GenOps *gen_ops(int id);

// helpers implemented in slp_api.cu
int current_device();
int sm_count(int dev);
int fill_grid_mult();
int fill_pace_gbps();  // store pacing target in GB/s (0 = off), slp_set_fill_pace
int fill_pace_burst();  // SLP_FILL_PACE_BURST
int cuda_fail(const char *what);
int check_launch(const char *what);
bool tma_ok(const void *out, int es, uint64_t T, uint64_t nstreams, uint64_t ld_out, int segs);
int make_store_tmap(CUtensorMap *map, void *out, int es, uint64_t T, uint64_t nstreams, uint64_t ld_out, int segs,
                    int jsh = 0);
bool tma_ok_pm(const void *out, int es, uint64_t T, uint64_t nstreams, uint64_t ld_out, int ch);
int make_store_tmap_pm(CUtensorMap *map, void *out, int es, uint64_t T, uint64_t nstreams, uint64_t ld_out, int ch,
                       int box_rows = 32);

// Stream-major rows that do not start on a 16-byte boundary (odd T for
// 8-byte outputs, T % 4 != 0 for 4-byte outputs, or an unaligned output
// base).  A TMA box must start 16-byte aligned (profiles/tma_align_probe.cu),
// and pieces that start inside a 32-byte sector leave partial sectors at
// every tile boundary, so row r first emits lead[r % g] outputs with element
// stores; its tiles then start on an a-byte boundary (a = 32 for 8-byte
// outputs, 16 for 4-byte outputs).  Rows are taken in groups of
// g = a / gcd(pitch, a): map p is a 3-D view (128-byte piece, row / g,
// piece index) of the rows of parity p, based at row p's first aligned
// output, with pitch g * pitch (a multiple of a), ceil((n - p) / g)
// rows and (T - lead[p]) / (128 / es) whole pieces, so rows past the end and
// partial pieces are clipped.
struct alignas(64) TmapGroup {
  CUtensorMap m[8];
  int lead[8];  // outputs before the first tile, per parity
  int g, gsh, lead_max;
};
bool tma_group_ok(const void *out, int es, uint64_t T, uint64_t nstreams, uint64_t ld_out, int segs);
int make_store_tmap_group(TmapGroup *tg, void *out, int es, uint64_t T, uint64_t nstreams, uint64_t ld_out, int segs);

}  // namespace slp
