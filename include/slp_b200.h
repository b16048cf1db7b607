/*
 * slp_b200.h -- C ABI of the B200-native bulk generator for the scrambled
 * linear generators of Blackman & Vigna (arXiv 1805.01407).
 *
 * The reference (`slprng`, pure Python) has no FFI; every entry point below
 * replaces one reference function on the bulk `next()` path, cited as
 * file:line relative to /root/reference/pkg/src/slprng/.  Plain pointers and
 * sizes only: no torch types cross this boundary.  Device pointers are
 * caller-owned (e.g. torch CUDA tensors); `stream` is a cudaStream_t passed
 * as void* (NULL = legacy default stream).
 *
 * Every function returns SLP_OK (0) or a negative slp_status.  The Python
 * layer maps SLP_ERR_INVALID / SLP_ERR_ZERO_STATE / SLP_ERR_ENGINE_MISMATCH to
 * ValueError, SLP_ERR_UNKNOWN_GENERATOR to KeyError and SLP_ERR_ALGEBRA to
 * Gf2Error, matching generators.py:120-124,194-215,315-323 and gf2.py:48-53.
 *
 * State layout on the device ("SoA"): word j of substream i lives at
 * states[j * ld + i], j < k, in the FLAT word order of engines.py:14-18,
 * as uint64 for w = 64 generators and uint32 for w = 32 generators.
 */
#ifndef SLP_B200_H
#define SLP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum slp_status {
  SLP_OK = 0,
  SLP_ERR_INVALID = -1,           /* ValueError: bad argument / parameter      */
  SLP_ERR_UNKNOWN_GENERATOR = -2, /* KeyError: unknown name or id              */
  SLP_ERR_UNSUPPORTED = -3,       /* combination the device path does not do   */
  SLP_ERR_ZERO_STATE = -4,        /* ValueError: all-zero state / zero jump    */
  SLP_ERR_CUDA = -5,              /* CUDA runtime error (see slp_last_error)   */
  SLP_ERR_ALGEBRA = -6,           /* Gf2Error: internal self-check failed      */
  SLP_ERR_BUFFER = -7             /* output buffer too small                   */
} slp_status;

/* Output element kinds for slp_fill. */
typedef enum slp_out_kind {
  SLP_OUT_NATIVE = 0, /* w-bit words: uint64 (w=64) or uint32 (w=32)             */
  SLP_OUT_U64 = 1,    /* uint64, 32-bit outputs zero-extended (generators.py:474) */
  SLP_OUT_F64 = 2,    /* double (x >> 11) * 2^-53, w = 64 (generators.py:307-311) */
  SLP_OUT_F32 = 3     /* float (x >> 8) * 2^-24, w = 32 (north_star; no ref fn)    */
} slp_out_kind;

/* Output layouts for slp_fill. */
typedef enum slp_layout {
  SLP_STREAM_MAJOR = 0,  /* out[i * ld_out + t]: substream i, position t         */
  SLP_POSITION_MAJOR = 1 /* out[t * ld_out + i]: the (T, L) buffer of generators.py:474 */
} slp_layout;

/* Consumer flags for slp_fused. */
typedef enum slp_fuse_flags {
  SLP_FUSE_INT = 1,   /* wrapping sum mod 2^64 and xor of all outputs                    */
  SLP_FUSE_F64 = 2,   /* + a float64 accumulation of the converted values (implies EXACT) */
  SLP_FUSE_EXACT = 4  /* + exact 128-bit sum and low-bit sum: exact float sum (mant)      */
} slp_fuse_flags;

typedef struct slp_gen_info {
  int32_t id, family, k, w, a, b, c; /* family: 0 xoroshiro, 1 xoshiro, 2 xorshift */
  int32_t scrambler, word_i, word_j, R;   /* scrambler: 0 none 1 + 2 * 3 ++ 4 ** */
  uint64_t S, T;
  char name[32];
} slp_gen_info;

/* Result of the fused consumer.  All integer fields are exact and independent
 * of summation order.  With SLP_FUSE_EXACT (or F64), sum_hi:sum_lo is the
 * exact sum and mant = (sum - low_sum) >> shift is the exact integer sum of
 * (x >> shift), shift = 11 (w=64) or 8 (w=32), so the float64 sum of the
 * converted values is mant * 2^-(53|24) rounded once.  Without it only sum_lo
 * (the wrapping checksum) and xor_all are defined. */
typedef struct slp_checksum {
  uint64_t sum_lo;  /* sum of outputs mod 2^64 (the wrapping checksum)          */
  uint64_t sum_hi;  /* bits 64..127 of the exact sum of outputs                  */
  uint64_t xor_all; /* xor of all outputs                                        */
  uint64_t low_sum; /* exact sum of (x & (2^shift - 1))                           */
  uint64_t count;   /* number of outputs consumed                                */
  double fsum;      /* float64 accumulation of converted values (SLP_FUSE_F64)   */
} slp_checksum;

/* ---- registry: generators.py:71-124 ------------------------------------ */
int slp_num_generators(void);
/* id of a registry name, or SLP_ERR_UNKNOWN_GENERATOR (get_spec, generators.py:120-124) */
int slp_generator_id(const char *name);
int slp_generator_info(int id, slp_gen_info *out);

/* Registers an arbitrary generator (custom_spec, generators.py:127-135) and
 * returns an id >= SLP_CUSTOM_ID0 (1024) usable with every entry point below
 * (or the registry id when the parameters equal a registry generator's).
 * Fields used: family, k, w, a, b, c, scrambler, word_i, word_j, S, R, T,
 * name; validation follows EngineKind / _check_params (engines.py:56-97) and
 * ScramblerSpec.validate (scramblers.py:68-82).  The host algebra accepts
 * every valid engine; the device kernels (run-time parameter instances)
 * cover xoroshiro 2x64, 16x64, 2x32, xoshiro 4x64, 8x64, 4x32, 8x32 and
 * xorshift 2x64, 2x32 -- other shapes return SLP_ERR_UNSUPPORTED from the
 * device entry points.  Registration is idempotent and thread-safe. */
int slp_register_generator(const slp_gen_info *spec);

/* ---- host GF(2) algebra (setup; not per output) ------------------------- */
/* characteristic polynomial of the engine step matrix, bit i = coeff of x^i,
 * little-endian words; replaces engine_char_poly (generators.py:387-394,
 * gf2.py:418-469).  poly_words >= n/64 + 1. */
int slp_char_poly(int id, uint64_t *poly, int poly_words);
/* x^steps mod P, steps a little-endian multiword integer; replaces
 * compute_jump_poly (generators.py:397-402, gf2.py:214-227). */
int slp_jump_poly(int id, const uint64_t *steps, int steps_words, uint64_t *poly, int poly_words);
/* Polynomial `index` of the substream-initialisation plan slp_init_substreams
 * uses for `n` substreams `steps` apart: the plan starts with x^(i*steps) mod P
 * for i < direct (one K1 jump per substream; the doubling of
 * LanedStream.__init__, generators.py:443-456, done with jump polynomials),
 * followed by the polynomials of its radix-8 rounds.  Returns the number of
 * polynomials in the plan, or a negative status; `poly` may be NULL.  Host
 * only -- lets tests check a plan against slp_jump_poly without a GPU. */
int64_t slp_init_plan_poly(int id, const uint64_t *steps, int steps_words, uint64_t n, uint64_t index,
                           uint64_t *poly, int poly_words);
/* scalar jump of one flat state (k words, each < 2^w) on the host; replaces
 * Generator.jump (generators.py:315-334). */
int slp_host_jump(int id, const uint64_t *poly, int poly_words, uint64_t *flat_state);

/* Same for an arbitrary engine (custom_spec, generators.py:127-135):
 * family 0 xoroshiro / 1 xoshiro / 2 xorshift, k*w <= 1024, w <= 64.
 * Validation follows EngineKind / _check_params (engines.py:56-97). */
int slp_engine_char_poly(int family, int k, int w, int a, int b, int c, uint64_t *poly, int poly_words);
int slp_engine_jump_poly(int family, int k, int w, int a, int b, int c, const uint64_t *steps, int steps_words,
                         uint64_t *poly, int poly_words);

/* ---- device: substream initialisation (kernel K1) ----------------------- */
/* For each block b < nblocks and substream i < n:
 *   states[b*n + i] = base_b * M^(i * steps)
 * where base_b = base_flat[b*k .. b*k+k) (host memory, flat words) and
 * `steps` is the little-endian multiword stride (2^(n/2) for jump()).
 * Replaces the LanedStream lane doubling (generators.py:450-459) and
 * Generator.jump + compute_jump_poly for stream i (generators.py:315-334,397-402).
 * ld >= nblocks * n. */
int slp_init_substreams(int id, const uint64_t *base_flat, uint64_t nblocks, const uint64_t *steps,
                        int steps_words, void *states, uint64_t ld, uint64_t n, void *stream);
/* dst[i] = src[i] * p(M) for i < count (one polynomial for every state);
 * replaces LanedStream._vec_jump (generators.py:493-505) and the super-jump
 * between superbatches (:487-490).  src may equal dst. */
int slp_jump_states(int id, const uint64_t *poly, int poly_words, const void *src, uint64_t ld_src,
                    void *dst, uint64_t ld_dst, uint64_t count, void *stream);

/* seg_states[i*J + j] = states[i] * M^(j * seg_steps) for i < n, j < J:
 * splits each of n long substreams into J consecutive segments so that a
 * stream-major fill of the n*J segments (T = seg_steps outputs each) writes
 * exactly the stream-major output of the n substreams with T = J*seg_steps.
 * The B200 form of the reference's laned scheme (generators.py:426-463) for
 * few, long substreams.  ld_seg >= n*J. */
int slp_split_substreams(int id, const void *states, uint64_t ld, uint64_t n, const uint64_t *seg_steps,
                         int seg_words, uint64_t J, void *seg_states, uint64_t ld_seg, void *stream);

/* Segments per substream that slp_fill (stream-major contiguous rows;
 * padded stream-major rows when the output, its 16-byte row pitch and the
 * segment length are TMA-addressable; position-major), slp_fill_checksum
 * (contiguous rows) and slp_fused use internally for n substreams of T
 * outputs: 1 from 2^15 substreams up (one thread per substream fills the
 * GPU); else a power of two J dividing T, doubled up to n*J = 2^14 while
 * segments keep >= max(512, 2 * state bits) outputs, then up to 2^18 while
 * they keep >= max(2048, 8 * state bits).  The split runs in a
 * stream-ordered scratch buffer (cudaMallocAsync); results are identical
 * (checksums are order-free; the float64 sum covers the same set in another
 * order).  SLP_SPLIT=0 in the environment disables it.  Returns J >= 1 or
 * a negative status. */
int64_t slp_split_factor(int id, uint64_t nstreams, uint64_t T);

/* ---- device: bulk generation (kernels K2/K3/K5) ------------------------- */
/* Emits T outputs of each of nstreams substreams (scramble current state,
 * then step: Generator.next, generators.py:244-305) into `out`, converting
 * per out_kind, and writes the advanced states to states_out (may equal
 * states_in; NULL = do not write back).  ld_out = row pitch in elements
 * (>= T for stream-major, >= nstreams for position-major).  Replaces
 * LanedStream.chunks (generators.py:465-490; VecStepper.step engines.py:318-361;
 * ScramblerSpec.apply_vec scramblers.py:97-127; buf.T.flatten :482). */
int slp_fill(int id, const void *states_in, void *states_out, uint64_t ld, uint64_t nstreams,
             uint64_t T, int out_kind, int layout, void *out, uint64_t ld_out, void *stream);

/* One superbatch of the reference's laned single stream (LanedStream,
 * generators.py:426-490): lane j = base * M^(j * lane_len) is set
 * up in `states` (device SoA (k, lanes), ld = lanes), then lane_len outputs
 * of every lane are written stream-major to out[lanes][lane_len] -- i.e. the
 * next lanes*lane_len values of the scalar stream of `base_flat`, in order.
 * `states` is left advanced by lane_len; the next superbatch is
 * slp_jump_states by (lanes - 1) * lane_len, then slp_fill (:487-490).
 * out_kind: NATIVE, U64 (the reference's uint64 chunks for w = 32), F64/F32. */
int slp_laned_fill(int id, const uint64_t *base_flat, uint64_t lanes, uint64_t lane_len, int out_kind,
                   void *out, void *states, void *stream);

/* Store AND reduce in one pass: slp_fill (stream-major, TMA-eligible output)
 * that also writes the exact checksum of the integer outputs (as slp_fused
 * with SLP_FUSE_EXACT) to `result` (device).  BASELINE config 3 "store mode
 * plus fused checksum".  SLP_ERR_UNSUPPORTED when the output is not
 * TMA-addressable (then run slp_fill and slp_fused on the same states). */
int slp_fill_checksum(int id, const void *states_in, void *states_out, uint64_t ld, uint64_t nstreams, uint64_t T,
                      int out_kind, void *out, uint64_t ld_out, void *result, void *workspace,
                      size_t workspace_bytes, void *stream);

/* ---- device: fused consumer (kernel K4) ---------------------------------- */
/* Same outputs as slp_fill, reduced in-kernel instead of stored; writes one
 * slp_checksum to result (DEVICE memory).  workspace: device scratch of
 * slp_fused_workspace_bytes(nstreams) bytes. */
size_t slp_fused_workspace_bytes(int id, uint64_t nstreams);
int slp_fused(int id, const void *states_in, void *states_out, uint64_t ld, uint64_t nstreams,
              uint64_t T, int flags, void *result, void *workspace, size_t workspace_bytes,
              void *stream);

/* ---- device: Hamming-weight-dependency counting (kernel K6) -------------- */
/* Thread i < nthreads starts from states[:, i] (the generator's single
 * stream at test-value position c0 + i*tseg - warm, warm0 for thread 0),
 * rebuilds the signature from `warm` test values and then, for each of the
 * next min(tseg, total - i*tseg) test values, adds 1 to counts[sig] and its
 * Hamming weight to sums[sig] (DEVICE arrays of 3^k uint64, accumulated).
 * Test values are the w-bit outputs, or (split) the two 32-bit halves of
 * each 64-bit output, low half first; transitional mode xors each value with
 * itself shifted left by one bit, carrying the previous value's top bit.
 * Trit: weight < lo -> 0, <= hi -> 1, else 2; signature update
 * s <- floor(s/3) + trit * 3^(k-1).  Replaces HwdCounters._add / flush
 * (hwd.py:206-247) fed by run_generator (hwd.py:598-621), transitional_chunks
 * (:446-470) and split_chunks (:473-476).  The counts are exact: CTAs whose
 * packed 32-bit shared counters fail the conservation check recount with
 * 64-bit atomics; overflow_ctas (device, nullable) counts those CTAs. */
int slp_hwd_count(int id, const void *states, uint64_t ld, uint64_t nthreads, uint64_t tseg, uint64_t total,
                  uint64_t warm, uint64_t warm0, int k, int lo, int hi, int transitional, int split,
                  uint64_t *counts, uint64_t *sums, uint64_t *overflow_ctas, void *stream);

/* ---- misc ---------------------------------------------------------------- */
/* Bytes held by the device-side cache of `device` (init-plan polynomials and
 * K1t jump tables): a bounded LRU of SLP_DEVICE_CACHE_MB (default 1024) MiB
 * per device, built and freed stream-ordered (no host synchronisation). */
size_t slp_device_cache_bytes(int device);
/* Store pacing of the TMA fill paths (no reference counterpart; a tuning
 * knob that never changes results): the fill kernels offer their tile stores
 * at no more than `gbps` GB/s in aggregate, counted as output bytes plus 1.5x
 * the substream-state bytes read and written, because HBM sustains a paced
 * stream of row-piece stores faster than an unpaced one (DESIGN.md §4,
 * profiles/round2_pacing.md).  0 disables pacing, a negative value only
 * queries.  Returns the previous target.  Default: SLP_FILL_PACE_GBPS, else
 * the built-in 6600. */
int slp_set_fill_pace(int gbps);
const char *slp_status_str(int status);
/* last CUDA error string seen by this thread ("" if none) */
const char *slp_last_error(void);
/* library version / build info */
const char *slp_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* SLP_B200_H */
