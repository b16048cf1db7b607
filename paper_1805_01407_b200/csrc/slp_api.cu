// C ABI (device part): dispatch to the per-generator kernel instances,
// substream-initialisation driver (K1), TMA descriptor set-up and the final
// deterministic reduction of the fused consumer (K4).
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <stdexcept>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "slp_device.cuh"
#include "slp_internal.h"

#define SLP_PART_DECL(P) extern const ::slp::GenOps slp_ops_part_##P[SLP_NUM_GENERATORS];
SLP_PART_DECL(0)
SLP_PART_DECL(1)
SLP_PART_DECL(2)
SLP_PART_DECL(3)
SLP_PART_DECL(4)
SLP_PART_DECL(5)
#ifdef SLP_NO_RT_INSTANCES  // A/B variant builds (Makefile): registry kernels only
static const ::slp::GenOps slp_ops_rt_0[SLP_NUM_RT_SHAPES] = {}, slp_ops_rt_1[SLP_NUM_RT_SHAPES] = {},
                           slp_ops_rt_2[SLP_NUM_RT_SHAPES] = {};
#else
#define SLP_RT_PART_DECL(P) extern const ::slp::GenOps slp_ops_rt_##P[SLP_NUM_RT_SHAPES];
SLP_RT_PART_DECL(0)
SLP_RT_PART_DECL(1)
SLP_RT_PART_DECL(2)
#endif

namespace slp {

// kernel dispatch: registry ids -> their compile-time instances; registered
// custom generators -> the run-time parameter instance of their engine shape
const GenOps *gen_ops(int id) {
  static GenOps table[SLP_NUM_GENERATORS];
  static GenOps rt[SLP_NUM_RT_SHAPES];
  static std::once_flag once;
  std::call_once(once, [] {
    const GenOps *parts[] = {slp_ops_part_0, slp_ops_part_1, slp_ops_part_2,
                             slp_ops_part_3, slp_ops_part_4, slp_ops_part_5};
    for (int i = 0; i < SLP_NUM_GENERATORS; ++i)
      for (const GenOps *p : parts)
        if (p[i].fill) table[i] = p[i];
    const GenOps *rparts[] = {slp_ops_rt_0, slp_ops_rt_1, slp_ops_rt_2};
    for (int i = 0; i < SLP_NUM_RT_SHAPES; ++i)
      for (const GenOps *p : rparts)
        if (p[i].fill) rt[i] = p[i];
  });
  if (id >= SLP_CUSTOM_ID0) {
    const GenDesc *g = gen_desc(id);
    if (!g) return nullptr;
    const int sh = rt_shape(g->family, g->k, g->w);
    return sh >= 0 && rt[sh].fill ? &rt[sh] : nullptr;
  }
  if (id < 0 || id >= SLP_NUM_GENERATORS || !table[id].fill) return nullptr;
  return &table[id];
}

// run-time parameters of a generator for the GenR<> instances
GenRt gen_rt(int id) {
  GenRt r{};
  r.one = r.one2 = 1;
  const GenDesc *g = gen_desc(id);
  if (!g) return r;
  r.a = (uint32_t)g->a;
  r.b = (uint32_t)g->b;
  r.c = (uint32_t)g->c;
  r.sc = g->scrambler;
  r.wi = g->word_i;
  r.wj = g->word_j;
  r.R = (uint32_t)g->R;
  r.S = g->S;
  r.T = g->T;
  return r;
}

int current_device() {
  int d = -1;
  if (cudaGetDevice(&d) != cudaSuccess) return -1;
  return d;
}

int sm_count(int dev) {
  static std::atomic<int> cache[64];
  if (dev < 0 || dev >= 64) return 1;
  int c = cache[dev].load(std::memory_order_relaxed);
  if (!c) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    c = v > 0 ? v : 1;
    cache[dev].store(c, std::memory_order_relaxed);
  }
  return c;
}

static int env_int(const char *name, int dflt) {
  const char *v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// tuning knobs (read once): SLP_FILL_GRID_MULT, SLP_STORE_PATH (0 auto, 1 TMA, 2 staged)
int fill_grid_mult() {
  static int v = env_int("SLP_FILL_GRID_MULT", 1);
  return v > 0 ? v : 1;
}

int fill_pace_burst() {
  static int v = env_int("SLP_FILL_PACE_BURST", 4);
  return v > 0 ? v : 1;
}

// store pacing of the TMA fill modes (pace_store in slp_gen.cuh): the target
// aggregate store rate in GB/s, SLP_FILL_PACE_GBPS or slp_set_fill_pace; 0 = off
static std::atomic<int> g_pace_gbps{-1};
int fill_pace_gbps() {
  int v = g_pace_gbps.load(std::memory_order_relaxed);
  if (v < 0) {
    v = env_int("SLP_FILL_PACE_GBPS", kDefaultPaceGbps);
    if (v < 0) v = 0;
    g_pace_gbps.store(v, std::memory_order_relaxed);
  }
  return v;
}

int cuda_fail(const char *what) {
  cudaError_t e = cudaGetLastError();
  set_last_error(std::string(what) + ": " + cudaGetErrorString(e));
  return SLP_ERR_CUDA;
}

int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_last_error(std::string(what) + ": " + cudaGetErrorString(e));
    return SLP_ERR_CUDA;
  }
  return SLP_OK;
}

bool tma_ok(const void *out, int es, uint64_t T, uint64_t nstreams, uint64_t ld_out, int segs) {
  static int path = env_int("SLP_STORE_PATH", 0);
  if (path == 2) return false;
  const uint64_t seg = 128 / es;  // elements per 128-byte segment
  return ((uintptr_t)out % 128) == 0 && (ld_out * es) % 16 == 0 && T >= (uint64_t)segs * seg && T < (1ull << 40) &&
         nstreams < (1ull << 31) && ld_out * es < (1ull << 40) && ld_out >= T;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Stream-major output viewed as a 4-D tensor (element within a 128-byte
// piece, segment j, substream i, piece index): rows are the `nstreams`
// segments v = i * J + j (J = 1 << jsh, T outputs each) of nstreams >> jsh
// substreams with row pitch ld_out, segment j at column j * T -- J = 1 is the
// plain [nstreams][ld_out] layout.  One box {128/es, Jb, 32/Jb, segs},
// Jb = min(J, 32), is the 32 segment rows of a warp x segs contiguous
// pieces; in shared memory its lines come out in warp-row order
// ((seg * 32 + lane) * 128 B), the layout of k_fill's tile.
int make_store_tmap(CUtensorMap *map, void *out, int es, uint64_t T, uint64_t nstreams, uint64_t ld_out,
                    int segs, int jsh) {
  auto fn = encode_fn();
  if (!fn) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return SLP_ERR_CUDA;
  }
  const uint64_t seg = 128 / es;
  const uint64_t J = 1ull << jsh, Jb = J < 32 ? J : 32;
  cuuint64_t gdim[4] = {(cuuint64_t)seg, (cuuint64_t)J, (cuuint64_t)(nstreams >> jsh), (cuuint64_t)(T / seg)};
  cuuint64_t gstride[3] = {(cuuint64_t)((J > 1 ? T : ld_out) * es), (cuuint64_t)(ld_out * es), 128};
  cuuint32_t box[4] = {(cuuint32_t)seg, (cuuint32_t)Jb, (cuuint32_t)(32 / Jb), (cuuint32_t)segs};
  cuuint32_t estride[4] = {1, 1, 1, 1};
  CUresult r = fn(map, es == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, out, gdim,
                  gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    return SLP_ERR_CUDA;
  }
  return SLP_OK;
}

// Position-major output [T][ld_out] as a 2-D tensor (substream, position):
// one box {box_rows, ch} is ch positions x box_rows consecutive substreams,
// no swizzle (the shared tile is [position][substream]).
bool tma_ok_pm(const void *out, int es, uint64_t T, uint64_t nstreams, uint64_t ld_out, int ch) {
  static int path = env_int("SLP_STORE_PATH", 0);
  if (path == 2) return false;
  return ((uintptr_t)out % 16) == 0 && (ld_out * es) % 16 == 0 && T >= (uint64_t)ch && T < (1ull << 31) &&
         nstreams < (1ull << 31) && ld_out >= nstreams && ld_out * es < (1ull << 40) && ch <= 256;
}

int make_store_tmap_pm(CUtensorMap *map, void *out, int es, uint64_t T, uint64_t nstreams, uint64_t ld_out, int ch,
                       int box_rows) {
  auto fn = encode_fn();
  if (!fn) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return SLP_ERR_CUDA;
  }
  cuuint64_t gdim[2] = {(cuuint64_t)nstreams, (cuuint64_t)T};
  cuuint64_t gstride[1] = {(cuuint64_t)(ld_out * es)};
  cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)ch};
  cuuint32_t estride[2] = {1, 1};
  CUresult r = fn(map, es == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, out, gdim, gstride,
                  box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_last_error("cuTensorMapEncodeTiled (position-major) failed: " + std::to_string((int)r));
    return SLP_ERR_CUDA;
  }
  return SLP_OK;
}

// Row alignment of the tile pieces: a 32-byte sector for 8-byte outputs
// (odd T: 4.2-4.9 TB/s against 3.8-4.3 with 16-byte alignment); 16 bytes for
// 4-byte outputs, where sector alignment needs g = 8 rows of 4 per box and
// measured slower (profiles/round1_ragged.jsonl).
// row-group TMA: rows start on a 32-byte sector (8-byte outputs: g <= 4) or
// 16 bytes (4-byte outputs); SLP_ROW_ALIGN64=16 (A/B) aligns 8-byte rows to
// 16 bytes (g <= 2: half the boxes per tile, partial sectors at the edges)
static uint64_t row_align(int es) {
  static const int a64 = env_int("SLP_ROW_ALIGN64", 32) == 16 ? 16 : 32;
  return es == 8 ? (uint64_t)a64 : 16;
}
static uint64_t row_group(uint64_t pitch_bytes, int es) {  // row_align / gcd(pitch, row_align)
  const uint64_t a = row_align(es);
  uint64_t g = 1;
  while (g < a && ((pitch_bytes * g) % a) != 0) g *= 2;
  return g;
}

bool tma_group_ok(const void *out, int es, uint64_t T, uint64_t nstreams, uint64_t ld_out, int segs) {
  static int path = env_int("SLP_STORE_PATH", 0);
  if (path == 2 || path == 3) return false;  // 3: staged instead of row groups (A/B)
  const uint64_t seg = 128 / es;
  const uint64_t g = row_group(ld_out * es, es);
  return ((uintptr_t)out % es) == 0 && T >= (uint64_t)segs * seg + row_align(es) / es && ld_out >= T && nstreams >= g &&
         g <= 4 &&  // k_fill's tile addressing needs 32 / g rows per piece to be a multiple of 8
         T < (1ull << 31) && g * ld_out * es < (1ull << 40) && nstreams < (1ull << 31);
}

int make_store_tmap_group(TmapGroup *tg, void *out, int es, uint64_t T, uint64_t nstreams, uint64_t ld_out,
                          int segs) {
  auto fn = encode_fn();
  if (!fn) {
    set_last_error("cuTensorMapEncodeTiled unavailable");
    return SLP_ERR_CUDA;
  }
  const uint64_t g = row_group(ld_out * es, es);
  const uint64_t seg = 128 / es;
  const uintptr_t addr = (uintptr_t)out;
  tg->g = (int)g;
  tg->gsh = g == 8 ? 3 : (g == 4 ? 2 : (g == 2 ? 1 : 0));
  tg->lead_max = 0;
  for (int r = 0; r < 8; ++r) tg->lead[r] = 0;
  for (uint64_t r = 0; r < g; ++r) {
    const uintptr_t row = addr + r * ld_out * es;
    const int lead = (int)(((row_align(es) - row % row_align(es)) % row_align(es)) / es);
    tg->lead[r] = lead;
    if (lead > tg->lead_max) tg->lead_max = lead;
    cuuint64_t gdim[3] = {(cuuint64_t)seg, (cuuint64_t)((nstreams - r + g - 1) / g), (cuuint64_t)((T - lead) / seg)};
    cuuint64_t gstride[2] = {(cuuint64_t)(g * ld_out * es), 128};
    cuuint32_t box[3] = {(cuuint32_t)seg, (cuuint32_t)(32 / g), (cuuint32_t)segs};
    cuuint32_t estride[3] = {1, 1, 1};
    CUresult rc = fn(&tg->m[r], es == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32, 3,
                     reinterpret_cast<void *>(row + lead * es), gdim, gstride, box, estride,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) {
      set_last_error("cuTensorMapEncodeTiled (row groups) failed: " + std::to_string((int)rc));
      return SLP_ERR_CUDA;
    }
  }
  return SLP_OK;
}

namespace dev {
__global__ void k_fused_final(const slp_checksum *parts, int nparts, slp_checksum *result, uint64_t count,
                              double fscale) {
  __shared__ uint64_t s_lo[256], s_hi[256], s_x[256], s_low[256];
  __shared__ double s_f[256];
  const int t = threadIdx.x;
  uint64_t lo = 0, hi = 0, x = 0, low = 0;
  double f = 0.0;
  for (int i = t; i < nparts; i += 256) {
    const slp_checksum c = parts[i];
    const uint64_t nlo = lo + c.sum_lo;
    hi += c.sum_hi + (nlo < lo ? 1 : 0);
    lo = nlo;
    x ^= c.xor_all;
    low += c.low_sum;
    f += c.fsum;
  }
  s_lo[t] = lo;
  s_hi[t] = hi;
  s_x[t] = x;
  s_low[t] = low;
  s_f[t] = f;
  __syncthreads();
  if (t == 0) {
    for (int i = 1; i < 256; ++i) {
      const uint64_t nlo = lo + s_lo[i];
      hi += s_hi[i] + (nlo < lo ? 1 : 0);
      lo = nlo;
      x ^= s_x[i];
      low += s_low[i];
      f += s_f[i];
    }
    result->sum_lo = lo;
    result->sum_hi = hi;
    result->xor_all = x;
    result->low_sum = low;
    result->count = count;
    result->fsum = f * fscale;
  }
}
// states_out[j][i] = seg[j][i*J + J-1]: substream i ends where its last segment ends
template <class W>
__global__ void k_segment_ends(const W *seg, uint64_t n, uint64_t J, int k, W *out, uint64_t ld, int jmajor) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * (uint64_t)k) return;
  const uint64_t j = t / n, i = t - j * n;
  out[j * ld + i] = seg[j * n * J + (jmajor ? (J - 1) * n + i : i * J + J - 1)];
}
// segment states i * J + j  ->  j * n + i (position-major split: a warp's
// lanes are consecutive substreams of one row block), every word row
template <class W>
__global__ void k_segments_jmajor(const W *in, W *out, uint64_t n, uint64_t J, int k) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t m = n * J;
  if (t >= m * (uint64_t)k) return;
  const uint64_t w = t / m, v = t - w * m;  // v = j * n + i (coalesced writes)
  const uint64_t j = v / n, i = v - j * n;
  out[w * m + v] = in[w * m + i * J + j];
}
}  // namespace dev

// ---- device-side caches ----------------------------------------------------
// Init-plan polynomials and K1t jump tables live in one bounded LRU per
// device (SLP_DEVICE_CACHE_MB, default 1024).  Nothing here synchronises the
// host, so a fill stays asynchronous (and capturable) even when it needs a new
// plan: an entry is built stream-ordered on the caller's stream
// (cudaMallocAsync + copies + kernels) and published with a `ready` event
// that every later user waits on (cudaStreamWaitEvent) before its launches.
// Every use records a per-stream `last use` event; evicting an entry orders
// its cudaFreeAsync after those events, so memory is never freed under a
// kernel that still reads it.  Entries are pinned while a call holds them.
namespace {
struct DevEntry {
  void *ptr = nullptr;
  size_t bytes = 0;
  uint64_t tick = 0;
  int pins = 0;
  cudaEvent_t ready = nullptr;
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> uses;
  uint64_t first_poly = 0, count = 0;  // table sets: polynomials [first, first + count) of the plan
};
enum { CACHE_PLAN_POLYS = 0, CACHE_PLAN_TABLES = 1, CACHE_POLY_TABLE = 2 };
using DevKey = std::tuple<int, int, std::vector<uint64_t>>;  // (kind, device, key words)

std::mutex g_cache_mu;
std::map<DevKey, std::unique_ptr<DevEntry>> g_cache;
std::map<int, size_t> g_cache_bytes;
uint64_t g_cache_tick = 0;

size_t cache_budget() {
  static size_t b = (size_t)std::max(64, env_int("SLP_DEVICE_CACHE_MB", 1024)) << 20;
  return b;
}

// a stream being captured into a CUDA graph: waits on and records of events
// that live outside the graph must be external nodes
bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive;
}

// with g_cache_mu held: the entry, pinned and waited on by `st`, or nullptr
DevEntry *cache_find(const DevKey &key, cudaStream_t st) {
  auto it = g_cache.find(key);
  if (it == g_cache.end()) return nullptr;
  DevEntry *e = it->second.get();
  e->tick = ++g_cache_tick;
  ++e->pins;
  if (e->ready) cudaStreamWaitEvent(st, e->ready, capturing(st) ? cudaEventWaitExternal : 0);
  return e;
}

void release_entry(DevEntry &e, cudaStream_t st) {  // frees after every recorded use (stream-ordered)
  for (auto &u : e.uses) {
    cudaStreamWaitEvent(st, u.second, 0);
    cudaEventDestroy(u.second);
  }
  if (e.ready) {
    cudaStreamWaitEvent(st, e.ready, 0);
    cudaEventDestroy(e.ready);
  }
  if (e.ptr) cudaFreeAsync(e.ptr, st);
}

// with g_cache_mu held: publish a freshly built entry (pinned), evicting
// least-recently-used unpinned entries of the device beyond the budget
DevEntry *cache_insert(const DevKey &key, std::unique_ptr<DevEntry> e, cudaStream_t st) {
  const int dev = std::get<1>(key);
  e->tick = ++g_cache_tick;
  e->pins = 1;
  if (cudaEventCreateWithFlags(&e->ready, cudaEventDisableTiming) == cudaSuccess) cudaEventRecord(e->ready, st);
  g_cache_bytes[dev] += e->bytes;
  DevEntry *raw = e.get();
  g_cache[key] = std::move(e);
  while (g_cache_bytes[dev] > cache_budget()) {
    auto lru = g_cache.end();
    for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
      if (std::get<1>(it->first) == dev && it->second->pins == 0 &&
          (lru == g_cache.end() || it->second->tick < lru->second->tick))
        lru = it;
    if (lru == g_cache.end()) break;  // everything else is in use: stay over budget for now
    g_cache_bytes[dev] -= lru->second->bytes;
    release_entry(*lru->second, st);
    g_cache.erase(lru);
  }
  return raw;
}

// the caller's launches on `st` that read the entry are enqueued: record the
// last use on this stream and unpin
void cache_unpin(DevEntry *e, cudaStream_t st) {
  if (!e) return;
  std::lock_guard<std::mutex> lk(g_cache_mu);
  cudaEvent_t ev = nullptr;
  for (auto &u : e->uses)
    if (u.first == st) ev = u.second;
  if (!ev && cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) e->uses.emplace_back(st, ev);
  if (ev) cudaEventRecordWithFlags(ev, st, capturing(st) ? cudaEventRecordExternal : cudaEventRecordDefault);
  --e->pins;
}

// unpins on scope exit
struct Pinned {
  DevEntry *e = nullptr;
  cudaStream_t st = nullptr;
  Pinned() = default;
  Pinned(const Pinned &) = delete;
  Pinned &operator=(const Pinned &) = delete;
  ~Pinned() { cache_unpin(e, st); }
};
}  // namespace

// device copy of a plan's polynomials (H2D on `st`, stream-ordered)
static int plan_polys_on_device(const InitPlan &plan, int dev, cudaStream_t st, Pinned &pin) {
  const DevKey key{CACHE_PLAN_POLYS, dev, {plan.uid}};
  std::lock_guard<std::mutex> lk(g_cache_mu);
  pin.st = st;
  if ((pin.e = cache_find(key, st))) return SLP_OK;
  auto e = std::make_unique<DevEntry>();
  e->bytes = plan.polys.size() * sizeof(uint64_t);
  if (cudaMallocAsync(&e->ptr, e->bytes, st) != cudaSuccess) return cuda_fail("cudaMallocAsync(init polys)");
  if (cudaMemcpyAsync(e->ptr, plan.polys.data(), e->bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) {
    cudaFreeAsync(e->ptr, st);
    return cuda_fail("cudaMemcpyAsync(init polys)");
  }
  pin.e = cache_insert(key, std::move(e), st);
  return SLP_OK;
}

// builds `count` K1t tables on `st` (stream-ordered, no host synchronisation):
// table i from polynomial i of the device array `d_polys` (or, when d_polys
// is null, from the single host polynomial `host_poly` passed as a kernel
// parameter).  Row r of a jump matrix is unit vector r jumped by K1 (one
// launch over the n unit vectors), then expanded into four-Russians tables.
static int build_jump_tables(int id, const uint64_t *d_polys, uint64_t first_poly, const uint64_t *host_poly,
                             uint64_t count, cudaStream_t st, uint32_t **out) {
  const GenDesc &g = *gen_desc(id);
  const GenOps *ops = gen_ops(id);
  const int nb = g.n();
  const size_t esz = g.w / 8;
  std::vector<uint8_t> ident((size_t)g.k * nb * esz, 0);
  for (int i = 0; i < nb; ++i) {
    const size_t off = ((size_t)(i / g.w) * nb + i) * esz;  // SoA [k][nb]: word i / w of state i
    const uint64_t bit = 1ull << (i % g.w);
    std::memcpy(&ident[off], &bit, esz);
  }
  const uint64_t tw = ops->table_words();
  void *d_ident = nullptr, *d_rows = nullptr;
  uint32_t *tables = nullptr;
  if (cudaMallocAsync(&d_ident, ident.size(), st) != cudaSuccess) return cuda_fail("cudaMallocAsync(jump tables)");
  if (cudaMallocAsync(&d_rows, ident.size(), st) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void **>(&tables), count * tw * sizeof(uint32_t), st) != cudaSuccess) {
    cudaFreeAsync(d_ident, st);
    if (d_rows) cudaFreeAsync(d_rows, st);
    return cuda_fail("cudaMallocAsync(jump tables)");
  }
  // pageable source: staged by the driver before the call returns
  int rc = cudaMemcpyAsync(d_ident, ident.data(), ident.size(), cudaMemcpyHostToDevice, st) == cudaSuccess
               ? SLP_OK
               : cuda_fail("cudaMemcpyAsync(identity)");
  BaseStates base;
  std::memset(&base, 0, sizeof base);
  if (host_poly)
    for (int i = 0; i < g.n() / 64; ++i) base.w[i] = host_poly[i];
  for (uint64_t i = 0; i < count && rc == SLP_OK; ++i) {
    JumpParams p{};
    p.rt = gen_rt(id);
    p.src = d_ident;
    p.ld_src = nb;
    p.dst = d_rows;
    p.ld_dst = nb;
    p.polys = d_polys;  // null: the polynomial is in the BaseStates parameter block
    p.poly0 = first_poly + i;
    p.pmode = 0;
    p.count = nb;
    rc = ops->jump(p, host_poly ? &base : nullptr, true, 1, st);
    if (rc == SLP_OK) rc = ops->build_table(d_rows, tables + i * tw, st);
  }
  cudaFreeAsync(d_ident, st);  // after the kernels above (stream order)
  cudaFreeAsync(d_rows, st);
  if (rc != SLP_OK) {
    cudaFreeAsync(tables, st);
    return rc;
  }
  *out = tables;
  return SLP_OK;
}

// K1t tables of an init plan's round polynomials
static int plan_tables_on_device(const InitPlan &plan, int id, int dev, const uint64_t *d_polys, cudaStream_t st,
                                 Pinned &pin) {
  const DevKey key{CACHE_PLAN_TABLES, dev, {plan.uid}};
  std::lock_guard<std::mutex> lk(g_cache_mu);
  pin.st = st;
  if ((pin.e = cache_find(key, st))) return SLP_OK;
  auto e = std::make_unique<DevEntry>();
  e->first_poly = plan.launches.size() > 1 ? plan.launches[1].poly0 : plan.polys.size() / plan.pw;
  e->count = plan.polys.size() / plan.pw - e->first_poly;
  if (e->count > 0) {
    uint32_t *t = nullptr;
    const int rc = build_jump_tables(id, d_polys, e->first_poly, nullptr, e->count, st, &t);
    if (rc != SLP_OK) return rc;
    e->ptr = t;
    e->bytes = e->count * gen_ops(id)->table_words() * sizeof(uint32_t);
  }
  pin.e = cache_insert(key, std::move(e), st);
  return SLP_OK;
}

// K1t table of a single jump polynomial (slp_jump_states), per (engine, device, polynomial)
static int poly_table_on_device(int id, int dev, const uint64_t *poly, cudaStream_t st, Pinned &pin) {
  const GenDesc &g = *gen_desc(id);
  std::vector<uint64_t> kw(poly, poly + g.n() / 64);
  kw.push_back((uint64_t)engine_id(id));
  const DevKey key{CACHE_POLY_TABLE, dev, kw};
  std::lock_guard<std::mutex> lk(g_cache_mu);
  pin.st = st;
  if ((pin.e = cache_find(key, st))) return SLP_OK;
  uint32_t *t = nullptr;
  const int rc = build_jump_tables(id, nullptr, 0, poly, 1, st, &t);
  if (rc != SLP_OK) return rc;
  auto e = std::make_unique<DevEntry>();
  e->ptr = t;
  e->bytes = gen_ops(id)->table_words() * sizeof(uint32_t);
  e->count = 1;
  pin.e = cache_insert(key, std::move(e), st);
  return SLP_OK;
}

// K1t replaces the uniform radix rounds of at least this many states
// (SLP_INIT_TABLES=0 disables it)
// slp_jump_states: K1t from this many states on (a table costs ~n unit-vector
// jumps to build, then is cached per polynomial)
constexpr uint64_t kJumpTableMinStates = 65536;

static bool use_jump_tables(uint64_t count) {
  // SLP_INIT_TABLES=0 disables K1t; =N sets the threshold (A/B).  Read on every
  // call (a getenv per launch is noise) so that tests can switch it in-process.
  const char *v = std::getenv("SLP_INIT_TABLES");
  const long min_states = (v && *v == '0') ? -1L : (v && *v ? std::atol(v) : 16384L);
  return min_states >= 0 && count >= (uint64_t)min_states;
}

}  // namespace slp

using namespace slp;

static bool state_ok(const GenDesc &g, const uint64_t *words) {
  const uint64_t mask = g.w == 64 ? ~0ull : ((1ull << g.w) - 1);
  bool any = false;
  for (int j = 0; j < g.k; ++j) {
    if (words[j] & ~mask) return false;
    any |= words[j] != 0;
  }
  return any;
}

extern "C" {

// Radix rounds 1.. of an init plan over nblocks batches of n states
// (batch b at states + b * n): stream m*c + s of a batch is stream s jumped
// by x^(c*m*stride), K1t for the table-sized rounds, else K1.
static int plan_rounds(const InitPlan &plan, int id, const GenOps *ops, int dev, const uint64_t *d_polys,
                       void *states, uint64_t ld, uint64_t n, uint64_t nblocks, cudaStream_t st) {
  int rc = SLP_OK;
  Pinned tpin;  // the plan's K1t table set, pinned until the launches below are enqueued
  const DevEntry *tabs = nullptr;
  for (size_t li = 1; li < plan.launches.size(); ++li) {
    InitLaunch L = plan.launches[li];
    if (L.dst0 >= n) break;
    if (L.count > n - L.dst0) L.count = n - L.dst0;
    if (L.uniform && use_jump_tables(L.count * nblocks)) {
      if (!tabs) {
        rc = plan_tables_on_device(plan, id, dev, d_polys, st, tpin);
        if (rc != SLP_OK) return rc;
        tabs = tpin.e;
      }
    }
    if (L.uniform && tabs && tabs->ptr && use_jump_tables(L.count * nblocks)) {
      TableJumpParams tp{};
      tp.rt = gen_rt(id);
      tp.src = states;
      tp.ld_src = ld;
      tp.dst = states;
      tp.ld_dst = ld;
      tp.tables = static_cast<const uint32_t *>(tabs->ptr);
      tp.table0 = L.poly0 - tabs->first_poly;
      tp.count = L.count;
      tp.m = L.m;
      tp.src_off = 0;
      tp.dst_off = L.dst0;
      tp.batch_stride = n;
      rc = ops->jump_table(tp, nblocks, st);
      if (rc != SLP_OK) return rc;
      continue;
    }
    JumpParams p{};
    p.rt = gen_rt(id);
    p.src = states;
    p.ld_src = ld;
    p.dst = states;
    p.ld_dst = ld;
    p.polys = d_polys;
    p.poly0 = L.poly0;
    p.pmode = 1;
    p.use_base = 0;
    p.count = L.count;
    p.m = L.m;
    p.src_off = 0;
    p.dst_off = L.dst0;
    p.batch_stride = n;
    rc = ops->jump(p, nullptr, L.uniform, nblocks, st);
    if (rc != SLP_OK) return rc;
  }
  return SLP_OK;
}

int slp_init_substreams(int id, const uint64_t *base_flat, uint64_t nblocks, const uint64_t *steps, int steps_words,
                        void *states, uint64_t ld, uint64_t n, void *stream) {
  const GenDesc *g = gen_desc(id);
  if (!g) return SLP_ERR_UNKNOWN_GENERATOR;
  const GenOps *ops = gen_ops(id);
  if (!ops) return SLP_ERR_UNSUPPORTED;
  if (!base_flat || !states || nblocks == 0 || n == 0 || ld < nblocks * n || steps_words < 0 ||
      (steps_words > 0 && !steps) || nblocks > 65535)
    return SLP_ERR_INVALID;
  for (uint64_t b = 0; b < nblocks; ++b)
    if (!state_ok(*g, base_flat + b * g->k)) return SLP_ERR_ZERO_STATE;
  std::shared_ptr<const InitPlan> plan;
  try {
    plan = init_plan(id, steps, steps_words, n);
  } catch (const AlgebraError &e) {
    set_last_error(e.what());
    return SLP_ERR_ALGEBRA;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return SLP_ERR_INVALID;
  }
  const int dev = current_device();
  if (dev < 0) return cuda_fail("cudaGetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Pinned ppin;  // the plan's device polynomials, pinned until every launch is enqueued
  int rc = plan_polys_on_device(*plan, dev, st, ppin);
  if (rc != SLP_OK) return rc;
  const uint64_t *d_polys = static_cast<const uint64_t *>(ppin.e->ptr);
  const size_t esize = g->w / 8;
  // launch 0: every block base -> first m0 substreams (one polynomial per substream)
  const InitLaunch &l0 = plan->launches[0];
  for (uint64_t b0 = 0; b0 < nblocks; b0 += kMaxBaseBatches) {
    const uint64_t nb = nblocks - b0 < (uint64_t)kMaxBaseBatches ? nblocks - b0 : (uint64_t)kMaxBaseBatches;
    BaseStates base;
    std::memset(&base, 0, sizeof base);
    for (uint64_t b = 0; b < nb; ++b)
      for (int j = 0; j < g->k; ++j) base.w[b * g->k + j] = base_flat[(b0 + b) * g->k + j];
    JumpParams p{};
    p.rt = gen_rt(id);
    p.src = nullptr;
    p.dst = static_cast<uint8_t *>(states) + b0 * n * esize;
    p.ld_dst = ld;
    p.polys = d_polys;
    p.poly0 = l0.poly0;
    p.pmode = 2;
    p.use_base = 1;
    p.count = l0.count < n ? l0.count : n;  // plans serve every n up to theirs (init_plan)
    p.m = 0;
    p.dst_off = 0;
    p.batch_stride = n;
    rc = ops->jump(p, &base, false, nb, st);
    if (rc != SLP_OK) return rc;
  }
  return plan_rounds(*plan, id, ops, dev, d_polys, states, ld, n, nblocks, st);
}

int slp_split_substreams(int id, const void *states, uint64_t ld, uint64_t n, const uint64_t *seg_steps,
                         int seg_words, uint64_t J, void *seg_states, uint64_t ld_seg, void *stream) {
  const GenDesc *g = gen_desc(id);
  if (!g) return SLP_ERR_UNKNOWN_GENERATOR;
  const GenOps *ops = gen_ops(id);
  if (!ops) return SLP_ERR_UNSUPPORTED;
  if (n == 0 || J == 0) return SLP_OK;
  if (!states || !seg_states || ld < n || ld_seg < n * J || seg_words < 0 || (seg_words > 0 && !seg_steps) ||
      J > (1ull << 20))
    return SLP_ERR_INVALID;
  std::shared_ptr<const InitPlan> plan;
  try {
    plan = init_plan(id, seg_steps, seg_words, J);  // segment j = substream jumped by x^(j*seg)
  } catch (const AlgebraError &e) {
    set_last_error(e.what());
    return SLP_ERR_ALGEBRA;
  } catch (const std::exception &e) {
    set_last_error(e.what());
    return SLP_ERR_INVALID;
  }
  const int dev = current_device();
  if (dev < 0) return cuda_fail("cudaGetDevice");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Pinned ppin;  // the plan's device polynomials, pinned until every launch is enqueued
  int rc = plan_polys_on_device(*plan, dev, st, ppin);
  if (rc != SLP_OK) return rc;
  const uint64_t *d_polys = static_cast<const uint64_t *>(ppin.e->ptr);
  const size_t esize = g->w / 8;
  // the init plan with the n substreams as its batches: launch 0 jumps each
  // substream directly into its first segments, the radix rounds grow the rest
  const InitLaunch &l0 = plan->launches[0];
  for (uint64_t b0 = 0; b0 < n; b0 += 65535) {
    const uint64_t nb = n - b0 < 65535 ? n - b0 : 65535;
    void *seg = static_cast<uint8_t *>(seg_states) + b0 * J * esize;
    JumpParams p{};
    p.rt = gen_rt(id);
    p.src = static_cast<const uint8_t *>(states) + b0 * esize;
    p.ld_src = ld;
    p.dst = seg;
    p.ld_dst = ld_seg;
    p.polys = d_polys;
    p.poly0 = l0.poly0;
    p.pmode = 2;
    p.use_base = 0;
    p.count = l0.count < J ? l0.count : J;
    p.m = 1;  // source = the batch's own substream
    p.batch_stride = J;
    p.src_batch_stride = 1;
    uint64_t grid_batches = nb;
    if (p.count < 128) {  // fewer states than a CTA per substream: fold the substreams into x
      p.fold = p.count;
      p.count *= nb;
      grid_batches = 1;
    }
    rc = ops->jump(p, nullptr, false, grid_batches, st);
    if (rc != SLP_OK) return rc;
    rc = plan_rounds(*plan, id, ops, dev, d_polys, seg, ld_seg, J, nb, st);
    if (rc != SLP_OK) return rc;
  }
  return SLP_OK;
}

int slp_jump_states(int id, const uint64_t *poly, int poly_words, const void *src, uint64_t ld_src, void *dst,
                    uint64_t ld_dst, uint64_t count, void *stream) {
  const GenDesc *g = gen_desc(id);
  if (!g) return SLP_ERR_UNKNOWN_GENERATOR;
  const GenOps *ops = gen_ops(id);
  if (!ops) return SLP_ERR_UNSUPPORTED;
  if (!poly || poly_words <= 0 || !src || !dst || ld_src < count || ld_dst < count) return SLP_ERR_INVALID;
  const int pw = g->n() / 64;
  bool nonzero = false;
  for (int i = 0; i < poly_words; ++i) {
    if (i >= pw && poly[i]) return SLP_ERR_INVALID;  // degree must be < n (reduced mod P)
    nonzero |= poly[i] != 0;
  }
  if (!nonzero) return SLP_ERR_ZERO_STATE;
  BaseStates base;
  std::memset(&base, 0, sizeof base);
  int used = 0;
  for (int i = 0; i < pw && i < poly_words; ++i) {
    base.w[i] = poly[i];
    if (poly[i]) used = i + 1;
  }
  JumpParams p{};
  p.rt = gen_rt(id);
  p.src = src;
  p.ld_src = ld_src;
  p.dst = dst;
  p.ld_dst = ld_dst;
  p.polys = nullptr;  // polynomial in the BaseStates parameter block
  p.poly0 = 0;
  p.pmode = 0;
  p.use_base = 0;
  p.count = count;
  p.m = 0;
  p.batch_stride = 0;
  p.pw_used = used;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // many states: K1t with a cached table of this polynomial.  In place only
  // for n <= 256 (one table slice: a thread reads its whole state before
  // writing it); wider engines split the output words over CTAs, which would
  // race with the reads of the other slices.
  if (count >= kJumpTableMinStates && (src != dst || g->n() <= 256) && use_jump_tables(count)) {
    const int dev = current_device();
    if (dev < 0) return cuda_fail("cudaGetDevice");
    Pinned tpin;
    const int rc = poly_table_on_device(id, dev, base.w, st, tpin);
    if (rc != SLP_OK) return rc;
    const uint32_t *table = static_cast<const uint32_t *>(tpin.e->ptr);
    {
      TableJumpParams tp{};
      tp.rt = gen_rt(id);
      tp.src = src;
      tp.ld_src = ld_src;
      tp.dst = dst;
      tp.ld_dst = ld_dst;
      tp.tables = table;
      tp.table0 = 0;
      tp.count = count;
      tp.m = count;
      return ops->jump_table(tp, 1, st);
    }
  }
  return ops->jump(p, &base, true, 1, st);
}

int slp_laned_fill(int id, const uint64_t *base_flat, uint64_t lanes, uint64_t lane_len, int out_kind, void *out,
                   void *states, void *stream) {
  if (!gen_desc(id)) return SLP_ERR_UNKNOWN_GENERATOR;
  if (lanes == 0 || lane_len == 0) return SLP_OK;
  if (!base_flat || !out || !states) return SLP_ERR_INVALID;
  const uint64_t steps[1] = {lane_len};
  int rc = slp_init_substreams(id, base_flat, 1, steps, 1, states, lanes, lanes, stream);
  if (rc != SLP_OK) return rc;
  return slp_fill(id, states, states, lanes, lanes, lane_len, out_kind, SLP_STREAM_MAJOR, out, lane_len, stream);
}

// ---- few, long substreams: segment split --------------------------------------
// One thread per substream fills the GPU only from about one wave of
// substreams (148 SMs x 7 warps x 32 = 33152; profiles/round1_shape_scan.jsonl).
// Below 2^15 substreams each is split into J segments i*J + j starting j*T/J
// steps ahead (slp_split_substreams) in a stream-ordered scratch buffer: the
// segment rows are byte-for-byte the substream rows, the checksums are
// order-free, and substream i ends where segment i*J + J-1 ends.
// J doubles first up to half a wave of segments (2^14) while they keep
// >= max(512, 2 * state bits) outputs, then up to 2^18 segments while they
// keep >= max(2048, 8 * state bits) (long rows: more parallelism, jumps
// amortised).  A full first-phase wave measured slower: its extra jumps
// cost more than the fill gains (profiles/round1_shape_scan.jsonl).
static uint64_t split_factor(const GenDesc &g, uint64_t n, uint64_t T, uint64_t nmax = 1ull << 15) {
  if (env_int("SLP_SPLIT", 1) == 0 || n == 0 || n >= nmax) return 1;
  const uint64_t bits = (uint64_t)g.n();
  const uint64_t min_wave = std::max<uint64_t>(512, 2 * bits), min_long = std::max<uint64_t>(2048, 8 * bits);
  uint64_t J = 1;
  while (n * J < (1ull << 14) && T % (2 * J) == 0 && T / (2 * J) >= min_wave) J *= 2;
  while (n * J < (1ull << 18) && T % (2 * J) == 0 && T / (2 * J) >= min_long) J *= 2;
  return J;
}

int64_t slp_split_factor(int id, uint64_t nstreams, uint64_t T) {
  const GenDesc *g = gen_desc(id);
  if (!g) return SLP_ERR_UNKNOWN_GENERATOR;
  return (int64_t)split_factor(*g, nstreams, T);
}

namespace {
struct Segments {
  void *states = nullptr;
  cudaStream_t st = nullptr;
  Segments() = default;
  Segments(const Segments &) = delete;
  Segments &operator=(const Segments &) = delete;
  ~Segments() {
    if (states) cudaFreeAsync(states, st);  // stream-ordered: after the kernels that use it
  }
};
}  // namespace

static int make_segments(int id, const GenDesc &g, const void *states, uint64_t ld, uint64_t n, uint64_t T,
                         uint64_t J, cudaStream_t st, Segments &seg, bool jmajor = false) {
  seg.st = st;
  const int dev = current_device();
  static std::atomic<int> pool_set[64];
  if (dev >= 0 && dev < 64 && !pool_set[dev]) {
    // keep freed scratch in the device's default pool instead of unmapping it
    // at every synchronisation (the default threshold, 0, costs ~1 ms a call)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = 1ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool_set[dev] = 1;
  }
  const size_t bytes = (size_t)g.k * n * J * (g.w / 8);
  if (cudaMallocAsync(&seg.states, bytes, st) != cudaSuccess) {
    seg.states = nullptr;
    return cuda_fail("cudaMallocAsync(segments)");
  }
  const uint64_t steps[1] = {T / J};
  int rc = slp_split_substreams(id, states, ld, n, steps, 1, J, seg.states, n * J, st);
  if (rc != SLP_OK || !jmajor) return rc;
  void *tmp = nullptr;
  if (cudaMallocAsync(&tmp, bytes, st) != cudaSuccess) return cuda_fail("cudaMallocAsync(segments)");
  const uint64_t total = n * J * (uint64_t)g.k;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (g.w == 64)
    slp::dev::k_segments_jmajor<uint64_t><<<blocks, 256, 0, st>>>(static_cast<const uint64_t *>(seg.states),
                                                                  static_cast<uint64_t *>(tmp), n, J, g.k);
  else
    slp::dev::k_segments_jmajor<uint32_t><<<blocks, 256, 0, st>>>(static_cast<const uint32_t *>(seg.states),
                                                                  static_cast<uint32_t *>(tmp), n, J, g.k);
  rc = check_launch("k_segments_jmajor");
  cudaFreeAsync(seg.states, st);
  seg.states = tmp;
  return rc;
}

static int segment_ends(const GenDesc &g, const Segments &seg, uint64_t n, uint64_t J, void *states_out, uint64_t ld,
                        cudaStream_t st, int jmajor = 0) {
  const uint64_t total = n * (uint64_t)g.k;
  const unsigned blocks = (unsigned)((total + 255) / 256);
  if (g.w == 64)
    slp::dev::k_segment_ends<uint64_t><<<blocks, 256, 0, st>>>(static_cast<const uint64_t *>(seg.states), n, J, g.k,
                                                          static_cast<uint64_t *>(states_out), ld, jmajor);
  else
    slp::dev::k_segment_ends<uint32_t><<<blocks, 256, 0, st>>>(static_cast<const uint32_t *>(seg.states), n, J, g.k,
                                                          static_cast<uint32_t *>(states_out), ld, jmajor);
  return check_launch("k_segment_ends");
}

int slp_fill(int id, const void *states_in, void *states_out, uint64_t ld, uint64_t nstreams, uint64_t T,
             int out_kind, int layout, void *out, uint64_t ld_out, void *stream) {
  const GenDesc *g = gen_desc(id);
  if (!g) return SLP_ERR_UNKNOWN_GENERATOR;
  const GenOps *ops = gen_ops(id);
  if (!ops) return SLP_ERR_UNSUPPORTED;
  if (nstreams == 0) return SLP_OK;  // nothing to generate (pointers of empty tensors may be null)
  if (!states_in || ld < nstreams || (!out && T && nstreams)) return SLP_ERR_INVALID;
  if (layout == SLP_STREAM_MAJOR && ld_out < T) return SLP_ERR_INVALID;
  if (layout == SLP_POSITION_MAJOR && ld_out < nstreams) return SLP_ERR_INVALID;
  if (nstreams >= (1ull << 40)) return SLP_ERR_INVALID;
  FillParams p{};
  p.rt = gen_rt(id);
  p.sin = states_in;
  p.sout = states_out;
  p.ld = ld;
  p.nstreams = nstreams;
  p.T = T;
  p.out = out;
  p.ld_out = ld_out;
  if (nstreams == 0) return SLP_OK;
  if (T == 0) {
    if (states_out && states_out != states_in) {
      const size_t es = g->w / 8;
      for (int j = 0; j < g->k; ++j)
        if (cudaMemcpyAsync(static_cast<uint8_t *>(states_out) + j * ld * es,
                            static_cast<const uint8_t *>(states_in) + j * ld * es, nstreams * es,
                            cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)) != cudaSuccess)
          return cuda_fail("cudaMemcpyAsync(states)");
    }
    return SLP_OK;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // few, long substreams: segment split.  Contiguous stream-major rows: the
  // segments are plain rows of pitch T/J.  Padded stream-major rows: segment
  // (i, j) is row i, column j*T/J, through the 4-D store map (TMA-addressable
  // output only: 128-byte aligned base, 16-byte row pitch and segment
  // length).  Position-major: segments in j-major order (lanes = consecutive
  // substreams of one row block), written through the 2-D store map when a
  // warp's segments share a row block, else with element stores.
  uint64_t J = split_factor(*g, nstreams, T);
  if (J > 1 && layout == SLP_STREAM_MAJOR && ld_out != T) {
    const uint64_t es = out_kind == SLP_OUT_NATIVE ? g->w / 8 : (out_kind == SLP_OUT_F32 ? 4 : 8);
    if ((uintptr_t)out % 128 != 0 || (ld_out * es) % 16 != 0 || ((T / J) * es) % 16 != 0) J = 1;
  }
  if (J > 1) {
    const bool pm = layout == SLP_POSITION_MAJOR;
    Segments seg;
    int rc = make_segments(id, *g, states_in, ld, nstreams, T, J, st, seg, pm);
    if (rc != SLP_OK) return rc;
    FillParams q = p;
    q.sin = q.sout = seg.states;
    q.ld = q.nstreams = nstreams * J;
    q.T = T / J;
    if (pm) {
      q.pm_n = nstreams;
    } else if (ld_out == T) {
      q.ld_out = T / J;
    } else {
      int sh = 0;
      while ((1ull << sh) < J) ++sh;
      q.jsh = (uint32_t)sh;
    }
    rc = ops->fill(q, out_kind, layout, st);
    if (rc != SLP_OK || !states_out) return rc;
    return segment_ends(*g, seg, nstreams, J, states_out, ld, st, pm ? 1 : 0);
  }
  return ops->fill(p, out_kind, layout, st);
}

int slp_fill_checksum(int id, const void *states_in, void *states_out, uint64_t ld, uint64_t nstreams, uint64_t T,
                      int out_kind, void *out, uint64_t ld_out, void *result, void *workspace,
                      size_t workspace_bytes, void *stream) {
  const GenDesc *g = gen_desc(id);
  if (!g) return SLP_ERR_UNKNOWN_GENERATOR;
  const GenOps *ops = gen_ops(id);
  if (!ops) return SLP_ERR_UNSUPPORTED;
  if (!result || !workspace) return SLP_ERR_INVALID;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int grid = 0;
  if (nstreams > 0 && T > 0) {
    if (!states_in || !out || ld < nstreams || ld_out < T) return SLP_ERR_INVALID;
    FillParams p{};
    p.rt = gen_rt(id);
    p.sin = states_in;
    p.sout = states_out;
    p.ld = ld;
    p.nstreams = nstreams;
    p.T = T;
    p.out = out;
    p.ld_out = ld_out;
    p.partials = workspace;
    p.workspace_bytes = workspace_bytes;
    const uint64_t J = ld_out == T ? split_factor(*g, nstreams, T) : 1;
    if (J > 1) {
      Segments seg;
      int rc = make_segments(id, *g, states_in, ld, nstreams, T, J, st, seg);
      if (rc != SLP_OK) return rc;
      FillParams q = p;
      q.sin = q.sout = seg.states;
      q.ld = q.nstreams = nstreams * J;
      q.T = q.ld_out = T / J;
      rc = ops->fill_csum(q, out_kind, st, &grid);
      if (rc == SLP_OK && states_out) rc = segment_ends(*g, seg, nstreams, J, states_out, ld, st);
      if (rc != SLP_OK) return rc;
    } else {
      const int rc = ops->fill_csum(p, out_kind, st, &grid);
      if (rc != SLP_OK) return rc;
    }
  }
  const double fscale = g->w == 64 ? 0x1.0p-64 : 0x1.0p-24;  // fterm in k_fused
  dev::k_fused_final<<<1, 256, 0, st>>>(static_cast<const slp_checksum *>(workspace), grid,
                                        static_cast<slp_checksum *>(result), nstreams * T, fscale);
  return check_launch("k_fused_final");
}

size_t slp_fused_workspace_bytes(int id, uint64_t nstreams) {
  (void)nstreams;
  const GenOps *ops = gen_ops(id);
  if (!ops) return 0;
  const int dev = current_device();
  if (dev < 0) return 0;
  return (size_t)ops->fused_grid_cap(dev) * sizeof(slp_checksum);
}

int slp_fused(int id, const void *states_in, void *states_out, uint64_t ld, uint64_t nstreams, uint64_t T, int flags,
              void *result, void *workspace, size_t workspace_bytes, void *stream) {
  const GenDesc *g = gen_desc(id);
  if (!g) return SLP_ERR_UNKNOWN_GENERATOR;
  const GenOps *ops = gen_ops(id);
  if (!ops) return SLP_ERR_UNSUPPORTED;
  if (!states_in || !result || !workspace || ld < nstreams || !(flags & (SLP_FUSE_INT | SLP_FUSE_F64 | SLP_FUSE_EXACT)))
    return SLP_ERR_INVALID;
  FusedParams p{};
  p.rt = gen_rt(id);
  p.sin = states_in;
  p.sout = states_out;
  p.ld = ld;
  p.nstreams = nstreams;
  p.T = T;
  p.partials = workspace;
  p.workspace_bytes = workspace_bytes;
  p.one = 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int grid = 0;
  int rc;
  const uint64_t J = split_factor(*g, nstreams, T, (uint64_t)env_int("SLP_FUSED_SPLIT_NMAX", 1 << 15));
  if (J > 1) {
    Segments seg;
    rc = make_segments(id, *g, states_in, ld, nstreams, T, J, st, seg);
    if (rc != SLP_OK) return rc;
    FusedParams q = p;
    q.sin = q.sout = seg.states;
    q.ld = q.nstreams = nstreams * J;
    q.T = T / J;
    rc = ops->fused(q, flags, st, &grid);
    if (rc == SLP_OK && states_out) rc = segment_ends(*g, seg, nstreams, J, states_out, ld, st);
  } else {
    rc = ops->fused(p, flags, st, &grid);
  }
  if (rc != SLP_OK) return rc;
  const double fscale = g->w == 64 ? 0x1.0p-64 : 0x1.0p-24;  // fterm in k_fused
  dev::k_fused_final<<<1, 256, 0, st>>>(static_cast<const slp_checksum *>(workspace), grid,
                                        static_cast<slp_checksum *>(result), nstreams * T, fscale);
  return check_launch("k_fused_final");
}

int slp_hwd_count(int id, const void *states, uint64_t ld, uint64_t nthreads, uint64_t tseg, uint64_t total,
                  uint64_t warm, uint64_t warm0, int k, int lo, int hi, int transitional, int split,
                  uint64_t *counts, uint64_t *sums, uint64_t *overflow_ctas, void *stream) {
  const GenDesc *g = gen_desc(id);
  if (!g) return SLP_ERR_UNKNOWN_GENERATOR;
  const GenOps *ops = gen_ops(id);
  if (!ops) return SLP_ERR_UNSUPPORTED;
  if (!states || !counts || !sums || k < 1 || k > 16 || ld < nthreads || tseg == 0) return SLP_ERR_INVALID;
  if (split && g->w != 64) return SLP_ERR_INVALID;
  if (total > nthreads * tseg || (nthreads && total <= (nthreads - 1) * tseg)) return SLP_ERR_INVALID;
  if (tseg >= (1ull << 32) || warm > 64 || warm0 > 64) return SLP_ERR_INVALID;
  HwdParams p{};
  p.rt = gen_rt(id);
  p.sin = states;
  p.ld = ld;
  p.nthreads = nthreads;
  p.tseg = tseg;
  p.total = total;
  p.warm = warm;
  p.warm0 = warm0;
  p.lo = lo;
  p.hi = hi;
  uint32_t pw = 1;
  for (int j = 1; j < k; ++j) pw *= 3;
  p.pow3k1 = pw;
  p.ncells = pw * 3;
  // k <= 9: all 3^k packed cells in one CTA's shared memory (<= 77 KB).
  // k = 10, 11: slices of <= 24K cells (96 KB, two CTAs per SM), each CTA
  // regenerating its segments per slice (measured 1.5e11 / 5.1e10 values/s
  // against 6.2e10 / ~4e10 with global atomics).  Beyond kMaxHwdSlices slices
  // (k >= 12) the repeated generation costs more than 64-bit global atomics.
  // SLP_HWD_SLICES=0 forces global atomics for k > 9 (A/B, tests).
  constexpr uint32_t kSliceCells = 24576, kMaxHwdSlices = 8;
  const char *ev = std::getenv("SLP_HWD_SLICES");
  const bool allow_slices = !(ev && *ev == '0');
  if (p.ncells <= 19683) {
    p.global_cells = 0;
    p.slice_cells = p.ncells;
  } else {
    const uint32_t nsl = (p.ncells + kSliceCells - 1) / kSliceCells;
    p.global_cells = (allow_slices && nsl <= kMaxHwdSlices) ? 0 : 1;
    p.slice_cells = (p.ncells + nsl - 1) / nsl;
  }
  p.g_counts = reinterpret_cast<unsigned long long *>(counts);
  p.g_sums = reinterpret_cast<unsigned long long *>(sums);
  p.overflow_ctas = reinterpret_cast<unsigned long long *>(overflow_ctas);
  if (nthreads == 0) return SLP_OK;
  return ops->hwd(p, transitional, split, static_cast<cudaStream_t>(stream));
}

int slp_set_fill_pace(int gbps) {
  const int prev = fill_pace_gbps();
  if (gbps >= 0) g_pace_gbps.store(gbps, std::memory_order_relaxed);
  return prev;
}

size_t slp_device_cache_bytes(int device) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  auto it = g_cache_bytes.find(device);
  return it == g_cache_bytes.end() ? 0 : it->second;
}

const char *slp_build_info(void) {
  return "slp_b200 sm_100a (tcgen05-free integer path; TMA bulk tensor stores) built " __DATE__ " " __TIME__;
}

}  // extern "C"
