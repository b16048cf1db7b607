// Round 2 write-pattern study, part 3 (no generation): does a WARP-SPECIALISED
// store path beat the 3-D TMA row store of k_fill (6.15 TB/s, config 2)?
// Persistent grid, 1 CTA per SM, G "generator" warps that each own a 32 KiB
// tile (32 stream-major rows x 1 KiB piece) and spin S dependent ALU rounds per
// tile to mimic generation time (k_fill: ~10k cycles per tile per warp at
// config 2), then hand the tile off.  8 GiB per launch, best of 5 x 3 launches.
//
//   mech TMA:  the generator warp issues one 3-D TMA store of its tile (k_fill today);
//   mech STG:  the generator warp reads its tile back (LDS.128) and stores it
//              with STG.128 itself (the round-2 `stg1` k_fill variant);
//   mech TMAW: as TMA, but the buffer wait is for the store to COMPLETE
//              (cp.async.bulk.wait_group 0), bounding the writes in flight;
//   mech NONE: spin only (the generation-only time);
//   mech WS1/WS2: K = 1 or 2 extra store warps; generator warp g hands its tile
//              to store warp g % K through an mbarrier (full[g]) and waits for
//              the store warp to have read it back (empty[g]) before the next
//              tile; store warps do LDS.128 + STG.128, row by row.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a profiles/wpattern_r3.cu -o /tmp/wr3 -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

enum { TMA = 0, STG = 1, WS = 2, TMAW = 3, NONE = 4, TMAP = 5, TMAPC = 6 };
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st16(uint8_t *p, uint4 v) {
  asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void mb_init(uint32_t a, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint32_t a) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mb_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(
          a),
      "r"(parity)
      : "memory");
}

// stores one 32 x P tile (row r piece = P bytes at out + (row0 + r) * 8192 + c*P) with STG.128
__device__ __forceinline__ void store_tile_stg(const uint8_t *tile, uint8_t *out, uint64_t row0, uint64_t c, int P,
                                               int lane) {
  uint8_t *ub = out + row0 * 8192 + c * P;
  const int tile_bytes = 32 * P;
#pragma unroll 8
  for (int i = lane * 16; i < tile_bytes; i += 512) {
    const int r = i / P, o = i % P;
    st16(ub + (uint64_t)r * 8192 + o, *reinterpret_cast<const uint4 *>(tile + i));
  }
}

template <int MECH>
__global__ void k_w(const __grid_constant__ CUtensorMap map, uint8_t *out, uint64_t total, int G, int K, int spin,
                    uint32_t *sink, uint32_t period) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int P = 1024, TB = 32 * P;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + G * TB);  // full[G], empty[G]
  const uint32_t full0 = (uint32_t)__cvta_generic_to_shared(bars), empty0 = full0 + 8 * G;
  if (threadIdx.x == 0) {
    for (int g = 0; g < G; ++g) mb_init(full0 + 8 * g, 1), mb_init(empty0 + 8 * g, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x * 16; i < G * TB; i += blockDim.x * 16)
    *reinterpret_cast<uint4 *>(smem + i) = make_uint4(i, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint64_t tiles_per_unit = 8192 / P;
  const uint64_t nunits = total / (32ull * 8192);
  const uint64_t ustride = (uint64_t)gridDim.x * G;
  if (warp < G) {  // generator warp
    const int g = warp;
    uint8_t *mine = smem + g * TB;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(mine);
    uint32_t x = lane + 1;
    uint32_t n = 0;
    uint64_t next = 0;
    for (uint64_t u = (uint64_t)blockIdx.x * G + g; u < nunits; u += ustride) {
      for (uint64_t c = 0; c < tiles_per_unit; ++c, ++n) {
        for (int s = 0; s < spin; ++s) x ^= x << 13, x ^= x >> 17, x ^= x << 5;
        if constexpr (MECH == NONE) {
        } else if constexpr (MECH == TMA || MECH == TMAW || MECH == TMAP || MECH == TMAPC) {
          __syncwarp();
          if (lane == 0) {
            if constexpr (MECH == TMAP) {  // per-warp pacing on the global timer (ns)
              uint64_t now = gtimer();
              while (now < next) now = gtimer();
              next = (now > next + period ? now : next) + period;
            } else if constexpr (MECH == TMAPC) {  // per-warp pacing on the SM clock (cycles)
              uint64_t now = clock64();
              while (now < next) now = clock64();
              next = (now > next + period ? now : next) + period;
            }
            if constexpr (MECH == TMAW) {
              if (n >= 1) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            } else {
              if (n >= 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                             reinterpret_cast<uint64_t>(&map)),
                         "r"(base), "r"(0), "r"((int)(u * 32)), "r"((int)(c * P / 128))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          __syncwarp();
        } else if constexpr (MECH == STG) {
          store_tile_stg(mine, out, u * 32, c, P, lane);
          __syncwarp();
        } else {
          if (n >= 1) mb_wait(empty0 + 8 * g, (n - 1) & 1);
          // (the real kernel writes the tile here)
          *reinterpret_cast<uint32_t *>(mine + lane * 16) = x;
          __syncwarp();
          if (lane == 0) mb_arrive(full0 + 8 * g);
        }
      }
    }
    if constexpr (MECH == TMA || MECH == TMAW || MECH == TMAP || MECH == TMAPC)
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (x == 0x12345) sink[0] = x;
  } else if constexpr (MECH == WS) {  // store warp k serves generator warps g = k, k + K, ...
    const int k = warp - G;
    // every generator warp runs the same number of tiles except at the grid tail
    uint32_t n = 0;
    for (uint64_t ub = blockIdx.x * (uint64_t)G; ub < nunits; ub += ustride) {
      for (uint64_t c = 0; c < tiles_per_unit; ++c, ++n) {
        for (int g = k; g < G; g += K) {
          const uint64_t u = ub + g;
          if (u >= nunits) break;
          mb_wait(full0 + 8 * g, n & 1);
          store_tile_stg(smem + g * TB, out, u * 32, c, P, lane);
          __syncwarp();
          if (lane == 0) mb_arrive(empty0 + 8 * g);
        }
      }
    }
  }
}

// Paced pure-store pattern study: G warps per CTA (1 CTA per SM), each owning
// 32 stream-major 8 KiB rows and storing P-byte pieces (3-D TMA box of 32 rows
// x P/128 segments); tile buffers are ALIASED (warp g uses buffer g % nbuf),
// since only the address pattern matters here -- this lets the study go past
// the 227 KiB of shared memory (e.g. 14 warps x 1 KiB pieces).  period = ns
// between one warp's stores (0 = unpaced).
__global__ void k_p(const __grid_constant__ CUtensorMap map, uint64_t total, int G, int P, int nbuf, uint32_t period,
                    int spin, uint32_t *sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int TB = 32 * P;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem + (g % nbuf) * TB);
  const uint64_t tiles_per_unit = 8192 / P;
  const uint64_t nunits = total / (32ull * 8192);
  const uint64_t ustride = (uint64_t)gridDim.x * G;
  uint32_t x = lane + 1, n = 0;
  uint64_t next = 0;
  for (uint64_t u = (uint64_t)blockIdx.x * G + g; u < nunits; u += ustride) {
    for (uint64_t c = 0; c < tiles_per_unit; ++c, ++n) {
      for (int s = 0; s < spin; ++s) x ^= x << 13, x ^= x >> 17, x ^= x << 5;
      __syncwarp();
      if (lane == 0) {
        if (period) {
          uint64_t now = gtimer();
          while (now < next) now = gtimer();
          next = (now > next + period ? now : next) + period;
        }
        if (n >= 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                         reinterpret_cast<uint64_t>(&map)),
                     "r"(base), "r"(0), "r"((int)(u * 32)), "r"((int)(c * P / 128))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      __syncwarp();
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (x == 0x12345) sink[0] = x;
}

int main(int argc, char **argv) {
  const uint64_t total = 8ull << 30;
  uint8_t *buf;
  uint32_t *sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 64);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void *fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  CUtensorMap map;
  {
    const uint64_t nrows = total / 8192;
    cuuint64_t gdim[3] = {16, nrows, 8192 / 128};
    cuuint64_t gstr[2] = {8192, 128};
    cuuint32_t box[3] = {16, 32, 8};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  }
  auto run = [&](const char *mech, auto kern, int G, int K, int spin, uint32_t period = 0) {
    const int smem = G * 32 * 1024 + 16 * G + 64;
    const int threads = (G + K) * 32;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<sms, threads, smem>>>(map, buf, total, G, K, spin, sink, period);
    cudaError_t e = cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5 && e == cudaSuccess; ++rep) {
      cudaEventRecord(a);
      for (int i = 0; i < 3; ++i) kern<<<sms, threads, smem>>>(map, buf, total, G, K, spin, sink, period);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms / 3 < best) best = ms / 3;
    }
    e = e == cudaSuccess ? cudaGetLastError() : e;
    printf("{\"mech\": \"%s\", \"gen_warps\": %d, \"store_warps\": %d, \"spin\": %d, \"period\": %u, \"ms\": %.4f, "
           "\"GBps\": %.1f, \"err\": \"%s\"}\n",
           mech, G, K, spin, period, best, total / (best * 1e6), cudaGetErrorString(e));
    fflush(stdout);
  };
  if (argc > 1 && argv[1][0] == 'g') {  // warps x piece size under pacing (aliased buffers)
    auto mk = [&](int P) {
      CUtensorMap m;
      cuuint64_t gdim[3] = {16, total / 8192, 8192 / 128};
      cuuint64_t gstr[2] = {8192, 128};
      cuuint32_t box[3] = {16, 32, (cuuint32_t)(P / 128)};
      cuuint32_t es[3] = {1, 1, 1};
      encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      return m;
    };
    const int smem = 224 * 1024;
    cudaFuncSetAttribute(k_p, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int P : {512, 1024}) {
      const CUtensorMap m = mk(P);
      for (int G : {7, 14, 21}) {
        const int nbuf = smem / (32 * P) < G ? smem / (32 * P) : G;
        for (int gbps = 0; gbps <= 7400; gbps += (gbps == 0 ? 5800 : 200)) {
          const uint32_t period = gbps ? (uint32_t)(32.0 * P * G * sms / gbps) : 0;
          k_p<<<sms, G * 32, smem>>>(m, total, G, P, nbuf, period, 0, sink);
          cudaError_t e = cudaDeviceSynchronize();
          float best = 1e30f;
          for (int rep = 0; rep < 5 && e == cudaSuccess; ++rep) {
            cudaEventRecord(a);
            for (int i = 0; i < 3; ++i) k_p<<<sms, G * 32, smem>>>(m, total, G, P, nbuf, period, 0, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms / 3 < best) best = ms / 3;
          }
          printf("{\"mech\": \"TMAP\", \"warps\": %d, \"piece\": %d, \"target_gbps\": %d, \"ms\": %.4f, "
                 "\"GBps\": %.1f, \"err\": \"%s\"}\n",
                 G, P, gbps, best, total / (best * 1e6), cudaGetErrorString(e));
          fflush(stdout);
        }
      }
    }
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'p') {  // paced stores: per-warp period for a target aggregate rate
    const int nw = 7 * sms;
    for (int spin : {0, 200}) {
      run("TMA", k_w<TMA>, 7, 0, spin);
      for (int gbps = 6000; gbps <= 7400; gbps += 100) {
        const double per_ns = 32768.0 * nw / gbps;  // ns between a warp's tiles
        run("TMAP", k_w<TMAP>, 7, 0, spin, (uint32_t)per_ns);
      }
      for (int gbps = 6200; gbps <= 7200; gbps += 200) {
        const double per_cyc = 32768.0 * nw / gbps * 1.9;  // at ~1.9 GHz
        run("TMAPC", k_w<TMAPC>, 7, 0, spin, (uint32_t)per_cyc);
      }
    }
    return 0;
  }
  if (argc > 1 && argv[1][0] == 'f') {  // fine sweep around the rate-matched point
    for (int spin = 200; spin <= 400; spin += 20) {
      run("NONE", k_w<NONE>, 7, 0, spin);
      run("TMA", k_w<TMA>, 7, 0, spin);
      run("TMAW", k_w<TMAW>, 7, 0, spin);
      run("STG", k_w<STG>, 7, 0, spin);
    }
    for (int spin : {0, 100}) run("TMAW", k_w<TMAW>, 7, 0, spin);
    return 0;
  }
  const int spins[] = {0, 100, 200, 300, 400, 600};
  for (int spin : spins) {
    run("TMA", k_w<TMA>, 7, 0, spin);
    run("STG", k_w<STG>, 7, 0, spin);
    run("WS", k_w<WS>, 7, 1, spin);
    run("WS", k_w<WS>, 7, 2, spin);
    run("WS", k_w<WS>, 6, 2, spin);
  }
  return 0;
}
