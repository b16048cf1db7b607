// Round 2 write-pattern study (no generation): which store MECHANISM caps a
// persistent fill kernel (1 CTA per SM, W warps, a 32 KiB shared tile per
// warp)?  8 GiB per launch, best of 5 x 5 launches.
//
//   pattern ROWS: stream-major 8 KiB rows, warp owns 32 rows, writes a P-byte
//                 piece of each of its 32 rows per tile (k_fill's pattern);
//   pattern LIN:  warp tile = one contiguous 32 KiB block, tiles in unit order
//                 (the pattern of a segment-parallel fill: 8 lanes per row);
//   mechanism TMA3: 3-D bulk tensor store (k_fill today);
//   mechanism BULK: 1-D cp.async.bulk.global.shared::cta (LIN only);
//   mechanism STG:  the warp reads its tile back (LDS.128) and writes it with
//                   coalesced 16-byte stores (STG.128), 512 B per instruction;
//   mechanism STGCS: same with st.global.cs (streaming, evict-first);
//   mechanism STGNA: same with st.global.L1::no_allocate.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a profiles/wpattern_r2.cu -o /tmp/wr2 -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

enum { TMA3 = 0, BULK = 1, STG = 2, STGCS = 3, STGNA = 4 };
enum { ROWS = 0, LIN = 1 };

template <int MECH>
__device__ __forceinline__ void st16(uint8_t *p, uint4 v) {
  if constexpr (MECH == STGCS)
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  else if constexpr (MECH == STGNA)
    asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
  else
    asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// P = bytes per row piece (ROWS); a tile is 32 x P bytes.  spin = ALU work per
// tile (iterations of a dependent xorshift chain) to mimic generation time.
template <int MECH, int PAT>
__global__ void k_w(const __grid_constant__ CUtensorMap map, uint8_t *out, uint64_t total, int P, int spin,
                    uint32_t *sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
  const int tile_bytes = 32 * P;
  uint8_t *mine = smem + warp * tile_bytes;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(mine);
  for (int i = lane * 16; i < tile_bytes; i += 512) *reinterpret_cast<uint4 *>(mine + i) = make_uint4(i, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const uint64_t row_bytes = 8192;
  const uint64_t ntiles_total = total / tile_bytes;
  const uint64_t tiles_per_unit = PAT == ROWS ? row_bytes / P : 1;  // ROWS: a unit = 32 rows
  const uint64_t nunits = ntiles_total / tiles_per_unit;
  uint32_t x = lane + 1;
  int issued = 0;
  for (uint64_t u = (uint64_t)blockIdx.x * warps + warp; u < nunits; u += (uint64_t)gridDim.x * warps) {
    for (uint64_t c = 0; c < tiles_per_unit; ++c) {
      for (int s = 0; s < spin; ++s) x ^= x << 13, x ^= x >> 17, x ^= x << 5;
      if constexpr (MECH == TMA3 || MECH == BULK) {
        __syncwarp();
        if (lane == 0) {
          if (issued >= 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          if constexpr (MECH == TMA3) {
            if constexpr (PAT == ROWS)
              asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                               reinterpret_cast<uint64_t>(&map)),
                           "r"(base), "r"(0), "r"((int)(u * 32)), "r"((int)(c * P / 128))
                           : "memory");
            else  // LIN as 1 KiB virtual rows: 32 rows x 8 pieces of 128 B
              asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                               reinterpret_cast<uint64_t>(&map)),
                           "r"(base), "r"(0), "r"((int)(u * 32)), "r"(0)
                           : "memory");
          } else {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + u * tile_bytes),
                         "r"(base), "r"(tile_bytes)
                         : "memory");
          }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        __syncwarp();
      } else {
        if constexpr (PAT == ROWS) {
          // row r piece: 32 rows x P bytes, each row piece = P / 512 warp stores
          uint8_t *ub = out + u * 32 * row_bytes + c * P;
          for (int i = lane * 16; i < tile_bytes; i += 512) {
            const int r = i / P, o = i % P;
            const uint4 v = *reinterpret_cast<const uint4 *>(mine + i);
            st16<MECH>(ub + (uint64_t)r * row_bytes + o, v);
          }
        } else {
          uint8_t *ub = out + u * tile_bytes;
#pragma unroll 8
          for (int i = lane * 16; i < tile_bytes; i += 512) st16<MECH>(ub + i, *reinterpret_cast<const uint4 *>(mine + i));
        }
        __syncwarp();
      }
      ++issued;
    }
  }
  if constexpr (MECH == TMA3 || MECH == BULK)
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (x == 0x12345) sink[0] = x;
}

int main() {
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
  auto mkmap = [&](uint64_t rowlen_bytes, int P) {
    CUtensorMap map;
    const uint64_t nrows = total / rowlen_bytes;
    cuuint64_t gdim[3] = {16, nrows, rowlen_bytes / 128};
    cuuint64_t gstr[2] = {rowlen_bytes, 128};
    cuuint32_t box[3] = {16, 32, (cuuint32_t)(P / 128)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, buf, gdim, gstr, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
    return map;
  };
  auto run = [&](const char *mech, const char *pat, auto kern, const CUtensorMap &map, int P, int warps, int ctas,
                 int spin) {
    const int smem = warps * 32 * P + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem);
    if (per_sm < ctas) {
      printf("{\"mech\": \"%s\", \"pat\": \"%s\", \"P\": %d, \"warps\": %d, \"ctas_per_sm\": %d, \"skip\": \"occupancy %d\"}\n",
             mech, pat, P, warps, ctas, per_sm);
      return;
    }
    const int grid = sms * ctas;
    kern<<<grid, warps * 32, smem>>>(map, buf, total, P, spin, sink);
    cudaError_t e = cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5 && e == cudaSuccess; ++rep) {
      cudaEventRecord(a);
      for (int i = 0; i < 5; ++i) kern<<<grid, warps * 32, smem>>>(map, buf, total, P, spin, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms / 5 < best) best = ms / 5;
    }
    printf("{\"mech\": \"%s\", \"pat\": \"%s\", \"P\": %d, \"warps\": %d, \"ctas_per_sm\": %d, \"spin\": %d, "
           "\"GBps\": %.1f, \"err\": \"%s\"}\n",
           mech, pat, P, warps, ctas, spin, total / (best * 1e6), cudaGetErrorString(e));
    fflush(stdout);
  };
  const CUtensorMap m_rows = mkmap(8192, 1024), m_lin = mkmap(1024, 1024);
  for (int spin : {0, 64}) {
    for (int warps : {4, 7}) {
      run("TMA3", "ROWS", k_w<TMA3, ROWS>, m_rows, 1024, warps, 1, spin);
      run("TMA3", "LIN", k_w<TMA3, LIN>, m_lin, 1024, warps, 1, spin);
      run("BULK", "LIN", k_w<BULK, LIN>, m_lin, 1024, warps, 1, spin);
      run("STG", "ROWS", k_w<STG, ROWS>, m_rows, 1024, warps, 1, spin);
      run("STG", "LIN", k_w<STG, LIN>, m_lin, 1024, warps, 1, spin);
      run("STGCS", "ROWS", k_w<STGCS, ROWS>, m_rows, 1024, warps, 1, spin);
      run("STGCS", "LIN", k_w<STGCS, LIN>, m_lin, 1024, warps, 1, spin);
      run("STGNA", "LIN", k_w<STGNA, LIN>, m_lin, 1024, warps, 1, spin);
    }
    // more store-issuing warps: 2 CTAs x 3 warps, 1 CTA x 14 warps of 512 B pieces
    run("STG", "ROWS", k_w<STG, ROWS>, m_rows, 512, 14, 1, spin);
    run("STG", "LIN", k_w<STG, LIN>, m_lin, 512, 14, 1, spin);
    run("STGCS", "LIN", k_w<STGCS, LIN>, m_lin, 512, 14, 1, spin);
    run("STG", "LIN", k_w<STG, LIN>, m_lin, 256, 16, 2, spin);
  }
  return 0;
}
