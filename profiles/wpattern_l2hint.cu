// Can L2 eviction priorities turn the stream-major column sweep into whole-row
// DRAM write-backs?  TMA-only k_fill geometry (7 warps x 32 rows, 1 KiB row
// pieces, 1 buffer) with:  0 plain stores;  1 evict_first;  2 evict_last
// stores + applypriority evict_normal on the unit's rows once complete;
// 3 evict_last only.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a profiles/wpattern_l2hint.cu -o /tmp/wl2 -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int MODE>
__global__ void k_tma(const __grid_constant__ CUtensorMap map, uint8_t *out, int nunits, int ntiles, int segs,
                      int warps, uint64_t row_bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem) + warp * 32 * segs * 128;
  for (int i = lane; i < 32 * segs * 128 / 4; i += 32)
    reinterpret_cast<uint32_t *>(smem + (base - (uint32_t)__cvta_generic_to_shared(smem)))[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  uint64_t pol = 0;
  if (MODE == 1) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (MODE >= 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  int issued = 0;
  int prev_u = -1;
  for (int u = blockIdx.x * warps + warp; u < nunits; u += gridDim.x * warps) {
    for (int c = 0; c < ntiles; ++c) {
      if (lane == 0) {
        if (issued >= 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if (MODE == 0)
          asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                           reinterpret_cast<uint64_t>(&map)),
                       "r"(base), "r"(0), "r"(u * 32), "r"(c * segs)
                       : "memory");
        else
          asm volatile(
              "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3, %4}], [%1], %5;" ::"l"(
                  reinterpret_cast<uint64_t>(&map)),
              "r"(base), "r"(0), "r"(u * 32), "r"(c * segs), "l"(pol)
              : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      ++issued;
      __syncwarp();
    }
    if (MODE == 2) {
      // previous unit is complete (its stores were committed a whole unit ago):
      // demote its lines so L2 writes back whole rows
      if (prev_u >= 0) {
        uint8_t *p0 = out + (uint64_t)prev_u * 32 * row_bytes;
        for (uint64_t off = lane * 128; off < 32 * row_bytes; off += 32 * 128)
          asm volatile("applypriority.global.L2::evict_normal [%0], 128;" ::"l"(p0 + off) : "memory");
      }
      prev_u = u;
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const uint64_t T = 1024, N = 1 << 20;  // u64 elements
  uint8_t *buf;
  cudaMalloc(&buf, T * N * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void *fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int segs = 8, warps = 7;
  const int smem = warps * 32 * segs * 128 + 1024;
  CUtensorMap map;
  cuuint64_t gdim[3] = {16, N, T / 16};
  cuuint64_t gstr[2] = {T * 8, 128};
  cuuint32_t box[3] = {16, 32, (cuuint32_t)segs};
  cuuint32_t es[3] = {1, 1, 1};
  encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int nunits = N / 32, ntiles = T / (16 * segs);
  auto run = [&](const char *name, auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<sms, warps * 32, smem>>>(map, buf, nunits, ntiles, segs, warps, T * 8);
    cudaError_t e = cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      kern<<<sms, warps * 32, smem>>>(map, buf, nunits, ntiles, segs, warps, T * 8);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("{\"mode\": \"%s\", \"GBps\": %.1f, \"err\": \"%s\"}\n", name, T * N * 8 / (best * 1e6), cudaGetErrorString(e));
  };
  run("plain", k_tma<0>);
  run("evict_first", k_tma<1>);
  run("evict_last+applypriority_normal", k_tma<2>);
  run("evict_last", k_tma<3>);
  return 0;
}
