// TMA write-pattern ceiling (no generation): each warp streams 3-D TMA stores
// of a constant 32-row x (segs x 128 B) shared-memory tile along its 32 rows,
// exactly the geometry of k_fill's FILL_TMA mode, for several segs and
// buffers per warp (the TMA-only ceiling of each fill configuration).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a profiles/wpattern_tma.cu -o profiles/wpattern_tma.bin
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void k_tma(const __grid_constant__ CUtensorMap map, int nunits, int ntiles, int segs, int warps, int bufs) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem) + warp * bufs * 32 * segs * 128;
  for (int i = lane; i < bufs * 32 * segs * 128 / 4; i += 32) reinterpret_cast<uint32_t *>(smem + (base - (uint32_t)__cvta_generic_to_shared(smem)))[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  int issued = 0;
  for (int u = blockIdx.x * warps + warp; u < nunits; u += gridDim.x * warps) {
    for (int c = 0; c < ntiles; ++c) {
      if (lane == 0) {
        if (bufs == 1 && issued >= 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if (bufs == 2 && issued >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        const uint32_t src = base + (issued % bufs) * 32 * segs * 128;
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                         reinterpret_cast<uint64_t>(&map)),
                     "r"(src), "r"(0), "r"(u * 32), "r"(c * segs)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      ++issued;
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const uint64_t T = 1024, N = 1 << 20;  // u64 elements
  uint8_t *buf;
  cudaMalloc(&buf, (T + 256) * N * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void *fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int segss[] = {1, 2, 4, 8};
  int warpss[] = {4, 7};
  int pads[] = {0, 16, 32, 64, 256};
  for (int pad : pads)
  for (int segs : segss)
    for (int warps : warpss)
    for (int bufs = 1; bufs <= 2; ++bufs) {
      if (pad != 0 && (segs == 8 || bufs == 1)) continue;  // padding: old sweep only
      const int smem = warps * bufs * 32 * segs * 128 + 1024;
      if (smem > 227 * 1024) continue;
      CUtensorMap map;
      cuuint64_t gdim[3] = {16, N, T / 16};
      cuuint64_t gstr[2] = {(T + pad) * 8, 128};
      cuuint32_t box[3] = {16, 32, (cuuint32_t)segs};
      cuuint32_t es[3] = {1, 1, 1};
      CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, buf, gdim, gstr, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", (int)r);
        continue;
      }
      cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tma, warps * 32, smem);
      const int grid = sms * per_sm;
      const int nunits = N / 32, ntiles = T / (16 * segs);
      k_tma<<<grid, warps * 32, smem>>>(map, nunits, ntiles, segs, warps, bufs);
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      for (int i = 0; i < 10; ++i) k_tma<<<grid, warps * 32, smem>>>(map, nunits, ntiles, segs, warps, bufs);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("{\"pad\": %d, \"segs\": %d, \"warps_per_cta\": %d, \"bufs\": %d, \"ctas_per_sm\": %d, \"GBps\": %.1f, \"err\": \"%s\"}\n",
             pad, segs, warps, bufs, per_sm, T * N * 8 * 10 / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
