// TMA write-pattern ceiling for the POSITION-major layout out[t][stream]
// (no generation): each CTA owns `rows` consecutive substreams and streams
// 2-D TMA stores of a constant [ch positions][rows] tile along t.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a profiles/wpattern_tma_pm.cu -o profiles/wpattern_tma_pm.bin
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void k_tma(const __grid_constant__ CUtensorMap map, int nunits, int ntiles, int ch, int rows, int tile_bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem);
  for (int i = threadIdx.x; i < 3 * tile_bytes / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(smem)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  int issued = 0;
  for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
    for (int c = 0; c < ntiles; ++c) {
      if (issued >= 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      const uint32_t src = base + (issued % 3) * tile_bytes;
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                       reinterpret_cast<uint64_t>(&map)),
                   "r"(src), "r"(u * rows), "r"(c * ch)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      ++issued;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
  int rowss[] = {32, 128, 256};
  int chs[] = {4, 8, 16};
  for (int rows : rowss)
    for (int ch : chs) {
      const int tile_bytes = rows * ch * 8;
      const int smem = 3 * tile_bytes + 1024;
      if (smem > 227 * 1024) continue;
      CUtensorMap map;
      cuuint64_t gdim[2] = {N, T};
      cuuint64_t gstr[1] = {N * 8};
      cuuint32_t box[2] = {(cuuint32_t)rows, (cuuint32_t)ch};
      cuuint32_t es[2] = {1, 1};
      CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, buf, gdim, gstr, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("encode failed %d (rows %d ch %d)\n", (int)r, rows, ch);
        continue;
      }
      cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tma, 128, smem);
      const int grid = sms * per_sm;
      const int nunits = N / rows, ntiles = T / ch;
      k_tma<<<grid, 128, smem>>>(map, nunits, ntiles, ch, rows, tile_bytes);
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      for (int i = 0; i < 10; ++i) k_tma<<<grid, 128, smem>>>(map, nunits, ntiles, ch, rows, tile_bytes);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("{\"layout\": \"position\", \"rows\": %d, \"ch\": %d, \"ctas_per_sm\": %d, \"GBps\": %.1f, \"err\": \"%s\"}\n",
             rows, ch, per_sm, T * N * 8 * 10 / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
