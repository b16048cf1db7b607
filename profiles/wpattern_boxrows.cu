// Round 2: does the TMA box height cap the stream-major row pattern?  The
// config-2 geometry (warp = 32 rows of 8 KiB, 1 KiB pieces, one 32 KiB smem
// tile per warp, 7 warps, one CTA per SM) stored as 32/R boxes of R rows x
// 1 KiB per tile (R = 32: k_fill's aligned path; R = 8: FILL_TMA_G's row
// groups for odd T), and as 32 one-row 1-D bulk copies of 1 KiB.  No
// generation.  8 GiB per launch, best of 5 x 5 launches.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a profiles/wpattern_boxrows.cu -o /tmp/wbox -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void k_box(const __grid_constant__ CUtensorMap map, uint8_t *out, uint64_t nrows, int R, int bulk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, warps = blockDim.x >> 5;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem) + warp * 32768;
  for (int i = lane * 16; i < 32768; i += 512) *reinterpret_cast<uint4 *>(smem + warp * 32768 + i) = make_uint4(i, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const uint64_t nunits = nrows / 32;
  int issued = 0;
  for (uint64_t u = (uint64_t)blockIdx.x * warps + warp; u < nunits; u += (uint64_t)gridDim.x * warps) {
    for (int c = 0; c < 8; ++c) {
      if (lane == 0) {
        if (issued >= 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        if (bulk) {
          for (int r = 0; r < 32; ++r)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 1024;" ::"l"(
                             out + ((u * 32 + r) * 8 + c) * 1024),
                         "r"(base + r * 1024)
                         : "memory");
        } else {
          for (int g = 0; g < 32 / R; ++g)
            asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                             reinterpret_cast<uint64_t>(&map)),
                         "r"(base + g * R * 1024), "r"(0), "r"((int)(u * 32 + g * R)), "r"(c * 8)
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      __syncwarp();
      ++issued;
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const uint64_t N = 1 << 20, T = 1024;  // u64
  uint8_t *buf;
  cudaMalloc(&buf, N * T * 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void *fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int smem = 7 * 32768 + 1024;
  cudaFuncSetAttribute(k_box, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int R : {32, 16, 8, 0}) {
    CUtensorMap map;
    cuuint64_t gdim[3] = {16, N, T / 16};
    cuuint64_t gstr[2] = {T * 8, 128};
    cuuint32_t box[3] = {16, (cuuint32_t)(R ? R : 32), 8};
    cuuint32_t es[3] = {1, 1, 1};
    encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k_box<<<sms, 224, smem>>>(map, buf, N, R ? R : 32, R == 0);
    cudaError_t e = cudaDeviceSynchronize();
    float best = 1e30f;
    for (int rep = 0; rep < 5 && e == cudaSuccess; ++rep) {
      cudaEventRecord(a);
      for (int i = 0; i < 5; ++i) k_box<<<sms, 224, smem>>>(map, buf, N, R ? R : 32, R == 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms / 5 < best) best = ms / 5;
    }
    printf("{\"box_rows\": %d, \"mode\": \"%s\", \"GBps\": %.1f, \"err\": \"%s\"}\n", R ? R : 1,
           R ? "3-D tensor" : "1-D bulk per row", N * T * 8 / (best * 1e6), cudaGetErrorString(e));
  }
  return 0;
}
