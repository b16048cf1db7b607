// Legacy warp-level 1-bit MMA (mma.sync m16n8k256 b1 AND+POPC -> BMMA) throughput
// on sm_100a: dependency-free streams, all SMs (one op = one bit AND + popc
// accumulate, i.e. one GF(2) multiply-accumulate).  Decides whether a
// mma.sync GF(2) jump could beat the four-Russians K1t (it needs
// n^2 multiply-accumulates per state).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a profiles/bmma_peak.cu -o /tmp/bmma
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 4, ITERS = 2048;

__global__ void k(int *out) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 0x01010101u + i;
  for (int i = 0; i < 2; ++i) b[i] = threadIdx.x * 0x01000101u + i;
  int c[CH][4] = {};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  int r = 0;
  for (int j = 0; j < CH; ++j) r += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (r == 123456789) out[0] = r;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int *out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    const int grid = sms * 2, block = warps * 32;
    k<<<grid, block>>>(out);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      k<<<grid, block>>>(out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    const double ops = (double)grid * warps * ITERS * CH * 16 * 8 * 256;
    printf("{\"warps_per_cta\": %d, \"bit_AND_POPC_TOPS\": %.1f}\n", warps, ops / (best / 1e3) / 1e12);
  }
  return 0;
}
