// Write-pattern microbenchmark (no generation): how fast can B200 HBM absorb
// the stream-major fill's write pattern?  A CTA owns R consecutive rows of
// L bytes; in each step it writes a P-byte piece of every one of its rows
// (column sweep), exactly like the fill kernel's tiles, with 16-byte stores.
// Compared against a sequential grid-stride write (memset-like ceiling).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a profiles/wpattern.cu -o /tmp/wpattern
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_seq(uint4 *out, size_t n16) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const uint4 v = make_uint4(i, 1, 2, 3);
  for (; i < n16; i += stride) out[i] = v;
}

// rows of L bytes; CTA unit = R rows; piece P bytes per row per step
__global__ void k_rows(uint8_t *out, size_t nrows, int L, int R, int P) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per_row16 = P / 16;
  const size_t nunits = nrows / R;
  const uint4 v = make_uint4(tid, 7, 8, 9);
  for (size_t u = blockIdx.x; u < nunits; u += gridDim.x) {
    uint8_t *base = out + u * (size_t)R * L;
    for (int col = 0; col < L; col += P) {
      // R*P/16 16-byte stores per step, threads sweep rows fastest within a piece
      for (int k = tid; k < R * per_row16; k += nt) {
        const int r = k / per_row16, c = k % per_row16;
        *reinterpret_cast<uint4 *>(base + (size_t)r * L + col + c * 16) = v;
      }
    }
  }
}

int main() {
  const size_t bytes = 8ull << 30;
  uint8_t *buf;
  cudaMalloc(&buf, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  auto run = [&](const char *name, auto fn) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) fn();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"pattern\": \"%s\", \"GBps\": %.1f}\n", name, bytes * 10 / (ms * 1e6));
  };
  run("seq_grid_sms_x4_x256", [&] { k_seq<<<sms * 4, 256>>>((uint4 *)buf, bytes / 16); });
  run("seq_grid_sms_x8_x256", [&] { k_seq<<<sms * 8, 256>>>((uint4 *)buf, bytes / 16); });
  const int L = 8192;
  const size_t nrows = bytes / L;
  int Rs[] = {32, 256};
  int Ps[] = {64, 128, 256, 512, 1024, 8192};
  for (int R : Rs)
    for (int P : Ps) {
      char name[64];
      snprintf(name, sizeof name, "rows_R%d_P%d", R, P);
      int ctas = sms * (R == 32 ? 16 : 4);
      int nt = R == 32 ? 64 : 256;
      run(name, [&] { k_rows<<<ctas, nt>>>(buf, nrows, L, R, P); });
    }
  return 0;
}
