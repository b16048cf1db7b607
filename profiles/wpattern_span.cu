// Does HBM write bandwidth depend on the address span written concurrently?
// (1) one-shot grid of 4 KiB chunks, CTA order permuted inside windows of W
//     bytes (W = 4 KiB: sequential sweep; W = 8 GiB: scattered);
// (2) stream-major rows (8 KiB, warp owns 32 rows, 1 KiB pieces) with the
//     number of warps in flight varied -> concurrently written span = warps x 256 KiB.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a profiles/wpattern_span.cu -o /tmp/wspan
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void st256(void *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

// chunk i -> window (i / wc), position inside the window (i % wc) * mul mod wc (mul odd)
__global__ void k_chunk_perm(uint8_t *out, uint64_t wc, uint64_t mul) {
  const uint64_t i = blockIdx.x;
  const uint64_t c = (i / wc) * wc + ((i % wc) * mul) % wc;
  uint8_t *base = out + c * 4096;
  for (int o = threadIdx.x * 32; o < 4096; o += blockDim.x * 32) st256(base + o, o, 1, 2, 3);
}

__global__ void k_rows(uint8_t *out, size_t nrows, int L, int P) {
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  const int per_row = P / 32;
  for (size_t u = warp; u < nrows / 32; u += nwarps) {
    uint8_t *base = out + u * 32 * (size_t)L;
    for (int col = 0; col < L; col += P)
      for (int k = lane; k < 32 * per_row; k += 32) {
        const int r = k / per_row, c = k % per_row;
        st256(base + (size_t)r * L + col + c * 32, k, 1, 2, 3);
      }
  }
}

// phase-major rows: the whole grid writes columns [col, col+P) of all rows
// before moving on (state save/restore between phases would be needed for a
// generator); span per phase = all rows but only P bytes of each
__global__ void k_rows_phase(uint8_t *out, size_t nrows, int L, int P, int col) {
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  const int per_row = P / 32;
  for (size_t u = warp; u < nrows / 32; u += nwarps) {
    uint8_t *base = out + u * 32 * (size_t)L;
    for (int k = lane; k < 32 * per_row; k += 32) {
      const int r = k / per_row, c = k % per_row;
      st256(base + (size_t)r * L + col + c * 32, k, 1, 2, 3);
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
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("{\"pattern\": \"%s\", \"error\": \"%s\"}\n", name, cudaGetErrorString(e));
      return;
    }
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("{\"pattern\": \"%s\", \"GBps\": %.1f}\n", name, bytes / (best * 1e6));
  };
  const uint64_t nch = bytes / 4096;
  for (uint64_t wmb : {0ull, 1ull, 4ull, 16ull, 64ull, 128ull, 256ull, 1024ull, 8192ull}) {
    const uint64_t wc = wmb == 0 ? 1 : wmb * 256;  // chunks per window
    char name[64];
    snprintf(name, sizeof name, "chunk_window_%lluMiB", (unsigned long long)wmb);
    run(name, [&] { k_chunk_perm<<<nch, 128>>>(buf, wc, wc == 1 ? 1 : 40503); });
  }
  const int L = 8192;
  const size_t nrows = bytes / L;
  for (int wps : {1, 2, 4, 7, 14}) {
    char name[64];
    snprintf(name, sizeof name, "rows_P1024_warps_per_sm_%d", wps);
    run(name, [&] { k_rows<<<sms, 32 * wps>>>(buf, nrows, L, 1024); });
    snprintf(name, sizeof name, "rows_P512_warps_per_sm_%d", wps);
    run(name, [&] { k_rows<<<sms, 32 * wps>>>(buf, nrows, L, 512); });
  }
  for (int P : {512, 1024, 2048}) {
    char name[64];
    snprintf(name, sizeof name, "rows_phase_P%d", P);
    run(name, [&] {
      for (int col = 0; col < L; col += P) k_rows_phase<<<sms * 7, 224>>>(buf, nrows, L, P, col);
    });
  }
  return 0;
}
