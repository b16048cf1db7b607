// Why does torch's fill_ (7.5 TB/s) beat a plain uint4 grid-stride store
// (6.1 TB/s)?  Sequential and stream-major write patterns with 128-bit vs
// 256-bit stores, grid-stride vs one-shot grids, and TMA bulk (linear) stores.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a profiles/wpattern_seq.cu -o /tmp/wseq
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void st256(void *p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void st128(void *p, uint64_t a, uint64_t b) {
  asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

// grid-stride, VB bytes per thread per iteration (16 or 32)
template <int VB>
__global__ void k_seq(uint8_t *out, size_t n) {
  size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * VB;
  const size_t stride = (size_t)gridDim.x * blockDim.x * VB;
  for (; i < n; i += stride) {
    if (VB == 32)
      st256(out + i, i, 1, 2, 3);
    else
      st128(out + i, i, 1);
  }
}

// one-shot grid: each CTA writes a contiguous chunk of CH bytes (torch-style
// vectorized elementwise: block_work_size contiguous per block)
template <int VB, int CH>
__global__ void k_chunk(uint8_t *out) {
  uint8_t *base = out + (size_t)blockIdx.x * CH;
#pragma unroll
  for (int o = threadIdx.x * VB; o < CH; o += blockDim.x * VB) {
    if (VB == 32)
      st256(base + o, o, 1, 2, 3);
    else
      st128(base + o, o, 1);
  }
}

// stream-major rows of L bytes, warp owns 32 rows, writes P bytes per row per step
// with VB-byte stores (lanes sweep a row piece, then the next row)
template <int VB>
__global__ void k_rows(uint8_t *out, size_t nrows, int L, int P) {
  const int lane = threadIdx.x & 31;
  const size_t warp = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nwarps = ((size_t)gridDim.x * blockDim.x) >> 5;
  const int per_row = P / VB;
  for (size_t u = warp; u < nrows / 32; u += nwarps) {
    uint8_t *base = out + u * 32 * (size_t)L;
    for (int col = 0; col < L; col += P)
      for (int k = lane; k < 32 * per_row; k += 32) {
        const int r = k / per_row, c = k % per_row;
        uint8_t *p = base + (size_t)r * L + col + c * VB;
        if (VB == 32)
          st256(p, k, 1, 2, 3);
        else
          st128(p, k, 1);
      }
  }
}

// TMA linear bulk store (cp.async.bulk.global.shared::cta) of CH-byte chunks,
// one elected thread per warp, NB buffers of CH bytes per warp
template <int CH>
__global__ void k_bulk(uint8_t *out, size_t n) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint8_t *mine = sm + warp * CH;
  for (int o = lane * 16; o < CH; o += 512) *reinterpret_cast<uint4 *>(mine + o) = make_uint4(o, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  const size_t nch = n / CH;
  for (size_t c = blockIdx.x * (size_t)nw + warp; c < nch; c += (size_t)gridDim.x * nw) {
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * CH),
                   "r"((uint32_t)__cvta_generic_to_shared(mine)), "r"(CH)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
  run("seq128_sms_x4_x256", [&] { k_seq<16><<<sms * 4, 256>>>(buf, bytes); });
  run("seq128_sms_x8_x256", [&] { k_seq<16><<<sms * 8, 256>>>(buf, bytes); });
  run("seq128_sms_x32_x256", [&] { k_seq<16><<<sms * 32, 256>>>(buf, bytes); });
  run("seq256_sms_x4_x256", [&] { k_seq<32><<<sms * 4, 256>>>(buf, bytes); });
  run("seq256_sms_x8_x256", [&] { k_seq<32><<<sms * 8, 256>>>(buf, bytes); });
  run("seq256_sms_x32_x256", [&] { k_seq<32><<<sms * 32, 256>>>(buf, bytes); });
  run("chunk128_4K_x128", [&] { k_chunk<16, 4096><<<bytes / 4096, 128>>>(buf); });
  run("chunk128_16K_x256", [&] { k_chunk<16, 16384><<<bytes / 16384, 256>>>(buf); });
  run("chunk256_4K_x128", [&] { k_chunk<32, 4096><<<bytes / 4096, 128>>>(buf); });
  run("chunk256_16K_x128", [&] { k_chunk<32, 16384><<<bytes / 16384, 128>>>(buf); });
  run("chunk256_16K_x256", [&] { k_chunk<32, 16384><<<bytes / 16384, 256>>>(buf); });
  for (int P : {256, 512, 1024}) {
    char name[64];
    const int L = 8192;
    snprintf(name, sizeof name, "rows128_P%d", P);
    run(name, [&] { k_rows<16><<<sms * 7, 224>>>(buf, bytes / L, L, P); });
    snprintf(name, sizeof name, "rows256_P%d", P);
    run(name, [&] { k_rows<32><<<sms * 7, 224>>>(buf, bytes / L, L, P); });
    snprintf(name, sizeof name, "rows256_P%d_16w", P);
    run(name, [&] { k_rows<32><<<sms * 4, 512>>>(buf, bytes / L, L, P); });
  }
  cudaFuncSetAttribute(k_bulk<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  cudaFuncSetAttribute(k_bulk<4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4096);
  run("bulk16K_8w", [&] { k_bulk<16384><<<sms, 256, 8 * 16384>>>(buf, bytes); });
  run("bulk4K_8w", [&] { k_bulk<4096><<<sms * 2, 256, 8 * 4096>>>(buf, bytes); });
  run("bulk4K_8w_x6", [&] { k_bulk<4096><<<sms * 6, 256, 8 * 4096>>>(buf, bytes); });
  run("memset", [&] { cudaMemsetAsync(buf, 7, bytes); });
  return 0;
}
