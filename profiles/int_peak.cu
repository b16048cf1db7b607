// Measured integer-pipe peaks on this B200 (the INT roofline of kernel K4):
// long dependency-free streams of LOP3 (ALU pipe), SHF.L.W (ALU pipe) and
// IMAD (FMA pipe), and an ALU+FMA mix, all SMs, CUDA events.
// Reports warp-instructions per second per GPU and per SM per cycle.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a profiles/int_peak.cu -o /tmp/int_peak
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 8;       // independent chains per thread
constexpr int ITERS = 4096;

template <int OP>
__global__ void k(uint32_t *out, uint32_t seed) {
  uint32_t a[CH], b[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    a[c] = seed + threadIdx.x * 7 + c;
    b[c] = seed ^ (c * 0x9E3779B9u);
  }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) {  // LOP3: 3-input xor
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(b[c]), "r"(i));
      } else if (OP == 1) {  // funnel shift (rotate)
        asm volatile("shf.l.wrap.b32 %0, %0, %1, 13;" : "+r"(a[c]) : "r"(b[c]));
      } else if (OP == 2) {  // IMAD
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(b[c]), "r"(i));
      } else if (OP == 4) {  // IMAD.WIDE (64-bit result)
        uint64_t w;
        asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(a[c]), "r"(b[c]), "l"((uint64_t)i));
        a[c] = (uint32_t)w ^ (uint32_t)(w >> 32);
      } else if (OP == 5) {  // IMAD.HI
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(b[c]));
      } else if (OP == 6) {  // LEA-style 64-bit x*5 = x + (x << 2) via add.cc (lo) / addc (hi)
        asm volatile("{\n\t.reg .u32 t;\n\tshl.b32 t, %0, 2;\n\tadd.u32 %0, %0, t;\n\t}" : "+r"(a[c]));
      } else {  // ALU + FMA interleaved
        if (c & 1)
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(b[c]), "r"(i));
        else
          asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(b[c]), "r"(i));
      }
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) r ^= a[c];
  if (r == 0x12345678u) out[0] = r;
}

// Pipe overlap: NA chains of LOP3 (ALU pipe) next to CH - NA chains of OPB
// (0 none, 2 IMAD, 4 IMAD.WIDE, 5 IMAD.HI).  If the pipes overlap, the time is
// max(ALU part, FMA part); if OPB also occupies the ALU pipe (or the shared
// dispatch), it approaches their sum.  Decides whether moving shifts /
// rotations of K4 to IMAD.HI forms can pay (K4).
template <int NA, int OPB>
__global__ void kmix(uint32_t *out, uint32_t seed) {
  uint32_t a[CH], b[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) {
    a[c] = seed + threadIdx.x * 7 + c;
    b[c] = seed ^ (c * 0x9E3779B9u);
  }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (c < NA) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[c]) : "r"(b[c]), "r"(i));
      } else if (OPB == 2) {
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[c]) : "r"(b[c]), "r"(i));
      } else if (OPB == 4) {
        uint64_t w;
        asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(w) : "r"(a[c]), "r"(b[c]), "l"((uint64_t)i));
        a[c] = (uint32_t)(w >> 32);
      } else if (OPB == 5) {
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[c]) : "r"(b[c]));
      }
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) r ^= a[c];
  if (r == 0x12345678u) out[0] = r;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t *out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char *names[] = {"LOP3 (ALU)", "SHF.L.W (ALU)", "IMAD (FMA)", "LOP3+IMAD mix", "IMAD.WIDE (+1 LOP3 fold)",
                         "IMAD.HI", "x + (x << 2) (LEA)"};
  auto run = [&](int op, auto kern) {
    const int grid = sms * 8, block = 256;
    kern<<<grid, block>>>(out, 1);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      kern<<<grid, block>>>(out, 1);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    const double winst = (double)grid * block / 32 * ITERS * CH;
    const double per_s = winst / (best / 1e3);
    printf("{\"op\": \"%s\", \"warp_inst_per_s\": %.4g, \"per_sm_per_cycle_at_max_clock\": %.3f}\n", names[op], per_s,
           per_s / sms / (clk * 1e3));
  };
  run(0, k<0>);
  run(1, k<1>);
  run(2, k<2>);
  run(3, k<3>);
  run(4, k<4>);
  run(5, k<5>);
  run(6, k<6>);
  auto mix = [&](const char *what, int na, int nb, auto kern) {
    const int grid = sms * 8, block = 256;
    kern<<<grid, block>>>(out, 1);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      kern<<<grid, block>>>(out, 1);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    // SM cycles (at max clock) per warp iteration (na LOP3 + nb other)
    const double iters = (double)grid * block / 32 * ITERS;
    printf("{\"mix\": \"%s\", \"lop3\": %d, \"other\": %d, \"ms\": %.4f, \"sm_cycles_per_warp_iter\": %.3f}\n", what, na,
           nb, best, best / 1e3 * (clk * 1e3) * sms / iters);
  };
  mix("6 LOP3", 6, 0, kmix<6, 0>);
  mix("6 LOP3 + 2 IMAD", 6, 2, kmix<6, 2>);
  mix("6 LOP3 + 2 IMAD.HI", 6, 2, kmix<6, 5>);
  mix("6 LOP3 + 2 IMAD.WIDE", 6, 2, kmix<6, 4>);
  mix("4 LOP3", 4, 0, kmix<4, 0>);
  mix("4 LOP3 + 4 IMAD", 4, 4, kmix<4, 2>);
  mix("4 LOP3 + 4 IMAD.HI", 4, 4, kmix<4, 5>);
  mix("7 LOP3 + 1 IMAD.HI", 7, 1, kmix<7, 5>);
  mix("7 LOP3", 7, 0, kmix<7, 0>);
  mix("8 LOP3", 8, 0, kmix<8, 0>);
  mix("0 LOP3 + 8 IMAD.HI", 0, 8, kmix<0, 5>);
  mix("0 LOP3 + 8 IMAD", 0, 8, kmix<0, 2>);
  return 0;
}
