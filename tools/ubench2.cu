// Integer issue-model microbenchmark for sm_100a: throughput (lane-ops / SM / cycle) of single
// opcodes and of 1:1 mixes, with register-only and immediate operand forms.  8 independent
// chains per thread, no cross-chain dependences.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench2 tools/ubench2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N_ITERS 2048

template <int OP>
__device__ __forceinline__ uint32_t op1(uint32_t x, uint32_t m, int i) {
  uint32_t r;
  switch (OP) {
    case 0: asm volatile("lop3.b32 %0, %1, %2, %1, 0x96;" : "=r"(r) : "r"(x), "r"(m)); break;
    case 1: asm volatile("lop3.b32 %0, %1, 0x0F0F0F0F, %1, 0x6a;" : "=r"(r) : "r"(x)); break;
    case 2: asm volatile("mad.lo.u32 %0, %1, 0x01010101, %2;" : "=r"(r) : "r"(x), "r"(m)); break;
    case 3: asm volatile("mad.lo.u32 %0, %1, %2, %1;" : "=r"(r) : "r"(x), "r"(m)); break;
    case 4: asm volatile("shf.l.wrap.b32 %0, %1, %2, 8;" : "=r"(r) : "r"(x), "r"(m)); break;
    case 5: asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(r) : "r"(x), "r"(m)); break;
    case 6: asm volatile("add.u32 %0, %1, 0x01010101;" : "=r"(r) : "r"(x)); break;
    case 7: asm volatile("shl.b32 %0, %1, 3;" : "=r"(r) : "r"(x)); break;
    case 8: asm volatile("shr.u32 %0, %1, 3;" : "=r"(r) : "r"(x)); break;
    case 9: { float f = __uint_as_float(x); asm volatile("fma.rn.f32 %0, %1, 0f3F800001, 0f3F800000;" : "=f"(f) : "f"(f)); r = __float_as_uint(f); } break;
    // mixes (alternate by chain index)
    case 10: if (i & 1) asm volatile("lop3.b32 %0, %1, 0x0F0F0F0F, %1, 0x6a;" : "=r"(r) : "r"(x));
             else asm volatile("mad.lo.u32 %0, %1, 0x01010101, %2;" : "=r"(r) : "r"(x), "r"(m)); break;
    case 11: if (i & 1) asm volatile("lop3.b32 %0, %1, 0x0F0F0F0F, %1, 0x6a;" : "=r"(r) : "r"(x));
             else asm volatile("shl.b32 %0, %1, 3;" : "=r"(r) : "r"(x)); break;
    case 12: if (i & 1) asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(r) : "r"(x), "r"(m));
             else asm volatile("mad.lo.u32 %0, %1, 0x01010101, %2;" : "=r"(r) : "r"(x), "r"(m)); break;
    case 13: if (i & 1) asm volatile("lop3.b32 %0, %1, 0x0F0F0F0F, %1, 0x6a;" : "=r"(r) : "r"(x));
             else { float f = __uint_as_float(x); asm volatile("fma.rn.f32 %0, %1, 0f3F800001, 0f3F800000;" : "=f"(f) : "f"(f)); r = __float_as_uint(f); } break;
    case 14: if (i & 1) asm volatile("lop3.b32 %0, %1, 0x0F0F0F0F, %1, 0x6a;" : "=r"(r) : "r"(x));
             else asm volatile("add.u32 %0, %1, 0x01010101;" : "=r"(r) : "r"(x)); break;
    case 15: if (i & 1) asm volatile("shf.l.wrap.b32 %0, %1, %2, 8;" : "=r"(r) : "r"(x), "r"(m));
             else asm volatile("mad.lo.u32 %0, %1, 0x01010101, %2;" : "=r"(r) : "r"(x), "r"(m)); break;
    case 16: if (i % 3 == 0) asm volatile("lop3.b32 %0, %1, 0x0F0F0F0F, %1, 0x6a;" : "=r"(r) : "r"(x));
             else if (i % 3 == 1) asm volatile("mad.lo.u32 %0, %1, 0x01010101, %2;" : "=r"(r) : "r"(x), "r"(m));
             else { float f = __uint_as_float(x); asm volatile("fma.rn.f32 %0, %1, 0f3F800001, 0f3F800000;" : "=f"(f) : "f"(f)); r = __float_as_uint(f); } break;
    default: asm volatile("popc.b32 %0, %1;" : "=r"(r) : "r"(x)); break;
  }
  return r;
}

template <int OP>
__global__ void k(uint32_t *out, uint32_t seed) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = seed * (threadIdx.x + 17 * i + 1);
  const uint32_t m = seed | 0x01010101u;
  for (int it = 0; it < N_ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) a[i] = op1<OP>(a[i], m, i);
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char *name, uint32_t *out, int sms, double clk_ghz) {
  int blocks = sms * 8, threads = 256;
  k<OP><<<blocks, threads>>>(out, 3);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP><<<blocks, threads>>>(out, 5);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * N_ITERS * 8;
  printf("%-22s %8.3f ms %8.1f lane-ops/SM/cycle\n", name, ms, ops / (ms * 1e-3) / sms / (clk_ghz * 1e9));
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double g = clk / 1e6;
  uint32_t *out;
  cudaMalloc(&out, (size_t)sms * 8 * 256 * 4);
  run<0>("lop3 rrr", out, sms, g);
  run<1>("lop3 r,imm", out, sms, g);
  run<2>("imad r,imm,r", out, sms, g);
  run<3>("imad rrr", out, sms, g);
  run<4>("shf.l.wrap", out, sms, g);
  run<5>("prmt", out, sms, g);
  run<6>("add imm", out, sms, g);
  run<7>("shl imm", out, sms, g);
  run<8>("shr imm", out, sms, g);
  run<9>("ffma imm", out, sms, g);
  run<10>("lop3imm+imad", out, sms, g);
  run<11>("lop3imm+shl", out, sms, g);
  run<12>("prmt+imad", out, sms, g);
  run<13>("lop3imm+ffma", out, sms, g);
  run<14>("lop3imm+add", out, sms, g);
  run<15>("shf+imad", out, sms, g);
  run<16>("lop3+imad+ffma", out, sms, g);
  run<99>("popc", out, sms, g);
  printf("clock %d kHz, %d SMs, %s\n", clk, sms, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
