// Microbenchmark: issue throughput of integer ops on sm_100a (which pipe, what rate).
// Each thread runs 8 independent chains; reports lane-ops per SM per cycle.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define N_ITERS 4096

template <int OP>
__global__ void k(uint32_t *out, uint32_t seed) {
  uint32_t a[8];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = seed * (threadIdx.x + 17 * i + 1);
  uint32_t m = seed | 0x01010101u;
  for (int it = 0; it < N_ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      uint32_t x = a[i], r;
      if (OP == 0) {  // LOP3 (ALU)
        asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(x), "r"(m), "r"(a[(i + 1) & 7]));
      } else if (OP == 1) {  // IMAD (mad.lo)
        asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(m), "r"(a[(i + 1) & 7]));
      } else if (OP == 2) {  // mul.hi (IMAD.HI)
        asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(m));
        r += 0;
      } else if (OP == 3) {  // shr by constant (SHF)
        asm volatile("shr.b32 %0, %1, 7;" : "=r"(r) : "r"(x));
      } else if (OP == 4) {  // prmt (ALU)
        asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(r) : "r"(x), "r"(m));
      } else if (OP == 5) {  // add (IADD3 or IMAD.IADD)
        asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(m));
      } else if (OP == 6) {  // half LOP3, half mad: do both pipes overlap?
        if (i & 1)
          asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(x), "r"(m), "r"(a[(i + 1) & 7]));
        else
          asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(m), "r"(a[(i + 1) & 7]));
      } else if (OP == 7) {  // half LOP3, half mul.hi
        if (i & 1)
          asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(x), "r"(m), "r"(a[(i + 1) & 7]));
        else
          asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(m));
      } else if (OP == 8) {  // popc
        asm volatile("popc.b32 %0, %1;" : "=r"(r) : "r"(x));
        r ^= x;
      } else {  // shf.l.wrap (funnel)
        asm volatile("shf.l.wrap.b32 %0, %1, %2, 8;" : "=r"(r) : "r"(x), "r"(a[(i + 1) & 7]));
      }
      a[i] = r;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  uint32_t *out;
  cudaMalloc(&out, (size_t)sms * 8 * 1024 * 4);
  const char *names[] = {"lop3", "mad.lo", "mul.hi", "shr", "prmt", "add", "lop3+mad", "lop3+mulhi",
                         "popc", "shf.l.wrap"};
  void (*fns[])(uint32_t *, uint32_t) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>};
  for (int op = 0; op < 10; op++) {
    int blocks = sms * 8, threads = 256;
    fns[op]<<<blocks, threads>>>(out, 3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    fns[op]<<<blocks, threads>>>(out, 5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * N_ITERS * 8;
    double per_sm_cycle = ops / (ms * 1e-3) / sms / 1.965e9;  // assume max clock
    printf("%-12s %8.3f ms  %7.1f lane-ops/SM/cycle (@1.965GHz)\n", names[op], ms, per_sm_cycle);
  }
  printf("clock attr %d kHz, %d SMs, err=%s\n", clk, sms, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
