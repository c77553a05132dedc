// Micro-benchmark: per-SM issue rate of the integer/DPX instructions the SW
// recurrence uses, on sm_100a. Each thread runs ILP independent chains of one
// op for ITERS iterations; rate = thread-ops / (elapsed SM cycles * #SMs).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ILP 8
#define ITERS 4096

template <int OP>
__global__ void bench(unsigned *out, unsigned seed, long long *cyc) {
  unsigned v[ILP];
  unsigned a = seed ^ threadIdx.x, b = seed * 3u + 1u, c = seed + 7u;
#pragma unroll
  for (int k = 0; k < ILP; ++k) v[k] = a + k * 0x10001u;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      if (OP == 0) v[k] = (unsigned)__viaddmax_s32((int)v[k], (int)b, (int)c);
      if (OP == 1) v[k] = __viaddmax_s16x2(v[k], b, c);
      if (OP == 2) v[k] = (unsigned)__vimax3_s32((int)v[k], (int)b, (int)c);
      if (OP == 3) v[k] = __vimax3_s16x2_relu(v[k], b, c);
      if (OP == 4) v[k] = (unsigned)max((int)v[k], (int)c) + b;   // IMNMX + IADD
      if (OP == 5) v[k] = v[k] + b + c;                            // IADD3
      if (OP == 6) v[k] = __viaddmax_s16x2_relu(v[k], b, c);
      if (OP == 7) v[k] = (unsigned)__vimax_s32_relu((int)v[k], (int)c);
      if (OP == 8) v[k] = __byte_perm(v[k], b, 0x5410);            // PRMT
      if (OP == 9) v[k] = (unsigned)__viaddmax_s32_relu((int)v[k], (int)b, (int)c);
      if (OP == 10) v[k] = v[k] * b + c;                            // IMAD
    }
  }
  long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) acc ^= v[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char *name, int sms) {
  int blocks = sms * 4, threads = 512;  // 64 warps/SM
  unsigned *out; long long *cyc;
  cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
  bench<OP><<<blocks, threads>>>(out, 1, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<OP><<<blocks, threads>>>(out, 2, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long h[4096]; cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double mc = 0; for (int i = 0; i < blocks; ++i) mc = h[i] > mc ? h[i] : mc;
  double ops = (double)blocks * threads * ILP * ITERS;
  // per-SM per-cycle rate using the slowest block's cycle count (4 blocks co-resident per SM)
  double per_sm_clk = ops / sms / mc;
  printf("%-26s %8.2f thread-ops/clk/SM  (%.1f warp-instr/clk/SM)  %.3f Tops/s  %.3f ms\n", name,
         per_sm_clk, per_sm_clk / 32, ops / ms / 1e9, ms);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  printf("%s  SMs=%d  clock=%d kHz\n", p.name, sms, p.clockRate);
  run<0>("viaddmax_s32", sms);
  run<1>("viaddmax_s16x2", sms);
  run<2>("vimax3_s32", sms);
  run<3>("vimax3_s16x2_relu", sms);
  run<4>("imnmx+iadd (2 ops)", sms);
  run<5>("iadd3 (1 op)", sms);
  run<6>("viaddmax_s16x2_relu", sms);
  run<7>("vimax_s32_relu", sms);
  run<8>("prmt", sms);
  run<9>("viaddmax_s32_relu", sms);
  run<10>("imad", sms);
  return 0;
}
