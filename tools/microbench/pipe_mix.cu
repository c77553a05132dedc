// Micro-benchmark: which integer pipes co-issue with the DPX (VIADDMNMX) pipe on
// sm_100a. Each kernel interleaves one DPX op with one "other" op per chain.
#include <cstdio>
#include <cuda_runtime.h>

#define ILP 8
#define ITERS 2048

__device__ __forceinline__ unsigned prmt(unsigned a, unsigned b, unsigned s) {
  unsigned d; asm volatile("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(s)); return d; }
__device__ __forceinline__ unsigned lop3(unsigned a, unsigned b, unsigned c) {
  unsigned d; asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ unsigned iadd3(unsigned a, unsigned b, unsigned c) {
  unsigned d; asm volatile("add.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); asm volatile("add.u32 %0, %0, %1;" : "+r"(d) : "r"(c)); return d; }
__device__ __forceinline__ unsigned imad(unsigned a, unsigned b, unsigned c) {
  unsigned d; asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ unsigned vmax2(unsigned a, unsigned b) {
  unsigned d; asm volatile("max.s16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned vmax32(unsigned a, unsigned b) {
  unsigned d; asm volatile("max.s32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned addm(unsigned a, unsigned b, unsigned c) {  // DPX
  return __viaddmax_s16x2(a, b, c); }

// OP selects the pair: 0 dpx only, 1 dpx+imad, 2 dpx+prmt, 3 dpx+lop3, 4 dpx+iadd,
// 5 dpx+vmax2, 6 dpx+vmax32, 7 vmax2 only, 8 lop3 only, 9 iadd only, 10 imad only,
// 11 dpx+shfl, 12 dpx + 2*imad, 13 dpx+imad+vmax2
template <int OP>
__global__ void bench(unsigned *out, unsigned seed, long long *cyc) {
  unsigned v[ILP], w[ILP];
  unsigned b = seed * 3u + 1u, c = seed + 7u;
#pragma unroll
  for (int k = 0; k < ILP; ++k) { v[k] = seed ^ (threadIdx.x + k); w[k] = v[k] * 7u; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      if (OP <= 6 || OP >= 11) v[k] = addm(v[k], b, c);
      if (OP == 1 || OP == 10 || OP == 12 || OP == 13) w[k] = imad(w[k], b, c);
      if (OP == 12) w[k] = imad(w[k], c, b);
      if (OP == 2) w[k] = prmt(w[k], b, 0x5410);
      if (OP == 3 || OP == 8) w[k] = lop3(w[k], b, c);
      if (OP == 4 || OP == 9) w[k] = iadd3(w[k], b, c);
      if (OP == 5 || OP == 7 || OP == 13) w[k] = vmax2(w[k], c + k);
      if (OP == 6) w[k] = vmax32(w[k], c + k);
      if (OP == 11) w[k] = __shfl_up_sync(0xffffffffu, w[k], 1);
    }
  }
  long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) acc ^= v[k] ^ w[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char *name, int sms, int nops) {
  int blocks = sms * 4, threads = 512;
  unsigned *out; long long *cyc;
  cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
  bench<OP><<<blocks, threads>>>(out, 1, cyc);
  bench<OP><<<blocks, threads>>>(out, 2, cyc);
  cudaDeviceSynchronize();
  long long h[4096]; cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double mc = 0; for (int i = 0; i < blocks; ++i) mc = h[i] > mc ? h[i] : mc;
  double steps = (double)blocks * threads * ILP * ITERS;  // each step = nops thread-ops
  double per_sm_clk = steps / sms / mc;
  printf("%-22s %7.2f steps/clk/SM  = %6.2f thread-ops/clk/SM  (%.2f warp-instr/clk/SMSP)\n", name,
         per_sm_clk, per_sm_clk * nops, per_sm_clk * nops / 32 / 4);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  run<0>("dpx", sms, 1);
  run<1>("dpx+imad", sms, 2);
  run<2>("dpx+prmt", sms, 2);
  run<3>("dpx+lop3", sms, 2);
  run<4>("dpx+2iadd", sms, 3);
  run<5>("dpx+vmax.s16x2", sms, 2);
  run<6>("dpx+vmax.s32", sms, 2);
  run<7>("vmax.s16x2", sms, 1);
  run<8>("lop3", sms, 1);
  run<9>("2iadd", sms, 2);
  run<10>("imad", sms, 1);
  run<11>("dpx+shfl", sms, 2);
  run<12>("dpx+2imad", sms, 3);
  run<13>("dpx+imad+vmax2", sms, 3);
  return 0;
}
