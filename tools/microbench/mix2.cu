// Micro-benchmark 2: issue cost of non-DPX integer mixes on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#define ILP 8
#define ITERS 2048
__device__ __forceinline__ unsigned vmax32(unsigned a, unsigned b) { unsigned d; asm volatile("max.s32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned vmaxu2(unsigned a, unsigned b) { unsigned d; asm volatile("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned imad(unsigned a, unsigned b, unsigned c) { unsigned d; asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ unsigned add3(unsigned a, unsigned b, unsigned c) { unsigned d; asm volatile("{.reg .u32 t; add.u32 t, %1, %2; add.u32 %0, t, %3;}" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ unsigned prmt(unsigned a, unsigned b) { unsigned d; asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned vmax3(unsigned a, unsigned b, unsigned c) { return (unsigned)__vimax3_s32((int)a, (int)b, (int)c); }

template <int OP>
__global__ void bench(unsigned *out, unsigned seed, long long *cyc) {
  unsigned v[ILP], w[ILP], x[ILP];
  unsigned b = seed * 3u + 1u, c = seed + 7u;
#pragma unroll
  for (int k = 0; k < ILP; ++k) { v[k] = seed ^ (threadIdx.x + k); w[k] = v[k] * 7u; x[k] = v[k] ^ 0x55u; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      if (OP == 0) { v[k] = vmax32(v[k], c + k); }
      if (OP == 1) { v[k] = vmax32(v[k], c + k); w[k] = imad(w[k], b, c); }
      if (OP == 2) { v[k] = vmax32(v[k], c + k); w[k] = add3(w[k], b, c); }
      if (OP == 3) { v[k] = vmax32(v[k], c + k); w[k] = prmt(w[k], b); }
      if (OP == 4) { v[k] = vmaxu2(v[k], c + k); }
      if (OP == 5) { v[k] = vmax32(v[k], c + k); w[k] = vmax3(w[k], b, c); }
      if (OP == 6) { w[k] = add3(w[k], b, c); }
      if (OP == 7) { w[k] = add3(w[k], b, c); x[k] = imad(x[k], b, c); }
      if (OP == 8) {  // proposed packed K1 cell-pair: PRMT, IADD3, 5 VIMNMX, 3 IMAD
        unsigned s = prmt(w[k], b);
        unsigned e = imad(x[k], 1u, 0xfffefffeu);
        e = vmaxu2(e, v[k]);
        unsigned f = imad(w[k], 1u, 0xfffefffeu);
        f = vmaxu2(f, x[k]);
        unsigned d = add3(v[k], s, c);
        unsigned h = vmaxu2(vmaxu2(d, e), f);
        h = vmaxu2(h, b);
        x[k] = e; w[k] = f ^ s; v[k] = imad(h, 1u, 0xfff0fff0u);
      }
      if (OP == 9) { v[k] = vmaxu2(v[k], c + k); w[k] = imad(w[k], b, c); }
      if (OP == 10) { v[k] = vmax32(v[k], c + k); x[k] = vmax32(x[k], b + k); w[k] = imad(w[k], b, c); }
    }
  }
  long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) acc ^= v[k] ^ w[k] ^ x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int OP>
void run(const char *name, int sms, double ninstr) {
  int blocks = sms * 4, threads = 512;
  unsigned *out; long long *cyc;
  cudaMalloc(&out, blocks * threads * 4); cudaMalloc(&cyc, blocks * 8);
  bench<OP><<<blocks, threads>>>(out, 1, cyc);
  bench<OP><<<blocks, threads>>>(out, 2, cyc);
  cudaDeviceSynchronize();
  long long h[4096]; cudaMemcpy(h, cyc, blocks * 8, cudaMemcpyDeviceToHost);
  double mc = 0; for (int i = 0; i < blocks; ++i) mc = h[i] > mc ? h[i] : mc;
  double iters = (double)blocks * threads * ILP * ITERS / 32.0;  // warp-iterations
  double per_smsp = iters / (sms * 4.0) ;
  printf("%-34s %6.2f cycles/iter/SMSP  (%.2f warp-instr/clk/SMSP for %.0f instrs)\n", name,
         mc / per_smsp, ninstr * per_smsp / mc, ninstr);
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  run<0>("vimnmx.s32", sms, 1);
  run<1>("vimnmx.s32 + imad", sms, 2);
  run<2>("vimnmx.s32 + iadd3", sms, 2);
  run<3>("vimnmx.s32 + prmt", sms, 2);
  run<4>("vimnmx.u16x2", sms, 1);
  run<5>("vimnmx.s32 + vimnmx3", sms, 2);
  run<6>("iadd3", sms, 1);
  run<7>("iadd3 + imad", sms, 2);
  run<8>("packed cell-pair mix (10 instr)", sms, 10);
  run<9>("vimnmx.u16x2 + imad", sms, 2);
  run<10>("2 vimnmx + imad", sms, 3);
  return 0;
}
