// Micro-benchmark 3: which pipe takes packed 16-bit maxima?  Candidates for
// moving maxima off the integer ALU pipe: HMNMX2 (max.f16x2 / max.bf16x2 on
// biased u16 bit patterns: for finite positive normals the float order equals
// the integer order) and FMNMX, mixed with VIMNMX.U16x2 / VIADDMNMX.U16x2 / IMAD.
#include <cstdio>
#include <cuda_runtime.h>
#define ILP 8
#define ITERS 2048
__device__ __forceinline__ unsigned vmaxu2(unsigned a, unsigned b) { unsigned d; asm volatile("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned hmax2(unsigned a, unsigned b) { unsigned d; asm volatile("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned bmax2(unsigned a, unsigned b) { unsigned d; asm volatile("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned fmax1(unsigned a, unsigned b) { unsigned d; asm volatile("max.f32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned imad(unsigned a, unsigned b, unsigned c) { unsigned d; asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ unsigned vadmx(unsigned a, unsigned b, unsigned c) { unsigned d; asm volatile("{.reg .b32 t; add.u16x2 t, %1, %2; max.u16x2 %0, t, %3;}" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ unsigned hadd2(unsigned a, unsigned b) { unsigned d; asm volatile("add.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned prmt(unsigned a, unsigned b) { unsigned d; asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned vmax3u2(unsigned a, unsigned b, unsigned c) { return __vimax3_u16x2(a, b, c); }

template <int OP>
__global__ void bench(unsigned *out, unsigned seed, long long *cyc) {
  unsigned v[ILP], w[ILP], x[ILP];
  unsigned b = (seed * 3u + 1u) & 0x3fff3fffu, c = (seed + 7u) & 0x3fff3fffu;
#pragma unroll
  for (int k = 0; k < ILP; ++k) { v[k] = (seed ^ (threadIdx.x + k)) & 0x3fff3fffu | 0x04000400u; w[k] = v[k] ^ 0x70007u; x[k] = v[k] ^ 0x55u; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      if (OP == 0) { v[k] = hmax2(v[k], c + k); }
      if (OP == 1) { v[k] = hmax2(v[k], c + k); w[k] = vmaxu2(w[k], b + k); }
      if (OP == 2) { v[k] = hmax2(v[k], c + k); w[k] = vadmx(w[k], b, c); }
      if (OP == 3) { v[k] = bmax2(v[k], c + k); }
      if (OP == 4) { v[k] = bmax2(v[k], c + k); w[k] = vmaxu2(w[k], b + k); }
      if (OP == 5) { v[k] = fmax1(v[k], c + k); }
      if (OP == 6) { v[k] = fmax1(v[k], c + k); w[k] = vmaxu2(w[k], b + k); }
      if (OP == 7) { v[k] = hmax2(v[k], c + k); w[k] = imad(w[k], b, c); }
      if (OP == 8) { v[k] = vadmx(v[k], b, c); }
      if (OP == 9) { v[k] = vadmx(v[k], b, c); w[k] = imad(w[k], b, c); }
      if (OP == 10) { v[k] = hadd2(v[k], c + k); }
      if (OP == 11) { v[k] = vmaxu2(v[k], c + k); w[k] = hmax2(w[k], b + k); x[k] = imad(x[k], b, c); }
      if (OP == 12) { v[k] = vadmx(v[k], b, c); w[k] = hmax2(w[k], b + k); x[k] = imad(x[k], b, c); }
      if (OP == 13) {  // current packed cell pair (8 instr): PRMT, 3 VIADDMNMX, IMAD, VIMNMX3, IMAD, VIMNMX
        unsigned u = prmt(w[k], b);
        unsigned e = vadmx(x[k], c, v[k]);
        unsigned t = vmax3u2(v[k] + u, e, b);
        unsigned g = vadmx(w[k], c, t);
        unsigned h = vadmx(g, b, t);
        x[k] = e; w[k] = g ^ u; v[k] = imad(h, 1u, c);
        v[k] = vmaxu2(v[k], h);
      }
      if (OP == 14) {  // same with h and rowmax on HMNMX2, t's 3-way max split
        unsigned u = prmt(w[k], b);
        unsigned e = vadmx(x[k], c, v[k]);
        unsigned t = hmax2(vmaxu2(v[k] + u, e), b);
        unsigned g = vadmx(w[k], c, t);
        unsigned h = hmax2(g + b, t);
        x[k] = e; w[k] = g ^ u; v[k] = imad(h, 1u, c);
        v[k] = hmax2(v[k], h);
      }
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
  double iters = (double)blocks * threads * ILP * ITERS / 32.0;
  double per_smsp = iters / (sms * 4.0);
  printf("%-44s %6.2f cycles/iter/SMSP  (%.2f warp-instr/clk/SMSP for %.0f instrs)\n", name,
         mc / per_smsp, ninstr * per_smsp / mc, ninstr);
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  run<0>("hmnmx2 (max.f16x2)", sms, 1);
  run<1>("hmnmx2 + vimnmx.u16x2", sms, 2);
  run<2>("hmnmx2 + viaddmnmx.u16x2", sms, 2);
  run<3>("max.bf16x2", sms, 1);
  run<4>("max.bf16x2 + vimnmx.u16x2", sms, 2);
  run<5>("fmnmx", sms, 1);
  run<6>("fmnmx + vimnmx.u16x2", sms, 2);
  run<7>("hmnmx2 + imad", sms, 2);
  run<8>("viaddmnmx.u16x2", sms, 1);
  run<9>("viaddmnmx.u16x2 + imad", sms, 2);
  run<10>("add.u16x2", sms, 1);
  run<11>("vimnmx.u16x2 + hmnmx2 + imad", sms, 3);
  run<12>("viaddmnmx.u16x2 + hmnmx2 + imad", sms, 3);
  run<13>("packed cell pair, current (8 instr + 1 add)", sms, 9);
  run<14>("packed cell pair, HMNMX2 for h/rm/floor", sms, 10);
  return 0;
}
