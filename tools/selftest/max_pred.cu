// Probe: ptxas on sm_100a folds `h == f` after h = max(max(D,e),f) into the
// VIMNMX predicate output.  Check which formulations give correct results.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void k(const int *in, unsigned *out, int n) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  int D = in[3 * t], e = in[3 * t + 1], f = in[3 * t + 2];
  // A: intrinsic + equality
  int h = __vimax3_s32_relu(D, e, f);
  unsigned a = h == D ? 1u : (h == f ? 2u : 3u);
  a = h == 0 ? 0u : a;
  // B: plain max
  int h2 = max(max(max(D, e), f), 0);
  unsigned b = h2 == D ? 1u : (h2 == f ? 2u : 3u);
  b = h2 == 0 ? 0u : b;
  // C: explicit compares against the partial max
  int tt = __vimax_s32_relu(D, e);
  int h3 = max(tt, f);
  unsigned c = (D >= e && D >= f && D >= 0) ? 1u : ((f >= tt) ? 2u : 3u);
  c = h3 == 0 ? 0u : c;
  // D: xor equality
  unsigned d = ((h ^ D) == 0) ? 1u : (((h ^ f) == 0) ? 2u : 3u);
  d = h == 0 ? 0u : d;
  out[4 * t] = a; out[4 * t + 1] = b; out[4 * t + 2] = c; out[4 * t + 3] = d;
}
int main() {
  const int n = 1 << 20;
  int *h_in = (int *)malloc(n * 12);
  srand(1);
  for (int i = 0; i < 3 * n; ++i) h_in[i] = (rand() % 13) - 6;
  int *d_in; unsigned *d_out;
  cudaMalloc(&d_in, n * 12); cudaMalloc(&d_out, n * 16);
  cudaMemcpy(d_in, h_in, n * 12, cudaMemcpyHostToDevice);
  k<<<(n + 255) / 256, 256>>>(d_in, d_out, n);
  unsigned *h_out = (unsigned *)malloc(n * 16);
  cudaMemcpy(h_out, d_out, n * 16, cudaMemcpyDeviceToHost);
  int bad[4] = {0, 0, 0, 0};
  for (int t = 0; t < n; ++t) {
    int D = h_in[3 * t], e = h_in[3 * t + 1], f = h_in[3 * t + 2];
    int h = D; if (e > h) h = e; if (f > h) h = f; if (h < 0) h = 0;
    unsigned ref = h == 0 ? 0u : (h == D ? 1u : (h == f ? 2u : 3u));
    for (int v = 0; v < 4; ++v) bad[v] += h_out[4 * t + v] != ref;
  }
  printf("mismatches A(intrinsic)=%d B(plain)=%d C(partial)=%d D(xor)=%d of %d\n", bad[0], bad[1],
         bad[2], bad[3], n);
  return 0;
}
