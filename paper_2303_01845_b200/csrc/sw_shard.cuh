// sw_shard.cuh -- cell-balanced sharding of a pair batch over GPUs, planned
// on the device.
//
// Replaces the reference's lane split (AlignEngine, align.py:299-335: a
// contiguous ceil split of the pair list over worker processes, _chunk
// align.py:265-269, with no balancing).  Every shard sees the same batch and
// computes the same plan independently (no communication):
//   1. sort the pairs by cells = |a|*|b| descending (a stable radix sort of
//      32-bit keys ~cells -- |a|, |b| <= 65,000 so cells < 2^32; ties keep
//      input order, so the order is identical on every device);
//   2. deal them out in a snake: sorted position p = r*N + q goes to shard
//      q in even rounds r and to shard N-1-q in odd rounds.  Shard s owns
//      exactly one position per round, so its r-th pair is found directly
//      (no compaction), and every shard's load is within one pair's cells of
//      every other's while each shard also gets the same mix of shapes;
//   3. gather the shard's sequence bytes into a local arena (warp per pair,
//      128-bit loads of the source), reading the source arena wherever it
//      lives -- device memory, or pinned host memory over PCIe (zero-copy:
//      only this shard's bytes cross the link).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/pastis_sw.h"

namespace pastis {

// sorted positions shard s of N owns out of n
__host__ __device__ inline uint64_t shard_count(uint64_t n, int N, int s) {
  const uint64_t full = n / (uint64_t)N, rem = n % (uint64_t)N;
  const uint64_t q = (full % 2 == 0) ? (uint64_t)s : (uint64_t)(N - 1 - s);
  return full + (q < rem ? 1 : 0);
}
__host__ __device__ inline uint64_t shard_position(uint64_t r, int N, int s) {
  return r * (uint64_t)N + ((r % 2 == 0) ? (uint64_t)s : (uint64_t)(N - 1 - s));
}

__global__ void k_shard_keys(const sw_pair_t *__restrict__ pairs, uint64_t n, uint32_t *keys,
                             uint32_t *vals) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const sw_pair_t p = pairs[k];
  // lengths beyond 65,000 are rejected later (k_classify); clamp so the key
  // stays a 32-bit cell count either way
  const uint64_t c = (uint64_t)min(p.a_len, 65535u) * (uint64_t)min(p.b_len, 65535u);
  keys[k] = ~(uint32_t)c;
  vals[k] = (uint32_t)k;
}

__global__ void k_shard_select(const uint32_t *__restrict__ sorted_vals,
                               const sw_pair_t *__restrict__ pairs, int N, int s, uint64_t nl,
                               sw_pair_t *lpairs, uint32_t *lidx, uint64_t *llen) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nl) return;
  const uint32_t g = sorted_vals[shard_position(r, N, s)];
  const sw_pair_t p = pairs[g];
  lidx[r] = g;
  lpairs[r] = p;
  llen[r] = (uint64_t)p.a_len + p.b_len;
}

// copy src[off, off + len) to dst[o, o + len): one warp, 16-byte aligned
// loads (aligned on the absolute address: the over-read before the first and
// after the last byte stays inside the same 16-byte word, hence the same
// page), byte stores
__device__ __forceinline__ void warp_copy(const uint8_t *__restrict__ src, uint64_t off,
                                          uint32_t len, uint8_t *__restrict__ dst, uint64_t o,
                                          int lane) {
  if (len == 0) return;
  const uintptr_t a0 = (uintptr_t)(src + off), a1 = a0 + len;
  for (uintptr_t w = (a0 & ~(uintptr_t)15) + 16u * lane; w < a1; w += 16u * 32) {
    const uint4 v = *reinterpret_cast<const uint4 *>(w);
    const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      const uintptr_t pos = w + b;
      if (pos >= a0 && pos < a1) dst[o + (pos - a0)] = (uint8_t)(x[b >> 2] >> (8 * (b & 3)));
    }
  }
}

// warp per local pair: gather its a and b bytes into the local arena at
// loff[r] (exclusive scan of llen) and point the local pair at them.  A pair
// reaching outside the source arena is left pointing outside the local one,
// so the planning kernel rejects it (SW_EINVAL), as for any call.
__global__ void k_shard_gather(const uint8_t *__restrict__ src, uint64_t src_bytes,
                               sw_pair_t *lpairs, const uint64_t *__restrict__ loff, uint64_t nl,
                               uint8_t *__restrict__ dst, uint64_t dst_bytes) {
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < nl; r += nwarps) {
    const sw_pair_t p = lpairs[r];
    const uint64_t o = loff[r];
    const bool ok = p.a_off <= src_bytes && p.a_len <= src_bytes - p.a_off &&
                    p.b_off <= src_bytes && p.b_len <= src_bytes - p.b_off;
    if (ok) {
      warp_copy(src, p.a_off, p.a_len, dst, o, lane);
      warp_copy(src, p.b_off, p.b_len, dst, o + p.a_len, lane);
    }
    if (lane == 0) {
      sw_pair_t q = p;
      q.a_off = ok ? o : dst_bytes + 1;
      q.b_off = ok ? o + p.a_len : dst_bytes + 1;
      lpairs[r] = q;
    }
  }
}

// results of the shard back to input order: out[lidx[r]] = lout[r]
__global__ void k_shard_scatter(const sw_result_t *__restrict__ lout, const uint32_t *__restrict__ lidx,
                                uint64_t nl, sw_result_t *out) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nl) out[lidx[r]] = lout[r];
}

}  // namespace pastis
