// sw_kmer.cuh -- candidate discovery feeding the aligner.
//
// The reference finds candidate pairs as the overlap-semiring product A*A^T
// of the sequence-by-k-mer matrix (kmer.py:56-126) -- entry (i, j) counts the
// DISTINCT k-mers sequences i and j share -- computed as a blocked 2D sparse
// SUMMA with symmetry pruning (summa.py, balance.py) and filtered by
// count >= min_shared_kmers with orientation (min, max) (pipeline.py:290-303).
// Blocking and pruning only decide which block emits each unordered pair
// once, so the candidate set is: all i < j with >= min_shared distinct shared
// k-mers.  Here it is computed as sorts instead of a sparse product:
//   1. k_kmer_keys: key = code << seq_bits | seq for every k-mer occurrence
//      (code = base-25, first residue most significant: kmer.py:43-53);
//   2. radix sort + unique -> one key per distinct (code, seq);
//   3. run-length encode the codes -> buckets of sequences sharing a code;
//   4. k_bucket_pairs: every bucket of c sequences emits its c(c-1)/2 pairs
//      (i < j: the bucket is sorted by seq) as i << seq_bits | j;
//   5. radix sort + run-length encode the pair keys -> shared count per pair.
// Integer work only, HBM/sort bound.
#pragma once
#include <cstdint>

namespace pastis {

// Step 1: one warp per sequence (grid-stride), lanes over positions.  `lut`
// maps residue bytes to alphabet indices (unknown -> X = 22, align.py:27-30).
__global__ void k_kmer_keys(const uint8_t *__restrict__ arena, const uint64_t *__restrict__ seq_off,
                            const uint32_t *__restrict__ seq_len,
                            const uint64_t *__restrict__ pos_base, uint32_t n_seqs, int k,
                            int seq_bits, const uint8_t *__restrict__ lut, uint64_t *__restrict__ keys) {
  __shared__ uint8_t slut[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) slut[i] = lut[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t s = warp0; s < n_seqs; s += nwarps) {
    const uint32_t len = seq_len[s];
    if (len < (uint32_t)k) continue;
    const uint8_t *p = arena + seq_off[s];
    uint64_t *out = keys + pos_base[s];
    for (uint32_t pos = lane; pos + k <= len; pos += 32) {
      uint64_t code = 0;
      for (int t = 0; t < k; ++t) code = code * 25u + slut[p[pos + t]];
      out[pos] = (code << seq_bits) | s;
    }
  }
}

// Step 4: one warp per bucket (grid-stride).  `members` are the distinct
// (code, seq) keys sorted ascending; bucket r covers members[start[r],
// start[r] + count[r]); its pairs go to pairs[emit_off[r] ...].
__global__ void k_bucket_pairs(const uint64_t *__restrict__ members, const uint32_t *__restrict__ count,
                               const uint64_t *__restrict__ start,
                               const uint64_t *__restrict__ emit_off, uint64_t n_buckets,
                               int seq_bits, uint64_t *__restrict__ pairs) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t mask = (1ull << seq_bits) - 1;
  for (uint64_t r = warp0; r < n_buckets; r += nwarps) {
    const uint32_t c = count[r];
    if (c < 2) continue;
    const uint64_t *m = members + start[r];
    uint64_t *out = pairs + emit_off[r];
    // row a emits (a, b) for b in (a, c): offset of row a = a*c - a(a+1)/2
    for (uint32_t a = 0; a + 1 < c; ++a) {
      const uint64_t sa = m[a] & mask;
      const uint64_t row = (uint64_t)a * c - (uint64_t)a * (a + 1) / 2;
      for (uint32_t b = a + 1 + lane; b < c; b += 32)
        out[row + (b - a - 1)] = (sa << seq_bits) | (m[b] & mask);
    }
  }
}

struct KeyShift {   // (code << seq_bits | seq) -> code
  int bits;
  __host__ __device__ uint64_t operator()(uint64_t x) const { return x >> bits; }
};

struct PairsOf {    // bucket size c -> c(c-1)/2
  __host__ __device__ uint64_t operator()(uint32_t c) const { return (uint64_t)c * (c - 1) / 2; }
};

struct CountAtLeast {
  uint32_t t;
  __host__ __device__ bool operator()(uint32_t c) const { return c >= t; }
};

// Candidate records: pair key + count -> (i, j, count)
__global__ void k_write_candidates(const uint64_t *__restrict__ pair_keys,
                                   const uint32_t *__restrict__ counts, uint64_t n, int seq_bits,
                                   uint32_t min_shared, uint64_t *__restrict__ cursor,
                                   sw_candidate_t *__restrict__ out) {
  const uint64_t mask = (1ull << seq_bits) - 1;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = counts[t];
    if (c < min_shared) continue;
    // order-preserving compaction is done by the caller's exclusive scan
    const uint64_t pos = cursor[t];
    sw_candidate_t r;
    r.i = (uint32_t)(pair_keys[t] >> seq_bits);
    r.j = (uint32_t)(pair_keys[t] & mask);
    r.count = c;
    r.pad = 0;
    out[pos] = r;
  }
}

}  // namespace pastis
