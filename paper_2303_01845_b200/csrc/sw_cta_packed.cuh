// sw_cta_packed.cuh -- K1cp: TWO long pairs per CTA in biased u16x2 lanes.
//
// The forward pass of long pairs (>= 4 strips): the arithmetic of the packed
// forward (k_score_packed, sw_packed.cuh: pair A in the low halves, pair B in
// the high halves, 4 adds + VIMNMX3 + 4 maxes per row-word) with the strips of
// the duo spread over the kCtaWarps warps of a CTA as in k_score_cta: warp w
// computes strips w, w + W, ...  The bottom row of every strip goes to an
// 8-slot ring of rows in global memory (L2-resident) with per-warp progress
// counters in shared memory; a slot is rewritten 8 strips later, by which
// time the strip reading it has finished, so producers never wait.
//
// Output per pair: best and i_end (first row whose running maximum reaches
// best, from the per-row maxima as in k_score_packed).  j_end needs the H
// values of row i_end: each warp saves, for every strip it computes, the
// strip's top boundary row (both pairs, into a per-warp candidate slot in the
// pool) and keeps it when the strip strictly improves the warp's best.  The
// winning warp's slot holds the row above the strip containing i_end, and
// k_jend replays that strip (<= 256 rows, 1/nstrips of the work) exactly.
// Overflow (biased value near 65535) sends both pairs to the wide path; no
// pool room for the slots sends them to the scalar CTA kernel.
#pragma once
#include "sw_packed.cuh"
#include "sw_cta.cuh"

namespace pastis {

constexpr int kCtaPR = 8;              // rows per lane: 256-row strips
constexpr int kCtaPSlots = 8;          // ring of strip bottom rows per CTA
constexpr int kCtaPRowStride = 65064;  // uint2 entries per ring row (>= 65000 columns)

struct CtaPSync {
  volatile int prod[kCtaWarps];                 // cumulative bottom-row columns published
  int64_t item[2];
  unsigned long long slot_off[2];               // pool offset of each pair's 2 x kCtaWarps slots
  unsigned long long key[2][kCtaWarps];         // (best << 32) | (0xFFFF - row) << 16
  uint32_t vmax[kCtaWarps];
  int bidx[2][kCtaWarps];                       // which of the warp's 2 slots holds its best strip's top
};

__host__ __device__ constexpr int cta_packed_warp_bytes(int R) {
  return 2 * prof_bytes_p(R) + 2 * kRingSlot + kBndBytes;   // profiles, mirrored rings, row above
}
__host__ __device__ constexpr int smem_cta_packed(int R) {
  return kMatTBytes + kCtaWarps * cta_packed_warp_bytes(R) + (int)sizeof(CtaPSync) + 16;
}

template <int R>
#ifndef K1CP_MINB
#define K1CP_MINB 4   // 126 registers, 4 blocks of 4 warps (config 5 forward +0.6 % over 3 blocks at 166)
#endif
__global__ void __launch_bounds__(kCtaWarps * 32, K1CP_MINB)
k_score_cta_packed(KArgs A, int stage, int cls) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t *smatT = smem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t *profA = smem + kMatTBytes + warp * cta_packed_warp_bytes(R);
  uint8_t *profB = profA + prof_bytes_p(R);
  uint8_t *ringA = profB + prof_bytes_p(R);
  uint8_t *ringB = ringA + kRingSlot;
  uint2 *bnd = reinterpret_cast<uint2 *>(ringB + kRingSlot);   // 32 columns of the row above
  CtaPSync &S = *reinterpret_cast<CtaPSync *>(smem + kMatTBytes + kCtaWarps * cta_packed_warp_bytes(R));
  load_matrix_t(smatT, A.mat, A.prof_lo);
  uint2 *rows_ring = A.cta_rows + (uint64_t)blockIdx.x * kCtaPSlots * kCtaPRowStride;
  const uint32_t Bs = (uint32_t)A.bias16;
  const uint32_t BB = A.p_bb, OPEN2 = A.p_open2;
  const uint32_t NEG2 = A.p_ext2, HO0 = A.p_ho0, NEXT2 = A.p_next2, NOPEN2 = A.p_nopen2;
  for (;;) {
    if (threadIdx.x == 0) {
      const uint32_t pos = atomicAdd(&A.ctrs[kStages * kNumClasses + stage * kNumClasses + cls], 2u);
      const uint32_t cnt = *(volatile uint32_t *)&A.ctrs[stage * kNumClasses + cls];
      for (int h = 0; h < 2; ++h) {
        S.item[h] = pos + h < cnt ? (int64_t)list_of(A, stage, cls)[pos + h] : -1;
        S.slot_off[h] = ~0ull;
        if (S.item[h] >= 0) {
          const uint64_t bytes = ((uint64_t)2 * kCtaWarps * A.pairs[S.item[h]].b_len * 4 + 15) & ~15ull;
          const unsigned long long off = atomicAdd(A.pool_top, (unsigned long long)bytes);
          if (off + bytes <= A.pool_cap) S.slot_off[h] = off;
        }
      }
      for (int w = 0; w < kCtaWarps; ++w) S.prod[w] = 0;
    }
    __syncthreads();
    const int64_t k0 = S.item[0], k1 = S.item[1];
    if (k0 < 0) break;
    if (S.slot_off[0] == ~0ull || (k1 >= 0 && S.slot_off[1] == ~0ull)) {
      // no pool room for the boundary slots: the scalar one-CTA-per-pair path
      if (threadIdx.x == 0) {
        A.st[k0].flags = 0;
        list_push(A, 0, kCtaScalarClass, (uint32_t)k0);
        if (k1 >= 0) {
          A.st[k1].flags = 0;
          list_push(A, 0, kCtaScalarClass, (uint32_t)k1);
        }
      }
      __syncthreads();
      continue;
    }
    const sw_pair_t p0 = A.pairs[k0];
    sw_pair_t p1;
    p1.a_off = p1.b_off = 0;
    p1.a_len = p1.b_len = 0;
    if (k1 >= 0) p1 = A.pairs[k1];
    const int m0 = (int)p0.a_len, n0 = (int)p0.b_len, m1 = (int)p1.a_len, n1 = (int)p1.b_len;
    const RawView rows0{A.codes + p0.a_off, nullptr}, cols0{A.codes + p0.b_off, nullptr};
    const RawView rows1{A.codes + p1.a_off, nullptr}, cols1{A.codes + p1.b_off, nullptr};
    const int m = max(m0, m1), n = max(n0, n1);
    const int nstrips = (m + 32 * R - 1) / (32 * R);
    uint32_t *slot0 = reinterpret_cast<uint32_t *>(A.pool + S.slot_off[0]);
    uint32_t *slot1 = k1 >= 0 ? reinterpret_cast<uint32_t *>(A.pool + S.slot_off[1]) : nullptr;
    unsigned long long keyA = 0ull, keyB = 0ull;   // this warp's running best (first row)
    int bidxA = 0, bidxB = 0;                      // slot of the warp's best strip's top row
    uint32_t vmax2 = 0u;
    for (int strip = warp; strip < nstrips; strip += kCtaWarps) {
      const int row0 = strip * 32 * R;
      __syncwarp();
      build_profile_u8<R>(profA, smatT, rows0, m0, row0, lane);
      build_profile_u8<R>(profB, smatT, rows1, m1, row0, lane);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = -32 + 32 * q + lane;
        const uint8_t va = (c >= 0 && c < n0) ? (uint8_t)cols0.at(c) : (uint8_t)kPad;
        const uint8_t vb = (c >= 0 && c < n1) ? (uint8_t)cols1.at(c) : (uint8_t)kPad;
        ringA[c & 127] = va;
        ringB[c & 127] = vb;
        if ((c & 127) < 8) { ringA[(c & 127) + 128] = va; ringB[(c & 127) + 128] = vb; }
      }
      int nxtA = 96 + lane < n0 ? cols0.at(96 + lane) : kPad;   // next refill, loaded ahead
      int nxtB = 96 + lane < n1 ? cols1.at(96 + lane) : kPad;
      __syncwarp();
      PackedLane<R> L;
#pragma unroll
      for (int r = 0; r < R; ++r) { L.Ho[r] = HO0; L.E[r] = NEG2; L.rm[r] = BB; }
      L.hoUpPrev = HO0;
      L.botHo = HO0;
      L.botF = NEG2;
      const bool has_above = strip > 0, has_below = strip + 1 < nstrips;
      const uint2 *in_row = rows_ring + (uint64_t)((strip - 1) & (kCtaPSlots - 1)) * kCtaPRowStride;
      uint2 *out_row = rows_ring + (uint64_t)(strip & (kCtaPSlots - 1)) * kCtaPRowStride;
      const int in_w = (strip + kCtaWarps - 1) & (kCtaWarps - 1);
      const int in_base = has_above ? ((strip - 1) / kCtaWarps) * n : 0;
      const int out_base = (strip / kCtaWarps) * n;
      // this strip's top row is saved into the warp's candidate slot as it
      // is read (per pair: (H-open, F) biased u16 of that pair's half)
      uint32_t *candA = slot0 + (uint64_t)(warp * 2 + (bidxA ^ 1)) * n0;
      uint32_t *candB = slot1 ? slot1 + (uint64_t)(warp * 2 + (bidxB ^ 1)) * n1 : nullptr;
      uint2 cur = make_uint2(HO0, NEG2);
      const int steps = n + 31;
      for (int s0 = 0; s0 < steps; s0 += kScoreUnroll) {
        if ((s0 & 31) == 0) {
          if (s0 > 0) {    // refill column-code ring slots for columns s0+64 .. s0+95
            const int c = s0 + 64 + lane;
            ringA[c & 127] = (uint8_t)nxtA;
            ringB[c & 127] = (uint8_t)nxtB;
            if ((c & 127) < 8) { ringA[(c & 127) + 128] = (uint8_t)nxtA; ringB[(c & 127) + 128] = (uint8_t)nxtB; }
            nxtA = c + 32 < n0 ? cols0.at(c + 32) : kPad;
            nxtB = c + 32 < n1 ? cols1.at(c + 32) : kPad;
          }
          if (has_above && s0 < n) {
            const int need = min(s0 + 32, n);
            while (S.prod[in_w] < in_base + need) __nanosleep(32);
            __syncwarp();
            const int c = s0 + lane;
            cur = make_uint2(HO0, NEG2);
            if (c < n) {
              cur = __ldcg(in_row + c);
              if (c < n0) candA[c] = prmt(cur.x, cur.y, 0x5410u);
              if (candB && c < n1) candB[c] = prmt(cur.x, cur.y, 0x7632u);
            }
          }
          __syncwarp();
          bnd[lane] = cur;   // lane 0 reads column s from shared memory (one LDS, no shuffles)
          __syncwarp();
        }
        const int rbase = (s0 - lane) & 127;   // ring slot of this lane's column at step s0
        uint2 rowv[kScoreUnroll];
#pragma unroll
        for (int q = 0; q < kScoreUnroll; ++q) {
          const int s = s0 + q;
          const uint4 pa = load_profile_u8<R>(profA, ringA[rbase + q], lane);
          const uint4 pb = load_profile_u8<R>(profB, ringB[rbase + q], lane);
          const uint2 tv = bnd[s & 31];
          const uint32_t upHo = shfl_up_or(L.botHo, tv.x);
          const uint32_t upF = shfl_up_or(L.botF, tv.y);
          uint32_t diag = L.hoUpPrev;
          L.hoUpPrev = upHo;
          uint32_t G = upF + OPEN2, tprev = upHo + OPEN2;   // G = F + open (sw_packed.cuh)
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const uint32_t u2 = prmt(word_of(pa, r), word_of(pb, r), sel_pair(r & 3));
            L.E[r] = __viaddmax_u16x2(L.E[r], NEXT2, L.Ho[r]);
            const uint32_t t = vmax2u(vmax2u(diag + u2, L.E[r]), BB);
            G = __viaddmax_u16x2(G, NEXT2, tprev);
            const uint32_t h = __viaddmax_u16x2(G, NOPEN2, t);
            diag = L.Ho[r];
            L.Ho[r] = h - OPEN2;
            tprev = t;
            L.rm[r] = vmax2u(L.rm[r], h);
          }
          L.botHo = L.Ho[R - 1];
          L.botF = G - OPEN2;
          rowv[q] = make_uint2(L.botHo, L.botF);
        }
        if (has_below && lane == 31) {   // the chunk's bottom row, columns s0-31 .. s0-24
#pragma unroll
          for (int q = 0; q < kScoreUnroll; ++q) {
            const int cb = s0 + q - 31;
            if (cb >= 0 && cb < n) out_row[cb] = rowv[q];
          }
        }
        if (has_below) {
          __threadfence_block();
          if (lane == 31) S.prod[warp] = out_base + min(max(s0 + kScoreUnroll - 31, 0), n);
        }
      }
      // per-pair strip best (first row reaching it)
      unsigned long long kA = 0ull, kB = 0ull;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int x = row0 + lane * R + r;
        const uint32_t va = L.rm[r] & 0xFFFFu, vb = L.rm[r] >> 16;
        vmax2 = max(vmax2, max(va, vb));
        if (x < m0) {
          const unsigned long long kk = ((unsigned long long)(va - Bs) << 32) |
                                        ((unsigned long long)(0xFFFF - x) << 16);
          kA = kk > kA ? kk : kA;
        }
        if (x < m1) {
          const unsigned long long kk = ((unsigned long long)(vb - Bs) << 32) |
                                        ((unsigned long long)(0xFFFF - x) << 16);
          kB = kk > kB ? kk : kB;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a2 = __shfl_xor_sync(0xffffffffu, kA, o);
        kA = a2 > kA ? a2 : kA;
        const unsigned long long b2 = __shfl_xor_sync(0xffffffffu, kB, o);
        kB = b2 > kB ? b2 : kB;
      }
      // a strict improvement keeps this strip's top row (the candidate slot)
      if ((kA >> 32) > (keyA >> 32)) { keyA = kA; bidxA ^= 1; }
      if ((kB >> 32) > (keyB >> 32)) { keyB = kB; bidxB ^= 1; }
      if (has_below) {
        __threadfence_block();
        if (lane == 31) S.prod[warp] = out_base + n;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vmax2 = max(vmax2, (uint32_t)__shfl_xor_sync(0xffffffffu, vmax2, o));
    if (lane == 0) {
      S.key[0][warp] = keyA;
      S.key[1][warp] = keyB;
      S.bidx[0][warp] = bidxA;
      S.bidx[1][warp] = bidxB;
      S.vmax[warp] = vmax2;
    }
    __threadfence_block();
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t vm = 0u;
      for (int w = 0; w < kCtaWarps; ++w) vm = max(vm, S.vmax[w]);
      const bool overflow = vm > kPackedLimit;
      for (int h = 0; h < 2; ++h) {
        const int64_t kk = h ? k1 : k0;
        if (kk < 0) continue;
        PairState *st = A.st + kk;
        int ww = 0;
        unsigned long long best_key = 0ull;
        for (int w = 0; w < kCtaWarps; ++w)
          if (S.key[h][w] > best_key) { best_key = S.key[h][w]; ww = w; }
        const int32_t best = (int32_t)(best_key >> 32);
        const int32_t i_end = 0xFFFF - (int32_t)((best_key >> 16) & 0xFFFF);
        st->i0 = 0;
        st->j0 = 0;
        if (overflow) {
          st->flags = kFlagWide;
          list_push(A, 3, 0, (uint32_t)kk);
        } else if (best == 0) {
          st->best = 0;
          st->i_end = -1;
          st->j_end = -1;
          st->flags = 0;
        } else {
          const int nh = h ? n1 : n0;
          st->best = best;
          st->i_end = i_end;
          st->j_end = -1;
          st->flags = 0;
          st->code_off = S.slot_off[h] + (uint64_t)(ww * 2 + S.bidx[h][ww]) * nh * 4;
          list_push(A, 9, 0, (uint32_t)kk);
        }
      }
    }
    __syncthreads();
  }
}

// j_end of a pair from K1cp: replay the (<= 256-row) strip that holds i_end
// from the saved row above it (unscaled int32, so any packed-path score is
// exact) and take the first column of row i_end reaching best -- the
// row-major-first end cell of align.py:124.  Then queue the reverse pass (or,
// for homologs, the prefix box) like the forward kernels do.
template <int R>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_jend(KArgs A, int stage, int cls) {
  extern __shared__ __align__(16) uint8_t smem[];
  int8_t *smat = reinterpret_cast<int8_t *>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t *prof = smem + kMatBytes + warp * kProfBytes;
  load_matrix(smat, A.mat);
  const uint64_t gwarp = (uint64_t)blockIdx.x * kWarpsPerBlock + warp;
  int2 *bnd = A.bnd + gwarp * A.bnd_stride;
  const int32_t Bs = A.bias16;
  for (;;) {
    const int64_t k = next_item(A, stage, cls, lane);
    if (k < 0) break;
    const sw_pair_t p = A.pairs[k];
    PairState *st = A.st + k;
    const int32_t best = st->best, i_end = st->i_end;
    const int n = (int)p.b_len;
    const int strip = i_end / (32 * kCtaPR);
    const int row0 = strip * 32 * kCtaPR;
    if (strip > 0) {
      const uint32_t *slot = reinterpret_cast<const uint32_t *>(A.pool + st->code_off);
      for (int c = lane; c < n; c += 32) {
        const uint32_t w = slot[c];
        bnd[c] = make_int2((int32_t)(w & 0xFFFFu) - Bs, (int32_t)(w >> 16) - Bs);
      }
    }
    __syncwarp();
    const View rows{A.codes + p.a_off + row0, 1}, cols{A.codes + p.b_off, 1};
    const ScoreOut o = score_pair<R, 0, true>(prof, smat, rows, cols, i_end - row0 + 1, n, A.open_,
                                              A.ext, best, bnd, lane, strip > 0);   // stops at best
    if (lane == 0) {
      const int32_t j_end = 65535 - (int32_t)(o.fwd & 0xFFFF);
      const int32_t got = (int32_t)(o.fwd >> 32);
      st->j_end = j_end;
      if (got != best) {
        // cannot happen for exact arithmetic; keep the pair visible as an error
        st->flags = kFlagDone;
        sw_result_t r;
        r.score = best; r.i_begin = -1; r.i_end = i_end; r.j_begin = -1; r.j_end = j_end;
        r.matches = 0; r.aln_len = 0; r.status = SW_STATUS_INTERNAL;
        A.out[k] = r;
      } else {
        const uint64_t area = (uint64_t)(i_end + 1) * (uint64_t)(j_end + 1);
        // homolog: box = prefix.  So is a pair whose score does not fit the
        // reverse pass's scaled int32 domain (best >= kScaledLimit: only the
        // u16x2 forward reaches it without the wide re-run); the box fill is
        // plain int32.
        if ((uint64_t)best * best * 8ull > 49ull * area || best >= kScaledLimit) {
          st->i0 = 0;
          st->j0 = 0;
          list_push(A, 2, class_of(i_end + 1), (uint32_t)k);
        } else {
          list_push(A, 1, long_class(i_end + 1), (uint32_t)k);
        }
      }
    }
  }
}

}  // namespace pastis
