// sw_packed.cuh -- K1p: the packed forward pass (two pairs per warp).
//
// Same recurrence and wavefront as k_score<FWD> (align.py:103-121), but each
// 32-bit register holds the same cell of TWO pairs (pair A in the low half,
// pair B in the high half) as biased unsigned 16-bit values v + B, with
// B = open + ext + 128 (the bias keeps both halves in [0, 65535], so full-word
// IMAD adds never borrow across halves).  Per row r of a lane (G = F + open):
//   E  = max(E - ext, Ho_left)          VIADDMNMX.U16x2 (per-half add wraps)
//   t  = max(Ho_diag + (s + open), E, B)  IMAD + VIMNMX3  (B = biased zero)
//   G  = max(G - ext, t[r-1])           VIADDMNMX.U16x2 (short F chain: t, not H)
//   h  = max(G - open, t)               VIADDMNMX.U16x2
//   Ho = h - open                       IMAD
//   rowmax = max(rowmax, h)             VIMNMX.U16x2
// plus one PRMT merging the two pairs' profile bytes = 8 issue slots per two
// cells.  A/B on the box (config 2, forward GCUPS): unfused IMAD+VIMNMX for E
// and F 2,597; fused E+F 2,848; + s+open profile (no IADD3) 2,982; + G form
// 3,044.  The profile stores u = s + open (0..127: BLOSUM-like matrices with
// min >= -open; other parameters take the scalar path), so D needs no constant.
// Per-row maxima give best and i_end (first row reaching best); j_end is found
// by the traceback kernel from per-window row maxima stored in the column
// checkpoints (k_tb).  Values are exact while every biased value stays below
// 65535 - 128; a warp that gets near that re-runs both pairs in the wide path.
#pragma once
#include "sw_kernels.cuh"

namespace pastis {

constexpr int kWarpsPerBlockP = 4;
#ifndef K1P_UNROLL
#define K1P_UNROLL 8
#endif
constexpr int kUnrollP = K1P_UNROLL;   // wavefront steps per unrolled chunk
#ifndef K1P_PROF_UNROLL
#define K1P_PROF_UNROLL 7
#endif
constexpr int kProfUnroll = K1P_PROF_UNROLL;   // code groups per profile-build iteration
constexpr int kRingBytes = 2 * 128;              // column-code rings of the two pairs (K1cp)
// K1p's rings: 128 slots + a mirror of slots 0..7, so the 8 steps of a chunk
// read slots base + q without wrapping
constexpr int kRingSlot = 136;
constexpr int kBndBytes = 32 * 8;                 // K1p: the row above, 32 columns of (Ho2, F2)
constexpr uint32_t kPackedLimit = 65535u - 160u;  // overflow guard on biased values
constexpr int32_t kTileMax = 32767;               // largest score k_tb's int16 tiles hold
// Profile table of the packed kernels: matT[a][code] = s(code, a) + open as
// u8 (a = row residue, code = column residue; PAD row/column -> 0), rows
// padded to 32 bytes so four codes load as one word.  kMatTBytes replaces
// kMatBytes at the front of the packed kernels' shared memory.
constexpr int kMatTStride = 32;
constexpr int kMatTBytes = kCodes * kMatTStride + 32;

// u8 profile of one pair: part 0 = [code][lane][P0] (P0 = 4 or 8 bytes),
// part 1 = [code][lane][P1] for the remaining rows (R = 10 -> 8 + 2 bytes,
// R = 6 -> 4 + 2).  Rows 4k..4k+3 live in word k of the loaded uint4.
__host__ __device__ constexpr int prof_p0(int R) { return R <= 6 ? 4 : 8; }
__host__ __device__ constexpr int prof_p1(int R) {
  return R <= 4 ? 0 : R <= 6 ? 2 : R <= 8 ? 0 : R <= 10 ? 2 : R <= 12 ? 4 : 8;
}
__host__ __device__ constexpr int prof_bytes_p(int R) { return kCodes * 32 * (prof_p0(R) + prof_p1(R)); }
__host__ __device__ constexpr int warp_bytes_p(int R) {
  return (2 * prof_bytes_p(R) + 2 * kRingSlot + kBndBytes + 15) / 16 * 16;
}
__host__ __device__ constexpr int smem_packed(int R) { return kMatTBytes + kWarpsPerBlockP * warp_bytes_p(R); }
// resident blocks per SM the packed forward is compiled for (registers):
// small R has little per-lane state, so more warps hide the latency
#ifndef K1P_MINB_SMALL
#define K1P_MINB_SMALL 6
#endif
#ifndef K1P_MINB_MID
#define K1P_MINB_MID 4
#endif
#ifndef K1P_R4MAX
#define K1P_R4MAX 8
#endif
__host__ __device__ constexpr int packed_min_blocks(int R) {
  // R = 7, 8: 128 registers and 55 KB of shared memory, 4 blocks per SM
  // (A/B on the box against 3: forward +1.5 % on config 3)
  return R <= 4 ? K1P_MINB_SMALL : R <= 6 ? K1P_MINB_MID : R <= K1P_R4MAX ? 4 : 3;
}

__device__ __forceinline__ uint32_t vmax2u(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t splat16(uint32_t v) { return (v & 0xFFFFu) * 0x10001u; }

__device__ __forceinline__ void load_matrix_t(uint8_t *matT, const int8_t *mat, int lo) {
  for (int i = threadIdx.x; i < kMatTBytes; i += blockDim.x) {
    const int a = i / kMatTStride, code = i % kMatTStride;
    int v = 0;
    if (a < kPad && code < kPad) v = (int)mat[code * kCodes + a] - lo;
    matT[i] = (uint8_t)v;
  }
  __syncthreads();
}

// u8 profile (s - lo) for rows row0+lane*R .. +R-1 of one pair; PAD -> 0.
// Four codes of one row come from one 32-bit LDS of matT; a 4x4 byte
// transpose (8 PRMT) turns four rows x four codes into the per-code words
// [rows 4j .. 4j+3] of the profile layout.
template <int R, typename V>
__device__ __forceinline__ void build_profile_u8(uint8_t *prof, const uint8_t *matT, const V &rows,
                                                 int m, int row0, int lane) {
  constexpr int P0 = prof_p0(R), P1 = prof_p1(R);
  constexpr int NW = (R + 3) / 4;          // profile words per code
  const uint8_t *rowp[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int x = row0 + lane * R + r;
    rowp[r] = matT + (x < m ? rows.at(x) : kPad) * kMatTStride;
  }
#pragma unroll kProfUnroll
  for (int g = 0; g < (kCodes + 3) / 4; ++g) {
    uint32_t W[4][NW];                      // W[k][j]: code 4g+k, rows 4j .. 4j+3
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      uint32_t v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        v[i] = 4 * j + i < R ? *reinterpret_cast<const uint32_t *>(rowp[4 * j + i] + 4 * g) : 0u;
      const uint32_t t01l = prmt(v[0], v[1], 0x5140u), t01h = prmt(v[0], v[1], 0x7362u);
      const uint32_t t23l = prmt(v[2], v[3], 0x5140u), t23h = prmt(v[2], v[3], 0x7362u);
      W[0][j] = prmt(t01l, t23l, 0x5410u);
      W[1][j] = prmt(t01l, t23l, 0x7632u);
      W[2][j] = prmt(t01h, t23h, 0x5410u);
      W[3][j] = prmt(t01h, t23h, 0x7632u);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int code = 4 * g + k;
      if (code >= kCodes) break;
      uint8_t *p0 = prof + (code * 32 + lane) * P0;
      if (P0 == 4) *reinterpret_cast<uint32_t *>(p0) = W[k][0];
      else *reinterpret_cast<uint2 *>(p0) = make_uint2(W[k][0], W[k][1]);
      if (P1 > 0) {
        constexpr int k1 = P0 / 4;       // first word of part 1
        uint8_t *p1 = prof + kCodes * 32 * P0 + (code * 32 + lane) * P1;
        if (P1 == 2) *reinterpret_cast<uint16_t *>(p1) = (uint16_t)W[k][k1];
        else if (P1 == 4) *reinterpret_cast<uint32_t *>(p1) = W[k][k1];
        else *reinterpret_cast<uint2 *>(p1) = make_uint2(W[k][k1], W[k][k1 + 1]);
      }
    }
  }
}

// this lane's R profile bytes for column code `code`, as 4 words (rows 4k..4k+3)
template <int R>
__device__ __forceinline__ uint4 load_profile_u8(const uint8_t *prof, int code, int lane) {
  constexpr int P0 = prof_p0(R), P1 = prof_p1(R);
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  const uint8_t *p0 = prof + (code * 32 + lane) * P0;
  if (P0 == 4) {
    v.x = *reinterpret_cast<const uint32_t *>(p0);
  } else {
    const uint2 a = *reinterpret_cast<const uint2 *>(p0);
    v.x = a.x;
    v.y = a.y;
  }
  if (P1 > 0) {
    const uint8_t *p1 = prof + kCodes * 32 * P0 + (code * 32 + lane) * P1;
    uint32_t a = 0u, b = 0u;
    if (P1 == 2) a = *reinterpret_cast<const uint16_t *>(p1);
    else if (P1 == 4) a = *reinterpret_cast<const uint32_t *>(p1);
    else {
      const uint2 q = *reinterpret_cast<const uint2 *>(p1);
      a = q.x;
      b = q.y;
    }
    if (P0 == 4) v.y = a;            // part 1 continues at word P0 / 4
    else { v.z = a; v.w = b; }
  }
  return v;
}

// byte k of a (low half) and byte k of b (high half), zero-extended:
// selector nibbles {k, k|8, 4+k, (4+k)|8}; bytes are < 128 so the
// sign-replicated bytes are 0.
__device__ __forceinline__ uint32_t sel_pair(int k) {
  return (uint32_t)k | ((uint32_t)(k | 8) << 4) | ((uint32_t)(4 + k) << 8) |
         ((uint32_t)((4 + k) | 8) << 12);
}

// The previous strip's bottom row comes from the duo's row checkpoints of its
// lane 31 (boundary nb-1), indexed by that lane's step = column + 31: one
// (Ho2, F2) pair of u16x2 words per column; lane l holds column 32k + l of the
// current block (cur) and of the next (nxt, fetched a block ahead).
struct PackedBoundaryReader {
  uint2 cur, nxt;
  const uint2 *r;             // row-checkpoint row of the previous strip's boundary nb-1
  int n;
  __device__ __forceinline__ uint2 ld(int c, uint2 dflt) const { return c < n ? r[c + 31] : dflt; }
  __device__ __forceinline__ void init(const uint2 *r_, int n_, int lane, uint2 dflt) {
    r = r_; n = n_;
    cur = ld(lane, dflt);
    nxt = ld(32 + lane, dflt);
  }
};

template <int R>
struct PackedLane {
  uint32_t Ho[R], E[R], rm[R];
  uint32_t hoUpPrev, botHo, botF;
};

struct PackedPair {        // one of the two pairs a warp carries
  int64_t k;               // pair index (-1: none)
  int m, n;
  RawView rows, cols;
  uint32_t *ck;            // checkpoint region (nullptr: no room -> box path)
  unsigned long long ck_off;
};

template <int R>
__global__ void __launch_bounds__(kWarpsPerBlockP * 32, packed_min_blocks(R))
k_score_packed(KArgs A, int stage, int cls) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t *smatT = smem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t *profA = smem + kMatTBytes + warp * warp_bytes_p(R);
  uint8_t *profB = profA + prof_bytes_p(R);
  uint8_t *ringA = profB + prof_bytes_p(R);
  uint8_t *ringB = ringA + kRingSlot;
  load_matrix_t(smatT, A.mat, A.prof_lo);
  const uint32_t Bs = (uint32_t)A.bias16;
  const uint32_t BB = A.p_bb;
  const uint32_t OPEN2 = A.p_open2;
  const uint32_t NEG2 = A.p_ext2;                      // biased "-inf": E/F - ext == 0
  const uint32_t HO0 = A.p_ho0;                        // biased H - open for H == 0
  const uint32_t NEXT2 = A.p_next2, NOPEN2 = A.p_nopen2;  // per-half -ext, -open
  for (;;) {
    // two consecutive work items per warp
    uint32_t pos = 0;
    if (lane == 0) pos = atomicAdd(&A.ctrs[kStages * kNumClasses + stage * kNumClasses + cls], 2u);
    pos = __shfl_sync(0xffffffffu, pos, 0);
    const uint32_t cnt = *(volatile uint32_t *)&A.ctrs[stage * kNumClasses + cls];
    if (pos >= cnt) break;
    PackedPair P[2];
    uint64_t arena_end = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t idx = pos + h;
      P[h].k = idx < cnt ? (int64_t)list_of(A, stage, cls)[idx] : -1;
      if (P[h].k >= 0) {
        const sw_pair_t p = A.pairs[P[h].k];
        arena_end = max(arena_end, max(p.a_off + p.a_len, p.b_off + p.b_len));
        P[h].m = (int)p.a_len;
        P[h].n = (int)p.b_len;
        const bool raw = A.ready || A.pair_ready;   // host arena still arriving: raw bytes + LUT
        const uint8_t *seq = raw ? A.raw : A.codes;
        const uint8_t *lut = raw ? A.lut : nullptr;
        P[h].rows = RawView{seq + p.a_off, lut};
        P[h].cols = RawView{seq + p.b_off, lut};
      } else {
        P[h].m = 0;
        P[h].n = 0;
        P[h].rows = RawView{A.codes, nullptr};
        P[h].cols = RawView{A.codes, nullptr};
      }
      P[h].ck = nullptr;
      P[h].ck_off = 0;
    }
    wait_arena(A, arena_end, lane);   // host-pipelined arena: its slices may still be arriving
    wait_pairs(A, P[0].k, P[1].k, lane);   // gathered arena: this duo's bytes
    const int m = max(P[0].m, P[1].m), n = max(P[0].n, P[1].n);
    const int nstrips = (m + 32 * R - 1) / (32 * R);
    const CkLayout CL = ck_layout(R, n);
    // one pool allocation per duo: [pair A columns][pair B columns][duo rows]
    const int npair = 1 + (P[1].k >= 0);
    const uint64_t colb = (uint64_t)nstrips * CL.col_words * 4ull;
    const uint64_t bytes = npair * colb + (uint64_t)nstrips * CL.row_words * 4ull;
    uint2 *rowck = nullptr;
    {
      unsigned long long off = 0;
      if (lane == 0) off = atomicAdd(A.pool_top, (unsigned long long)bytes);
      off = __shfl_sync(0xffffffffu, off, 0);
      if (off + bytes <= A.pool_cap) {
        P[0].ck = reinterpret_cast<uint32_t *>(A.pool + off);
        P[0].ck_off = off;
        if (npair == 2) {
          P[1].ck = reinterpret_cast<uint32_t *>(A.pool + off + colb);
          P[1].ck_off = off + colb;
        }
        rowck = reinterpret_cast<uint2 *>(A.pool + off + npair * colb);
      }
    }
    // When the pool is full the duo's pairs are deferred to the next round
    // (stage 8; the pool is recycled between rounds), or -- a pair whose
    // checkpoints alone would take over a quarter of the pool -- sent to the
    // scalar path.
    auto defer = [&](int h) {
      PairState *st = A.st + P[h].k;
      const CkLayout OL = ck_layout(R, P[h].n);
      const uint64_t own = (uint64_t)((P[h].m + 32 * R - 1) / (32 * R)) *
                           (OL.col_words + OL.row_words) * 4ull;
      if (own > A.pool_cap / 4) {
        st->flags = 0;
        list_push(A, 0, kFallbackClass, (uint32_t)P[h].k);
      } else {
        st->flags = kFlagRetry;                 // k_walk leaves it alone this round
        list_push(A, 8, cls, (uint32_t)P[h].k);
      }
    };
    if (!rowck) {
      if (lane == 0) {
        defer(0);
        if (P[1].k >= 0) defer(1);
      }
      continue;
    }
    uint64_t keyA = 0ull, keyB = 0ull;
    uint32_t vmax2 = 0u;
    for (int strip = 0; strip < nstrips; ++strip) {
      const int row0 = strip * 32 * R;
      __syncwarp();
      build_profile_u8<R>(profA, smatT, P[0].rows, P[0].m, row0, lane);
      build_profile_u8<R>(profB, smatT, P[1].rows, P[1].m, row0, lane);
      __syncwarp();
      PackedLane<R> L;
#pragma unroll
      for (int r = 0; r < R; ++r) { L.Ho[r] = HO0; L.E[r] = NEG2; L.rm[r] = BB; }
      L.hoUpPrev = HO0;
      L.botHo = HO0;
      L.botF = NEG2;
      // column-code rings: slot c & 127 holds column c; prefill [-32, 96)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = -32 + 32 * q + lane;
        const uint8_t va = (c >= 0 && c < P[0].n) ? (uint8_t)P[0].cols.at(c) : (uint8_t)kPad;
        const uint8_t vb = (c >= 0 && c < P[1].n) ? (uint8_t)P[1].cols.at(c) : (uint8_t)kPad;
        ringA[c & 127] = va;
        ringB[c & 127] = vb;
        if ((c & 127) < 8) { ringA[(c & 127) + 128] = va; ringB[(c & 127) + 128] = vb; }
      }
      // the next refill's codes (columns 96 + lane), loaded one refill ahead
      // (A/B on the box: forward +1.2 % config 3, +0.9 % config 2)
      uint8_t nxtA = 96 + lane < P[0].n ? (uint8_t)P[0].cols.at(96 + lane) : (uint8_t)kPad;
      uint8_t nxtB = 96 + lane < P[1].n ? (uint8_t)P[1].cols.at(96 + lane) : (uint8_t)kPad;
      // Row above the strip (lane 0): the previous strip's bottom row; strip 0
      // gets an empty reader, which returns the zero row.  One loop for every
      // strip: a second copy without the reader for strip 0 was 3.4 % slower
      // on config 3 (instruction-cache misses: "no instruction" stalls 0.35
      // per issue with two copies of the 8-step loop) and 1.6 % faster on
      // config 2.
      PackedBoundaryReader br;
      const uint2 dflt = make_uint2(HO0, NEG2);   // (H-open at H=0, F=-inf), both halves
      br.init(rowck + ((uint64_t)max(strip - 1, 0) * CL.row_words + (uint64_t)(CL.nb - 1) * 2 * CL.spad) / 2,
              strip > 0 ? n : 0, lane, dflt);
      // checkpoint destinations for this strip
      uint32_t *colA = P[0].ck + (uint64_t)strip * CL.col_words + lane;
      uint32_t *colB = P[1].ck ? P[1].ck + (uint64_t)strip * CL.col_words + lane : nullptr;
      const int b = ck_boundary(lane, CL);
      // row checkpoints of this strip, [boundary][step] uint2
      uint4 *rowdst = reinterpret_cast<uint4 *>(rowck + (uint64_t)strip * CL.row_words / 2);
      const int steps = n + 31;
      // boundary lanes keep their bottom rows of 8 steps in registers and
      // write them as four 16-B stores (64 contiguous bytes of [boundary][step]);
      // A/B on the box against staging through shared memory and a warp-wide
      // flush: forward +4.5 % (config 3), +5.7 % (config 2)
      uint4 *rowmine = b >= 0 ? rowdst + (uint64_t)b * (CL.spad / 2) : nullptr;
      uint2 rowv[kUnrollP];
      // column checkpoint: state entering window w (after step 32w - 1)
      auto colck = [&](int w) {
        if (w < CL.nwin) {
          const uint64_t base = (uint64_t)w * 32 * ck_words(R);
          uint32_t lm = L.rm[0];   // running maximum over the lane's rows (k_tb's j_end search)
#pragma unroll
          for (int r = 1; r < R; ++r) lm = vmax2u(lm, L.rm[r]);
          {
            uint32_t *d = colA + base;
#pragma unroll
            for (int r = 0; r < R; ++r) d[32 * r] = prmt(L.Ho[r], L.E[r], 0x5410u);
            d[32 * R] = prmt(L.hoUpPrev, L.botF, 0x5410u);
            d[32 * (R + 1)] = lm & 0xFFFFu;
          }
          if (colB) {
            uint32_t *d = colB + base;
#pragma unroll
            for (int r = 0; r < R; ++r) d[32 * r] = prmt(L.Ho[r], L.E[r], 0x7632u);
            d[32 * R] = prmt(L.hoUpPrev, L.botF, 0x7632u);
            d[32 * (R + 1)] = lm >> 16;
          }
        }
      };
      // lane 0 reads the row above from shared memory: 32 columns staged at
      // each refill, one broadcast LDS per step instead of two shuffles (A/B
      // on the box: forward +2.3 % config 3, +0.8 % config 2)
      uint2 *bnd = reinterpret_cast<uint2 *>(ringB + kRingSlot);
      bnd[lane] = br.cur;
      __syncwarp();
      for (int s0 = 0; s0 < steps; s0 += kUnrollP) {
        if ((s0 & 31) == 0 && s0 > 0) {    // refill ring slots for columns s0+64 .. s0+95
          // the checkpoint of the window that just ended is stored here,
          // beside the refill, not at the end of the previous chunk (A/B on
          // the box: forward +0.8 % config 3, +1.5 % config 2)
          colck(s0 >> 5);
          const int c = s0 + 64 + lane;
          ringA[c & 127] = nxtA;
          ringB[c & 127] = nxtB;
          if ((c & 127) < 8) { ringA[(c & 127) + 128] = nxtA; ringB[(c & 127) + 128] = nxtB; }
          nxtA = c + 32 < P[0].n ? (uint8_t)P[0].cols.at(c + 32) : (uint8_t)kPad;
          nxtB = c + 32 < P[1].n ? (uint8_t)P[1].cols.at(c + 32) : (uint8_t)kPad;
          bnd[lane] = br.nxt;
          br.nxt = br.ld(s0 + 32 + lane, dflt);
          __syncwarp();
        }
        const int rbase = (s0 - lane) & 127;   // ring slot of this lane's column at step s0
#pragma unroll
        for (int q = 0; q < kUnrollP; ++q) {
          const int s = s0 + q;
          const uint4 pa = load_profile_u8<R>(profA, ringA[rbase + q], lane);
          const uint4 pb = load_profile_u8<R>(profB, ringB[rbase + q], lane);
          // the row above: from lane t-1, or (lane 0, whose shuffle source is
          // out of range) from the staged boundary row -- selected by the
          // shuffle's own valid predicate (A/B against a lane-index select:
          // forward +0.9 % config 3, +1.1 % config 2)
          const uint2 bv = bnd[s & 31];
          const uint32_t upHo = shfl_up_or(L.botHo, bv.x);
          const uint32_t upF = shfl_up_or(L.botF, bv.y);
          uint32_t diag = L.hoUpPrev;
          L.hoUpPrev = upHo;
          // F carried as G = F + open (biased): G[r] = max(G[r-1] - ext, t[r-1]),
          // t[-1] = H of the row above; H[r] = max(G[r] - open, t[r]).
          uint32_t G = upF + OPEN2, tprev = upHo + OPEN2;
#ifndef K1P_ONE_PASS
          // t[r] depends only on the previous step's values: compute them all
          // first, then run the F (G) chain, so the chain's latency overlaps
          // independent work (A/B on the box: forward +0.4 % config 3,
          // +0.9 % config 2)
          uint32_t tt[R];
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const uint32_t u2 = prmt(word_of(pa, r), word_of(pb, r), sel_pair(r & 3));
            L.E[r] = __viaddmax_u16x2(L.E[r], NEXT2, L.Ho[r]);
            tt[r] = vmax2u(vmax2u((r == 0 ? diag : L.Ho[r - 1]) + u2, L.E[r]), BB);
          }
#pragma unroll
          for (int r = 0; r < R; ++r) {
            G = __viaddmax_u16x2(G, NEXT2, r == 0 ? tprev : tt[r - 1]);
            const uint32_t h = __viaddmax_u16x2(G, NOPEN2, tt[r]);
            L.Ho[r] = h - OPEN2;
            L.rm[r] = vmax2u(L.rm[r], h);
          }
#else
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
#endif
          L.botHo = L.Ho[R - 1];
          L.botF = G - OPEN2;
          rowv[q] = make_uint2(L.botHo, L.botF);
        }
        if (rowmine) {
#pragma unroll
          for (int i = 0; i < kUnrollP / 2; ++i)
            rowmine[s0 / 2 + i] = make_uint4(rowv[2 * i].x, rowv[2 * i].y, rowv[2 * i + 1].x, rowv[2 * i + 1].y);
        }
      }
      {   // the window boundary the loop ended on, if any
        const int send = (steps + kUnrollP - 1) / kUnrollP * kUnrollP;
        if ((send & 31) == 0) colck(send >> 5);
      }
      // strip reduction: best and the first row reaching it, per pair
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int x = row0 + lane * R + r;
        const uint32_t va = L.rm[r] & 0xFFFFu, vb = L.rm[r] >> 16;
        vmax2 = max(vmax2, max(va, vb));
        if (x < P[0].m) {
          const uint64_t kk = ((uint64_t)(va - Bs) << 32) | ((uint64_t)(0xFFFF - x) << 16);
          keyA = kk > keyA ? kk : keyA;
        }
        if (x < P[1].m) {
          const uint64_t kk = ((uint64_t)(vb - Bs) << 32) | ((uint64_t)(0xFFFF - x) << 16);
          keyB = kk > keyB ? kk : keyB;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t a2 = __shfl_xor_sync(0xffffffffu, keyA, o);
      keyA = a2 > keyA ? a2 : keyA;
      const uint64_t b2 = __shfl_xor_sync(0xffffffffu, keyB, o);
      keyB = b2 > keyB ? b2 : keyB;
      vmax2 = max(vmax2, (uint32_t)__shfl_xor_sync(0xffffffffu, vmax2, o));
    }
    if (lane == 0) {
      const bool overflow = vmax2 > kPackedLimit;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (P[h].k < 0) continue;
        PairState *st = A.st + P[h].k;
        const uint64_t key = h == 0 ? keyA : keyB;
        const int32_t best = (int32_t)(key >> 32);
        const int32_t i_end = 0xFFFF - (int32_t)((key >> 16) & 0xFFFF);
        st->i0 = 0;
        st->j0 = 0;
        // The tile traceback (k_tb) replays H/E/F in int16 shared-memory
        // tiles: exact while best <= 32767 (every replayed value lies in
        // [-open, best]).  A pair scoring above that (only reachable with
        // large custom matrices: BLOSUM62 tops out at 11 per residue) takes
        // the int32 path: wide forward, reverse pass, box traceback.
        if (overflow || best > kTileMax) {     // overflow: both halves suspect
          st->flags = kFlagWide;
          list_push(A, 3, 0, (uint32_t)P[h].k);
        } else if (best == 0) {
          st->best = 0;
          st->i_end = -1;
          st->j_end = -1;
          st->flags = 0;
        } else if (P[h].ck) {
          st->best = best;
          st->i_end = i_end;
          st->j_end = -1;                      // resolved by k_tb from the checkpoints
          st->flags = kFlagNeedJ | (h ? kFlagHi : 0);
          st->code_off = P[h].ck_off;
          st->row_delta = (uint32_t)((uint64_t)((const uint8_t *)rowck - A.pool) - P[h].ck_off);
          st->box_cls = cls;
          st->box_m = m;
          st->box_n = n;
          list_push(A, 7, cls, (uint32_t)P[h].k);
        } else {                               // no checkpoint room
          defer(h);
        }
      }
    }
  }
}

}  // namespace pastis
