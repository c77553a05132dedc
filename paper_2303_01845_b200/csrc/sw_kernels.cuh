// sw_kernels.cuh -- sm_100a kernels of the batched Smith-Waterman aligner.
//
// Exact restatement, on the GPU, of the reference CPU aligner
// /root/reference/pkg/src/pastislite/align.py:79-181:
//   K1 k_score<FWD>  forward fill (align.py:103-121) + row-major-first argmax
//                    (align.py:124: max score, then min i, then min j)
//   K2 k_score<REV>  the same fill on the reversed prefixes a[0..i_end],
//                    b[0..j_end]; the cells reaching `best` there are the
//                    starts of optimal alignments -> min-box (i0, j0)
//   K3 k_box         fill of the box [i0..i_end]x[j0..j_end] emitting 4-bit
//                    traceback codes (Hsrc, Fopen, Eopen) per cell
//   K4 k_walk        the traceback state machine of align.py:133-169 over
//                    those codes (box lemma: SURVEY.md App. A.6)
//
// Layout: one warp per pair.  Lane t owns R consecutive rows of a 32*R-row
// strip; at wavefront step s it updates column c = s - t, receiving the row
// above (H-open, F) from lane t-1 by __shfl_up_sync.  Scores come from a
// per-warp int8 query profile in shared memory, prof[code][lane][16], read
// with one 128-bit LDS per step (conflict-free: lane stride 16 B).
//
// Forward/reverse passes run in a "scaled" int32 domain: every DP value is
// held as v * 2^16, so a single DPX op  key = max(h + cc, key)  tracks the
// per-row maximum AND the column where it was first reached (cc = 65535 - c).
// That keeps the per-cell cost at 4 DPX + 1 VIMNMX3 + 1 PRMT + 2 IADD.
// Values are exact while best < 2^15 - 128; a pair whose running maximum
// reaches that limit is re-run in the "wide" variant (unscaled int32 with
// 64-bit keys).  The box pass is always unscaled int32.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>
#include "../../include/pastis_sw.h"

namespace pastis {

constexpr int kAlpha = 25;
constexpr int kPad = 25;                 // code of virtual cells (outside the matrix)
constexpr int kCodes = 26;
constexpr int kLaneBytes = 16;           // profile bytes per lane per code (R <= 16)
constexpr int kProfStride = 32 * kLaneBytes;
constexpr int kProfBytes = kCodes * kProfStride;  // 13,312 B per warp
constexpr int kMatBytes = 688;           // 26*26 int8, padded to 16
constexpr int kWarpsPerBlock = 4;
constexpr int kNumClasses = 7;
constexpr int kLongClass = kNumClasses - 1;  // R = 16: the only class of the long-pair path
constexpr int kCtaClass = 0;    // long pairs with >= 4 strips: one CTA per pair (sw_cta.cuh)
// stage-0 list of the packed pass's no-checkpoint-room fallbacks.  Kept apart
// from kLongClass's list: that list is drained by a launch running
// concurrently with the packed pass, and a warp that finds a list empty still
// advances its cursor, so items appended behind it would never be fetched.
constexpr int kFallbackClass = 1;
// stage-0 list of long pairs the packed CTA kernel could not take (no pool
// room for its boundary slots): the scalar one-CTA-per-pair kernel
constexpr int kCtaScalarClass = 2;
constexpr int kCtaRowsR = 16;   // rows per lane of the CTA kernels
constexpr int kCtaStripsMin = 4;
__host__ __device__ inline int long_class(int m, bool packed_ok = true) {
  return packed_ok && (m + 32 * kCtaRowsR - 1) / (32 * kCtaRowsR) >= kCtaStripsMin ? kCtaClass
                                                                                    : kLongClass;
}
constexpr int kStages = 10; // 0 K1, 1 K2, 2 K3, 3 K1-wide, 4 K2-wide, 5 retry,
                            // 6 K1 with checkpoints, 7 tile traceback,
                            // 8 K1 with checkpoints deferred to the next round (pool full),
                            // 9 j_end replay of the packed long-pair forward (k_jend)
constexpr uint64_t kFusedMaxCells = 1ull << 22;  // pairs up to 2048x2048 take the fused path
constexpr int32_t kScaledLimit = 32767 - 128;
constexpr int32_t kNegInf = -(1 << 30);

// Length classes: R rows per lane, 32R rows per strip.  class_of (box
// traceback lists): the class whose strips pad m the least (ties: larger R,
// fewer strips).  packed_class_of (packed forward): the least modelled cost.
__host__ __device__ constexpr int class_rows(int cls) {
  return cls == 0 ? 4 : cls == 1 ? 6 : cls == 2 ? 7 : cls == 3 ? 8 : cls == 4 ? 9 : cls == 5 ? 10 : 16;
}
__host__ __device__ inline int class_of(int m) {
  int best = kNumClasses - 1;
  long best_rows = 1L << 40;
  for (int c = kNumClasses - 1; c >= 0; --c) {
    const long rows_per_strip = 32L * class_rows(c);
    const long rows = (m + rows_per_strip - 1) / rows_per_strip * rows_per_strip;
    if (rows < best_rows) { best_rows = rows; best = c; }
  }
  return best;
}
// Issue-slot model of the packed forward (k_score_packed<R>, profiled on the
// box): per strip, n + 31 wavefront steps of ~9R + 23 instructions (9 per
// packed row-word + ~23 per step: shuffles, profile/ring loads, row
// checkpoints), ~6 more per step when the row above comes from the previous
// strip, and ~260R to build the strip's profile; classes whose profiles
// limit residency to 2 blocks/SM (R >= 12) pay x1.5.
__host__ __device__ inline int packed_class_of(int m, int n) {
  int best = 0;
  float best_cost = 3.4e38f;
  for (int c = 0; c < kNumClasses; ++c) {
    const int R = class_rows(c);
    const int S = (m + 32 * R - 1) / (32 * R);
    float cost = (float)S * (float)(n + 31) * (float)(9 * R + 23) +
                 (float)(S - 1) * (float)(n + 31) * 6.f + (float)S * 260.f * (float)R;
    if (R >= 12) cost *= 1.5f;
    if (cost < best_cost) { best_cost = cost; best = c; }
  }
  return best;
}
__host__ __device__ constexpr int box_lane_bytes(int R) { return R <= 4 ? 2 : R <= 8 ? 4 : 8; }

enum : int32_t { kFlagWide = 1, kFlagRetry = 2, kFlagDone = 4, kFlagNeedJ = 8, kFlagInvalid = 16,
                 kFlagHi = 32 };  // kFlagHi: the pair is the high half of its duo's row checkpoints

struct PairState {         // per-pair scratch between the passes (48 B)
  int32_t best, i_end, j_end, flags;
  int32_t i0, j0, box_cls, box_n;  // traceback-code box origin, class (R) and width
  uint64_t code_off;               // byte offset of the box's codes in the pool
  int32_t box_m;
  uint32_t row_delta;              // packed path: duo row checkpoints at code_off + row_delta
};

struct KArgs {
  const uint8_t *codes;    // residue codes 0..24 of the arena (k_encode)
  const uint8_t *raw;      // raw arena bytes (for `matches`, align.py:142)
  const sw_pair_t *pairs;
  PairState *st;
  sw_result_t *out;
  const int8_t *mat;       // 26x26 int8 (row/col 25 = virtual, -128)
  uint32_t *lists;         // [kStages][kNumClasses][n_pairs]
  uint32_t *ctrs;          // count[kStages*kNumClasses], cursor[...] after it
  uint64_t n_pairs;
  uint64_t arena_bytes;     // pairs must lie inside [arena_lo, arena_bytes) (checked by k_classify)
  uint64_t arena_lo;        // first valid arena offset: raw/codes are virtual bases such that
                            // raw + off is valid for off in [arena_lo, arena_bytes) (a shard
                            // of a batch uploads only that byte range)
  const uint8_t *lut;      // raw byte -> residue code (align.py:27-30), 256 entries
  // host-pipelined arenas: ready = number of arena slices of slice_bytes that
  // have landed (written by the copy stream); nullptr = arena fully resident
  const volatile uint32_t *ready;
  uint64_t slice_bytes;
  // host arena gathered on the device (k_gather_arena): per-pair flags set
  // once the pair's bytes are in the device arena; nullptr = not gathering
  const volatile uint32_t *pair_ready;
  const uint8_t *gather_src;   // the pinned host arena (device-mapped) being gathered
  uint8_t *gather_dst;         // the device arena it is gathered into (same offsets)
  const volatile uint32_t *gather_count;   // pairs the gather kernel has copied so far
  uint2 *cta_rows;         // K1cp: per-CTA ring of strip bottom rows (sw_cta_packed.cuh)
  int2 *bnd;               // per-warp strip boundary rows
  uint64_t bnd_stride;     // int2 per warp
  uint8_t *pool;           // traceback code pool
  uint64_t pool_cap;
  unsigned long long *pool_top;
  int32_t open_, ext;
  int32_t bias16;           // B: checkpoint values are stored as u16 (v + B)
  int32_t prof_lo;          // packed profile stores s - prof_lo = s + open (0..127); PAD -> 0
  // packed (u16x2) constants, precomputed on the host so they live in the
  // constant bank: B, open, ext splatted to both halves, H-open at H=0, and
  // -ext, -open per half (for the wrapping per-half adds of VIADDMNMX.U16x2)
  uint32_t p_bb, p_open2, p_ext2, p_ho0, p_next2, p_nopen2;
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// value of lane - 1, or `fill` in lane 0 (the shuffle's valid predicate
// picks it, no lane-index compare)
__device__ __forceinline__ uint32_t shfl_up_or(uint32_t v, uint32_t fill) {
  uint32_t r;
  asm("{ .reg .pred p;\n\t"
      "shfl.sync.up.b32 %0|p, %1, 1, 0, 0xffffffff;\n\t"
      "@!p mov.b32 %0, %2;\n\t}"
      : "=r"(r) : "r"(v), "r"(fill));
  return r;
}
// byte k of w, sign-extended, times 65536 (scaled) or times 1 (plain)
__device__ __forceinline__ uint32_t sel_scaled(int k) {
  return 0x44u | ((uint32_t)k << 8) | ((uint32_t)(k | 8) << 12);
}
__device__ __forceinline__ uint32_t sel_plain(int k) {
  const uint32_t s = (uint32_t)(k | 8);
  return (uint32_t)k | (s << 4) | (s << 8) | (s << 12);
}
__device__ __forceinline__ uint32_t word_of(const uint4 &p, int r) {
  return r < 4 ? p.x : r < 8 ? p.y : r < 12 ? p.z : p.w;
}

__device__ __forceinline__ uint32_t *list_of(const KArgs &A, int stage, int cls) {
  return A.lists + ((uint64_t)stage * kNumClasses + cls) * A.n_pairs;
}
__device__ __forceinline__ void list_push(const KArgs &A, int stage, int cls, uint32_t k) {
  uint32_t pos = atomicAdd(&A.ctrs[stage * kNumClasses + cls], 1u);
  list_of(A, stage, cls)[pos] = k;
}
// warp-cooperative work fetch; returns pair index or -1
__device__ __forceinline__ int64_t next_item(const KArgs &A, int stage, int cls, int lane) {
  uint32_t pos = 0;
  if (lane == 0) pos = atomicAdd(&A.ctrs[kStages * kNumClasses + stage * kNumClasses + cls], 1u);
  pos = __shfl_sync(0xffffffffu, pos, 0);
  const uint32_t cnt = *(volatile uint32_t *)&A.ctrs[stage * kNumClasses + cls];
  if (pos >= cnt) return -1;
  return (int64_t)list_of(A, stage, cls)[pos];
}

// A sequence view: element x is codes[base + step * x].
struct View {
  const uint8_t *p;
  int step;
  __device__ __forceinline__ int at(int x) const { return p[(int64_t)step * x]; }
};
// The packed forward's sequence view.  Resident arena: p = encoded codes,
// lut = nullptr.  Host-pipelined arena: p = RAW bytes encoded on the fly
// (lut[raw]) with L1-bypassing loads, since slices may still be arriving
// while the kernel runs (A.ready).
struct RawView {
  const uint8_t *p;
  const uint8_t *lut;
  __device__ __forceinline__ int at(int x) const {
    return lut ? (int)__ldg(lut + __ldcg(p + x)) : (int)__ldg(p + x);
  }
};
// Wait until the arena slices holding [0, end) have landed (no-op when the
// arena is resident).  Lane 0 spins; the copy stream needs no SM.
__device__ __forceinline__ void wait_arena(const KArgs &A, uint64_t end, int lane) {
  if (A.ready == nullptr || end == 0) return;
  if (lane == 0) {
    const uint32_t need = (uint32_t)((end - A.arena_lo - 1) / A.slice_bytes + 1);
    while (*A.ready < need) __nanosleep(256);
  }
  __syncwarp();
}

// Gather of a pinned host arena into the device arena in the order the packed
// pass will consume it (segments: round r of the packed class lists -- list
// positions [r cnt/Rn, (r+1) cnt/Rn) of every class -- then the long-pair
// lists), one warp per pair: 128-bit loads over PCIe (zero-copy), byte
// stores, then the pair's ready flag.  Pairs sharing a sequence copy the same
// bytes twice (identical data).
struct GatherSeg {
  uint32_t list;    // stage * kNumClasses + cls
  uint32_t j0;      // first list position of the segment
  uint32_t start;   // global item index of the segment's first item
};
__device__ __forceinline__ void warp_copy16(const uint8_t *__restrict__ src, uint8_t *__restrict__ dst,
                                            uint32_t len, int lane) {
  // src + i -> dst + i for i < len; loads aligned on the source's absolute
  // address (the over-read stays inside the 16-byte words, hence the page)
  if (len == 0) return;
  const uintptr_t a0 = (uintptr_t)src, a1 = a0 + len;
  for (uintptr_t w = (a0 & ~(uintptr_t)15) + 16u * lane; w < a1; w += 16u * 32) {
    const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(w));   // streamed: read once
    const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int b = 0; b < 16; ++b) {
      const uintptr_t pos = w + b;
      if (pos >= a0 && pos < a1) dst[pos - a0] = (uint8_t)(x[b >> 2] >> (8 * (b & 3)));
    }
  }
}
// Wait until the gather kernel has copied pairs k0 (and k1 >= 0) into the
// device arena (no-op when the arena is resident).  The gather kernel runs
// beside the packed pass and is normally far ahead; if a pair is not ready
// while the gather makes no progress for 20 us -- e.g. the packed pass's
// blocks hold every SM and the gather kernel's blocks never became resident --
// the warp copies the pair itself (identical bytes; the gather may copy it
// again), so no schedule can deadlock.
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void wait_pairs(const KArgs &A, int64_t k0, int64_t k1, int lane) {
  if (A.pair_ready == nullptr) return;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int64_t k = h ? k1 : k0;
    if (k < 0) continue;
    int ok = 0;
    if (lane == 0) {
      // give up only when the gather has made no progress for 20 us
      uint64_t t0 = globaltimer_ns();
      uint32_t seen = *A.gather_count;
      while (!(ok = A.pair_ready[k] != 0u)) {
        __nanosleep(200);
        if (globaltimer_ns() - t0 > 20000ull) {
          const uint32_t now = *A.gather_count;
          if (now == seen) break;
          seen = now;
          t0 = globaltimer_ns();
        }
      }
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    if (!ok) {
      const sw_pair_t p = A.pairs[k];
      warp_copy16(A.gather_src + p.a_off, A.gather_dst + p.a_off, p.a_len, lane);
      warp_copy16(A.gather_src + p.b_off, A.gather_dst + p.b_off, p.b_len, lane);
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicExch(const_cast<uint32_t *>(A.pair_ready + k), 1u);
    }
  }
  if (lane == 0) __threadfence();
  __syncwarp();
}

__global__ void k_gather_arena(KArgs A, const uint8_t *__restrict__ src, uint8_t *dst,
                               const GatherSeg *__restrict__ seg, int nseg, uint32_t total,
                               uint32_t *ready) {
  const int lane = threadIdx.x & 31;
  const uint32_t nw = gridDim.x * (blockDim.x >> 5);
  for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < total; i += nw) {
    int lo = 0, hi = nseg - 1;                 // last segment with start <= i
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (seg[mid].start <= i) lo = mid; else hi = mid - 1;
    }
    const GatherSeg g = seg[lo];
    const uint32_t k = A.lists[(uint64_t)g.list * A.n_pairs + g.j0 + (i - g.start)];
    const sw_pair_t p = A.pairs[k];
    warp_copy16(src + p.a_off, dst + p.a_off, p.a_len, lane);
    warp_copy16(src + p.b_off, dst + p.b_off, p.b_len, lane);
    __threadfence();
    __syncwarp();
    if (lane == 0) {
      atomicExch(&ready[k], 1u);
      atomicAdd(const_cast<uint32_t *>(A.gather_count), 1u);
    }
  }
}

// Build this lane's slice of the query profile for rows row0+lane*R .. +R-1.
template <int R>
__device__ __forceinline__ void build_profile(uint8_t *prof, const int8_t *mat, const View &rows,
                                              int m, int row0, int lane) {
  int arow[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int x = row0 + lane * R + r;
    arow[r] = x < m ? rows.at(x) : kPad;
  }
#pragma unroll 2
  for (int code = 0; code < kCodes; ++code) {
    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int r = 0; r < R; ++r)
      w[r >> 2] |= (uint32_t)(uint8_t)mat[code * kCodes + arow[r]] << (8 * (r & 3));
    *reinterpret_cast<uint4 *>(prof + code * kProfStride + lane * kLaneBytes) =
        make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// Lane 0 of a strip > 0 reads the previous strip's bottom row through a
// 32-column register chunk (double-buffered, coalesced loads).
struct BoundaryReader {
  int2 cur, nxt;
  int lim;   // columns >= lim read as dflt (n, or the reverse pass's stop column of the row above)
  __device__ __forceinline__ void init(const int2 *bnd, int n, int lane, int2 dflt) {
    lim = n;
    cur = lane < n ? bnd[lane] : dflt;
    nxt = 32 + lane < n ? bnd[32 + lane] : dflt;
  }
  __device__ __forceinline__ int2 get(const int2 *bnd, int s, int, int lane, int2 dflt) {
    if ((s & 31) == 0 && s > 0) {
      cur = nxt;
      const int c = s + 32 + lane;
      nxt = c < lim ? bnd[c] : dflt;
    }
    int2 v;
    v.x = __shfl_sync(0xffffffffu, cur.x, s & 31);
    v.y = __shfl_sync(0xffffffffu, cur.y, s & 31);
    return v;
  }
};

// ---------------------------------------------------------------------------
// K1/K2: score pass.  MODE 0 = forward (argmax row-major-first),
// MODE 1 = reverse (max x, max y over cells == best).
// WIDE=false: scaled int32 (v << 16); WIDE=true: plain int32 + 64-bit keys.
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Checkpoints written by the forward pass (short/medium pairs) so that the
// traceback can replay only the 32-column tiles its path crosses:
//  * column checkpoints: at the end of every 32-step window w-1 each lane
//    stores its state entering window w: (Ho_r, E_r) for its R rows,
//    (hoUpPrev, F_bot), and the running maximum over its R rows -> R+2
//    words, values as biased u16 (v + B) (per-row maxima: 2R+1 words, ~1 %
//    slower forward on configs 2/3 for the rare second j_end tile they save);
//  * row checkpoints: "boundary" lanes (the last lane of each group of
//    G = 32/R lanes, and lane 31) store their bottom-row (Ho, F) every step.
// Per strip: [window][word 0..R+1][lane] words per pair (coalesced stores), and
// [boundary][step][2] words per duo -- the raw (Ho2, F2) u16x2 words of the
// packed pass, both pairs in one word (PairState.row_delta, kFlagHi).
// ---------------------------------------------------------------------------
// column-checkpoint words per lane and window: (Ho, E) of each of the R rows,
// (hoUpPrev, F_bot), and the running maximum over the lane's rows
__host__ __device__ constexpr int ck_words(int R) { return R + 2; }
struct CkLayout {
  int G, nb, nwin, spad;
  uint32_t col_words;   // per pair and strip: column checkpoints
  uint32_t row_words;   // per duo and strip: row checkpoints, [boundary][step][2] words
};
__host__ __device__ inline CkLayout ck_layout(int R, int n) {
  CkLayout L;
  L.G = 32 / R;
  L.nb = (32 + L.G - 1) / L.G;
  L.nwin = (n + 31 + 31) / 32;
  L.spad = L.nwin * 32;
  L.col_words = (uint32_t)L.nwin * 32u * (uint32_t)ck_words(R);
  L.row_words = 2u * (uint32_t)L.nb * (uint32_t)L.spad;
  return L;
}
// boundary index of lane t (-1 when t is not a boundary lane)
__host__ __device__ inline int ck_boundary(int t, const CkLayout &L) {
  if (t == 31) return L.nb - 1;
  return ((t + 1) % L.G == 0) ? (t + 1) / L.G - 1 : -1;
}
// pack the high halves (the unscaled values) of two scaled words
__device__ __forceinline__ uint32_t pack_hi16(int32_t lo, int32_t hi) {
  return prmt((uint32_t)lo, (uint32_t)hi, 0x7632u);
}

struct ScoreOut {
  uint64_t fwd;     // (best << 32) | (0xFFFF - row) << 16 | (0xFFFF - col)
  int32_t rev_x, rev_y;
  int32_t vmax;     // running max seen (overflow guard)
};

template <int R, bool WIDE>
struct ScoreLane {
  int32_t Ho[R], E[R];
  typename std::conditional<WIDE, long long, int32_t>::type key[R];
  int32_t hoUpPrev, botHo, botF;
  int code_next;
};

// One wavefront step of the score pass (lane t updates column s - t).
template <int R, int MODE, bool WIDE>
__device__ __forceinline__ void score_step(ScoreLane<R, WIDE> &L, const uint8_t *prof,
                                           const View &cols, const int s, const int n,
                                           const int lane, const bool has_above,
                                           const bool has_below, BoundaryReader &br, int2 *bnd,
                                           const int2 dflt, const int32_t OPEN,
                                           const int32_t nEXT, const int32_t FLOOR) {
  const int c = s - lane;
  const bool valid = (c >= 0) & (c < n);
  const int code = L.code_next;
  {
    const int cn = c + 1;
    L.code_next = (cn >= 0 && cn < n) ? cols.at(cn) : kPad;
  }
  const uint4 pw = *reinterpret_cast<const uint4 *>(prof + code * kProfStride + lane * kLaneBytes);
  int32_t upHo = __shfl_up_sync(0xffffffffu, L.botHo, 1);
  int32_t upF = __shfl_up_sync(0xffffffffu, L.botF, 1);
  if (has_above) {
    const int2 b = br.get(bnd, s, n, lane, dflt);
    if (lane == 0) { upHo = b.x; upF = b.y; }
  } else if (lane == 0) {
    // row 0: H = 0 (local) / -inf (anchored reverse pass, MODE 1)
    upHo = MODE == 1 ? dflt.x : -OPEN;
    upF = MODE == 1 ? dflt.y : kNegInf;
  }
  int32_t cc = 0;
  if (valid) cc = MODE == 0 ? 65535 - c : c + 1;
  int32_t diag = L.hoUpPrev;
  L.hoUpPrev = upHo;
  int32_t F = upF, hoUp = upHo;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    // short F chain (open >= ext): F[r+1] = max(F[r] - ext, max(D, E, 0) - open),
    // see sw_packed.cuh; H = max(t, F) stays off the chain
    const uint32_t w = word_of(pw, r);
    const int32_t sc = (int32_t)prmt(w, 0u, WIDE ? sel_plain(r & 3) : sel_scaled(r & 3));
    L.E[r] = __viaddmax_s32(L.E[r], nEXT, L.Ho[r]);
    const int32_t D = diag + sc + OPEN;
    // forward: local (relu); reverse: anchored, floored at FLOOR (see score_pair)
    const int32_t t = MODE == 1 ? __vimax3_s32(D, L.E[r], FLOOR) : __vimax_s32_relu(D, L.E[r]);
    F = __viaddmax_s32(F, nEXT, hoUp);
    const int32_t h = max(t, F);
    diag = L.Ho[r];
    const int32_t ho = h - OPEN;
    L.Ho[r] = ho;
    hoUp = t - OPEN;
    if constexpr (WIDE) {
      const long long kk = ((long long)h << 32) | (uint32_t)cc;
      L.key[r] = kk > L.key[r] ? kk : L.key[r];
    } else {
      L.key[r] = __viaddmax_s32(ho, cc + OPEN, L.key[r]);
    }
  }
  L.botHo = L.Ho[R - 1];
  L.botF = F;
  if (has_below && lane == 31 && valid) bnd[c] = make_int2(L.botHo, L.botF);
}

constexpr int kScoreUnroll = 8;  // steps per unrolled chunk (one 32-B row-checkpoint sector)

template <int R, int MODE, bool WIDE>
__device__ __forceinline__ ScoreOut score_pair(uint8_t *prof, const int8_t *mat, const View rows,
                                               const View cols, const int m, const int n,
                                               const int32_t open_, const int32_t ext,
                                               const int32_t best_known, int2 *bnd,
                                               const int lane, const bool top_from_bnd = false) {
  constexpr int SH = WIDE ? 0 : 16;
  const int32_t OPEN = open_ << SH;
  const int32_t nEXT = -(ext << SH);
  // Reverse pass (MODE 1) = SW on the reversed prefixes ANCHORED at the end
  // cell: only paths that start at reversed (0, 0) count (SURVEY App. A.6:
  // same set of cells reaching best as the local version).  No 0-restarts:
  // H = max(D, E, F, FLOOR), -inf boundaries except the anchor.  The floor
  // keeps the scaled int32 intermediates from wrapping; it cannot change the
  // set of cells == best (a restart at FLOOR reaches at most FLOOR + best <
  // best); it sits 168 above the int32 limit of the scaled domain so that
  // FLOOR - open - ext and FLOOR + s (s >= -128, the virtual cells) cannot
  // wrap.  Every proper suffix of an optimal alignment scores > 0, so the
  // optimal paths cross each row in H > 0 or, inside a gap, E/F > ext - open:
  // once a strip's bottom row (all that feeds the strips below) has H <= 0
  // and F <= ext - open everywhere, no later strip holds a cell == best and
  // the pass stops.  Random long pairs die within a strip or two.
  const int32_t FLOOR = WIDE ? -(1 << 28)
                             : (int32_t)max(-32600, -32766 + open_ + ext) * 65536;
  const int32_t ANC = FLOOR - OPEN;              // -inf in (H - open) form
  ScoreOut res{0ull, 0, 0, 0};
  const int nstrips = (m + 32 * R - 1) / (32 * R);
  int stop_above = n;   // MODE 1: the row above is dead from this column on (k_score_cta)
  for (int strip = 0; strip < nstrips; ++strip) {
    const int row0 = strip * 32 * R;
    __syncwarp();
    build_profile<R>(prof, mat, rows, m, row0, lane);
    __syncwarp();
    ScoreLane<R, WIDE> L;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      L.Ho[r] = MODE == 1 ? ANC : -OPEN;
      L.E[r] = MODE == 1 ? ANC : kNegInf;
      L.key[r] = 0;
    }
    L.hoUpPrev = (MODE == 1 && !(strip == 0 && lane == 0)) ? ANC : -OPEN;   // anchor: H(0,0) = 0
    L.botHo = MODE == 1 ? ANC : -OPEN;
    L.botF = MODE == 1 ? ANC : kNegInf;
    L.code_next = lane == 0 ? cols.at(0) : kPad;
    // top_from_bnd: the first strip's row above is given in bnd (a replay of
    // rows below a saved boundary row, k_jend)
    const bool has_above = strip > 0 || top_from_bnd, has_below = strip + 1 < nstrips;
    BoundaryReader br;
    const int2 dflt = MODE == 1 ? make_int2(ANC, ANC) : make_int2(-OPEN, kNegInf);
    bool alive = false;   // MODE 1: does the strip's bottom row still carry a live path?
    if (has_above) br.init(bnd, MODE == 1 ? min(n, stop_above) : n, lane, dflt);
    const int steps = n + 31;
    int stop = n;
    for (int s0 = 0; s0 < steps; s0 += kScoreUnroll) {
      if constexpr (MODE == 0) {
        // k_jend (best_known = the pair's best, rows up to i_end): every row
        // above i_end stays below best, so the first cell reaching best is
        // (i_end, j_end) and later columns cannot change the row-major-first
        // argmax -- stop there
        if (best_known > 0 && (s0 & 31) == 0 && s0 > 0) {
          bool hit = false;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            if constexpr (WIDE) hit |= (int32_t)(L.key[r] >> 32) >= best_known;
            else hit |= (L.key[r] >> 16) >= best_known;
          }
          if (__any_sync(0xffffffffu, hit)) break;
        }
      }
      if constexpr (MODE == 1) {
        // horizontal stop (see k_score_cta): the wavefront and the row above
        // right of lane 0 are dead -> nothing right of it can equal best
        if ((s0 & 31) == 0 && s0 > 0 && (!has_above || stop_above <= s0)) {
          bool live = (L.hoUpPrev > -OPEN) | (L.botF > -OPEN - nEXT);
#pragma unroll
          for (int r = 0; r < R; ++r) live |= __viaddmax_s32(L.E[r], nEXT, L.Ho[r]) > -OPEN;
          if (__all_sync(0xffffffffu, !live)) { stop = max(0, s0 - 31); break; }
        }
      }
#pragma unroll 2
      for (int q = 0; q < kScoreUnroll; ++q) {
        score_step<R, MODE, WIDE>(L, prof, cols, s0 + q, n, lane, has_above, has_below, br, bnd,
                                  dflt, OPEN, nEXT, FLOOR);
        if constexpr (MODE == 1) {
          const int cb = s0 + q - 31;   // lane 31's column (the strip's bottom row)
          alive |= (cb >= 0) & (cb < n) & ((L.botHo > -OPEN) | (L.botF > -OPEN - nEXT));
        }
      }
    }
    // strip reduction
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int x = row0 + lane * R + r;
      if (x >= m) continue;
      int32_t v, lo;
      if constexpr (WIDE) { v = (int32_t)(L.key[r] >> 32); lo = (int32_t)(L.key[r] & 0xFFFF); }
      else { v = L.key[r] >> 16; lo = L.key[r] & 0xFFFF; }
      res.vmax = v > res.vmax ? v : res.vmax;
      if (MODE == 0) {
        const uint64_t comp = ((uint64_t)(uint32_t)v << 32) | ((uint64_t)(0xFFFF - x) << 16) |
                              (uint64_t)lo;
        res.fwd = comp > res.fwd ? comp : res.fwd;
      } else {
        if (v >= best_known && lo >= 1) {  // v <= best always; avoid == on a max
          res.rev_x = x + 1 > res.rev_x ? x + 1 : res.rev_x;
          res.rev_y = lo > res.rev_y ? lo : res.rev_y;
        }
      }
    }
    if constexpr (MODE == 1) {
      if (!__shfl_sync(0xffffffffu, (int)alive, 31)) break;   // no optimal path below
      stop_above = stop;
    }
  }
  // warp reduction
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t f = __shfl_xor_sync(0xffffffffu, res.fwd, o);
    res.fwd = f > res.fwd ? f : res.fwd;
    const int32_t x = __shfl_xor_sync(0xffffffffu, res.rev_x, o);
    res.rev_x = x > res.rev_x ? x : res.rev_x;
    const int32_t y = __shfl_xor_sync(0xffffffffu, res.rev_y, o);
    res.rev_y = y > res.rev_y ? y : res.rev_y;
    const int32_t v = __shfl_xor_sync(0xffffffffu, res.vmax, o);
    res.vmax = v > res.vmax ? v : res.vmax;
  }
  return res;
}

__device__ __forceinline__ void load_matrix(int8_t *smat, const int8_t *mat) {
  for (int i = threadIdx.x; i < kCodes * kCodes; i += blockDim.x) smat[i] = mat[i];
  __syncthreads();
}

template <int R, int MODE, bool WIDE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_score(KArgs A, int stage, int cls) {
  extern __shared__ __align__(16) uint8_t smem[];
  int8_t *smat = reinterpret_cast<int8_t *>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t *prof = smem + kMatBytes + warp * kProfBytes;
  load_matrix(smat, A.mat);
  const uint64_t gwarp = (uint64_t)blockIdx.x * kWarpsPerBlock + warp;
  int2 *bnd = A.bnd + gwarp * A.bnd_stride;
  for (;;) {
    const int64_t k = next_item(A, stage, cls, lane);
    if (k < 0) break;
    const sw_pair_t p = A.pairs[k];
    PairState *st = A.st + k;
    if (MODE == 0) {
      const View rows{A.codes + p.a_off, 1}, cols{A.codes + p.b_off, 1};
      const ScoreOut o = score_pair<R, 0, WIDE>(prof, smat, rows, cols, (int)p.a_len,
                                                 (int)p.b_len, A.open_, A.ext, 0, bnd, lane);
      if (lane == 0) {
        const int32_t best = (int32_t)(o.fwd >> 32);
        const int32_t i_end = 0xFFFF - (int32_t)((o.fwd >> 16) & 0xFFFF);
        const int32_t j_end = 65535 - (int32_t)(o.fwd & 0xFFFF);
        if (!WIDE && o.vmax >= kScaledLimit) {
          st->flags = kFlagWide;
          list_push(A, 3, 0, (uint32_t)k);
        } else {
          st->best = best;
          st->i_end = best > 0 ? i_end : -1;
          st->j_end = best > 0 ? j_end : -1;
          st->flags = WIDE ? kFlagWide : 0;
          if (best > 0) {
            // The reverse pass only pays when it can shrink the traceback box
            // well below the prefix [0..i_end]x[0..j_end].  A homolog's box is
            // ~(best/3.5)^2 cells; when that is over half the prefix, use the
            // prefix itself as the box (exact either way: box lemma with
            // i0 = j0 = 0).  Pure performance choice.
            const uint64_t area = (uint64_t)(i_end + 1) * (uint64_t)(j_end + 1);
            const bool skip_rev = WIDE || (uint64_t)best * best * 8ull > 49ull * area;
            if (skip_rev) {
              st->i0 = 0;
              st->j0 = 0;
              list_push(A, 2, class_of(i_end + 1), (uint32_t)k);
            } else {
              list_push(A, 1, long_class(i_end + 1), (uint32_t)k);
            }
          }
        }
      }
    } else {
      const int32_t i_end = st->i_end, j_end = st->j_end, best = st->best;
      const View rows{A.codes + p.a_off + i_end, -1}, cols{A.codes + p.b_off + j_end, -1};
      const ScoreOut o = score_pair<R, 1, WIDE>(prof, smat, rows, cols, i_end + 1, j_end + 1,
                                                 A.open_, A.ext, best, bnd, lane);
      if (lane == 0) {
        const int32_t i0 = i_end + 1 - o.rev_x, j0 = j_end + 1 - o.rev_y;
        st->i0 = i0;
        st->j0 = j0;
        list_push(A, 2, class_of(i_end - i0 + 1), (uint32_t)k);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K3: box fill with 4-bit traceback codes, plain int32.
// nibble = Hsrc | Fopen << 2 | Eopen << 3, Hsrc: 0 stop (h==0), 1 diag,
// 2 up (h==F), 3 left (align.py:137-149 priority order).
// Code layout per pair: [strip][lane][step][box_lane_bytes(R)], steps padded
// to a multiple of box_steps_per_store(R) so every lane writes whole 16-byte
// words; a diagonal or horizontal walk step then stays inside the same
// 32-byte sector for several steps, a vertical one inside the same word.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int box_steps_per_store(int R) { return 16 / box_lane_bytes(R); }
__host__ __device__ inline int box_padded_steps(int n, int R) {
  const int f = box_steps_per_store(R);
  return (n + 31 + f - 1) / f * f;
}

template <int R, bool KEY>
struct BoxLane {
  int32_t Ho[R], E[R];
  int32_t key[KEY ? R : 1];
  int32_t hoUpPrev, botHo, botF;
  int code_next;
};

// One wavefront step of the box fill; returns the lane's R nibbles.
// SCALED: values held as v << 16 (fused pass, with the per-row argmax key);
// otherwise plain int32.
template <int R, bool SCALED>
__device__ __forceinline__ uint2 box_step(BoxLane<R, SCALED> &L, const uint8_t *prof,
                                          const View &cols, int s, int n, int lane, bool has_above,
                                          bool has_below, BoundaryReader &br, int2 *bnd,
                                          const int2 dflt, const int32_t OPEN, const int32_t EXT,
                                          const bool fwd_key) {
  const int c = s - lane;
  const bool valid = (c >= 0) & (c < n);
  const int code = L.code_next;
  {
    const int cn = c + 1;
    L.code_next = (cn >= 0 && cn < n) ? cols.at(cn) : kPad;
  }
  const uint4 pw = *reinterpret_cast<const uint4 *>(prof + code * kProfStride + lane * kLaneBytes);
  int32_t upHo = __shfl_up_sync(0xffffffffu, L.botHo, 1);
  int32_t upF = __shfl_up_sync(0xffffffffu, L.botF, 1);
  if (has_above) {
    const int2 b = br.get(bnd, s, n, lane, dflt);
    if (lane == 0) { upHo = b.x; upF = b.y; }
  } else if (lane == 0) {
    upHo = -OPEN; upF = kNegInf;
  }
  int32_t cc = 0;
  if (SCALED && valid) cc = fwd_key ? 65535 - c : c + 1;
  const int32_t ccx = cc + OPEN;
  int32_t diag = L.hoUpPrev;
  L.hoUpPrev = upHo;
  int32_t F = upF, hoUp = upHo;
  uint32_t lo = 0u, hi = 0u;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int32_t sc = (int32_t)prmt(word_of(pw, r), 0u, SCALED ? sel_scaled(r & 3) : sel_plain(r & 3));
    const int32_t ee = L.E[r] - EXT, hl = L.Ho[r];
    const int32_t e = max(ee, hl);
    const int32_t ff = F - EXT;
    const int32_t f = max(ff, hoUp);
    const int32_t D = diag + sc + OPEN;
    // NB: never test `x == max(...)`: ptxas 12.9 for sm_100a folds such
    // equalities into the VIMNMX predicate with the wrong polarity
    // (tools/selftest/max_pred.cu).  Decide from the max's inputs instead.
    const int32_t t = __vimax_s32_relu(D, e);  // max(D, e, 0)
    const int32_t h = max(t, f);
    const bool zero = (D <= 0) & (e <= 0) & (f <= 0);
    const bool dg = (D >= e) & (D >= f);
    const bool up = f >= t;
    const uint32_t src = zero ? 0u : (dg ? 1u : (up ? 2u : 3u));
    const uint32_t nib = src | (hoUp >= ff ? 4u : 0u) | (hl >= ee ? 8u : 0u);
    if (r < 8) lo |= nib << (4 * r);
    else hi |= nib << (4 * (r - 8));
    L.E[r] = e;
    F = f;
    diag = hl;
    const int32_t ho = h - OPEN;
    L.Ho[r] = ho;
    hoUp = ho;
    if constexpr (SCALED) L.key[r] = __viaddmax_s32(ho, ccx, L.key[r]);
  }
  L.botHo = hoUp;
  L.botF = F;
  if (has_below && lane == 31 && valid) bnd[c] = make_int2(L.botHo, L.botF);
  return make_uint2(lo, hi);
}

// K3 (FUSED=false): box [i0..i_end]x[j0..j_end] of a pair whose end cell is
//   known, plain int32, codes only.
// K1c (FUSED=true): the whole matrix of a short/medium pair in the scaled
//   domain: forward score + row-major-first end cell (as k_score<FWD>) AND the
//   traceback codes in one pass, so such pairs need neither K2 nor K3.
template <int R, bool FUSED>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
k_box(KArgs A, int stage, int cls) {
  extern __shared__ __align__(16) uint8_t smem[];
  int8_t *smat = reinterpret_cast<int8_t *>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t *prof = smem + kMatBytes + warp * kProfBytes;
  load_matrix(smat, A.mat);
  const uint64_t gwarp = (uint64_t)blockIdx.x * kWarpsPerBlock + warp;
  int2 *bnd = A.bnd + gwarp * A.bnd_stride;
  constexpr int BPL = box_lane_bytes(R);
  constexpr int SPS = box_steps_per_store(R);
  constexpr int SH = FUSED ? 16 : 0;
  const int32_t OPEN = A.open_ << SH, EXT = A.ext << SH;
  for (;;) {
    const int64_t k = next_item(A, stage, cls, lane);
    if (k < 0) break;
    const sw_pair_t p = A.pairs[k];
    PairState *st = A.st + k;
    int i0 = 0, j0 = 0, m, n;
    if (FUSED) {
      m = (int)p.a_len;
      n = (int)p.b_len;
    } else {
      i0 = st->i0;
      j0 = st->j0;
      m = st->i_end - i0 + 1;
      n = st->j_end - j0 + 1;
    }
    const int nstrips = (m + 32 * R - 1) / (32 * R);
    const int spad = box_padded_steps(n, R);
    const uint64_t bytes = (uint64_t)nstrips * 32 * spad * BPL;
    unsigned long long off = 0;
    if (lane == 0) off = atomicAdd(A.pool_top, (unsigned long long)bytes);
    off = __shfl_sync(0xffffffffu, off, 0);
    const bool fits = off + bytes <= A.pool_cap;
    if (!fits && !FUSED) {
      if (lane == 0) {
        st->flags |= kFlagRetry;
        list_push(A, 5, 0, (uint32_t)k);
      }
      continue;
    }
    const View rows{A.codes + p.a_off + i0, 1}, cols{A.codes + p.b_off + j0, 1};
    uint64_t fwd = 0ull;
    int32_t vmax = 0;
    for (int strip = 0; strip < nstrips; ++strip) {
      const int row0 = strip * 32 * R;
      __syncwarp();
      build_profile<R>(prof, smat, rows, m, row0, lane);
      __syncwarp();
      BoxLane<R, FUSED> L;
#pragma unroll
      for (int r = 0; r < R; ++r) { L.Ho[r] = -OPEN; L.E[r] = kNegInf; }
      if constexpr (FUSED) {
#pragma unroll
        for (int r = 0; r < R; ++r) L.key[r] = 0;
      }
      L.hoUpPrev = -OPEN; L.botHo = -OPEN; L.botF = kNegInf;
      L.code_next = lane == 0 ? cols.at(0) : kPad;
      const bool has_above = strip > 0, has_below = strip + 1 < nstrips;
      BoundaryReader br;
      const int2 dflt = make_int2(-OPEN, kNegInf);
      if (has_above) br.init(bnd, n, lane, dflt);
      uint4 *out = reinterpret_cast<uint4 *>(A.pool + off +
                                             ((uint64_t)strip * 32 + lane) * spad * BPL);
      for (int s0 = 0; s0 < spad; s0 += SPS) {
        uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int q = 0; q < SPS; ++q) {
          const uint2 v = box_step<R, FUSED>(L, prof, cols, s0 + q, n, lane, has_above, has_below,
                                             br, bnd, dflt, OPEN, EXT, true);
          if (BPL == 8) { w[2 * q] = v.x; w[2 * q + 1] = v.y; }
          else if (BPL == 4) { w[q] = v.x; }
          else { w[q >> 1] |= (v.x & 0xFFFFu) << (16 * (q & 1)); }
        }
        if (fits) out[s0 / SPS] = make_uint4(w[0], w[1], w[2], w[3]);
      }
      if constexpr (FUSED) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int x = row0 + lane * R + r;
          if (x >= m) continue;
          const int32_t v = L.key[r] >> 16, lo = L.key[r] & 0xFFFF;
          vmax = v > vmax ? v : vmax;
          const uint64_t comp = ((uint64_t)(uint32_t)v << 32) |
                                ((uint64_t)(0xFFFF - x) << 16) | (uint64_t)lo;
          fwd = comp > fwd ? comp : fwd;
        }
      }
    }
    if constexpr (FUSED) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t f2 = __shfl_xor_sync(0xffffffffu, fwd, o);
        fwd = f2 > fwd ? f2 : fwd;
        const int32_t v2 = __shfl_xor_sync(0xffffffffu, vmax, o);
        vmax = v2 > vmax ? v2 : vmax;
      }
    }
    if (lane == 0) {
      if (FUSED) {
        const int32_t best = (int32_t)(fwd >> 32);
        const int32_t i_end = 0xFFFF - (int32_t)((fwd >> 16) & 0xFFFF);
        const int32_t j_end = 65535 - (int32_t)(fwd & 0xFFFF);
        st->i0 = 0;
        st->j0 = 0;
        if (vmax >= kScaledLimit) {           // re-run in the wide score path
          st->flags = kFlagWide;
          list_push(A, 3, 0, (uint32_t)k);
        } else {
          st->best = best;
          st->i_end = best > 0 ? i_end : -1;
          st->j_end = best > 0 ? j_end : -1;
          if (fits) {
            st->flags = 0;
            st->code_off = off;
            st->box_cls = cls;
            st->box_m = m;
            st->box_n = n;
          } else if (best > 0) {              // no room for codes: prefix box via K3
            st->flags = kFlagRetry;
            list_push(A, 5, 0, (uint32_t)k);
          } else {
            st->flags = 0;
          }
        }
      } else {
        st->code_off = off;
        st->box_cls = cls;
        st->box_m = m;
        st->box_n = n;
        st->flags &= ~kFlagRetry;
      }
    }
  }
}

__device__ __forceinline__ int box_rows_of(int cls) { return class_rows(cls); }

__device__ __forceinline__ uint32_t code_at(const uint8_t *codes, int R, int BPL, int spad, int rho,
                                            int kap) {
  const int strip = rho / (32 * R);
  const int rr = rho - strip * 32 * R;
  const int t = rr / R, r = rr - t * R;
  const int s = kap + t;
  const uint8_t b = codes[(((uint64_t)strip * 32 + t) * spad + s) * BPL + (r >> 1)];
  return (r & 1) ? (uint32_t)(b >> 4) : (uint32_t)(b & 15u);
}

// ---------------------------------------------------------------------------
// K5: tile traceback for pairs whose forward pass wrote checkpoints.
// One warp per pair walks the state machine of align.py:133-169 backwards
// from the end cell.  The H/E/F values it needs are produced on demand for one
// tile at a time -- the rows of one lane group (G = 32/R forward lanes, <= 32
// rows, one row per replay lane) over one 32-step forward window -- by
// replaying the forward recurrence from the checkpoints into a shared-memory
// tile with a one-cell halo (row above, column left).  Only the tiles on the
// path are replayed, and only their part the walk can still reach (rows up to
// and columns up to the entry cell; the walk only moves up/left).  The walk is
// warp-uniform and compares loaded values exactly as the reference does.
// ---------------------------------------------------------------------------
constexpr int kTbWarps = 4;
// residue bytes of a tile: read-only during K5 and reused by neighbouring
// tiles, so through L1 (A/B against L1-bypassing loads: +0.5 % config 3)
#define LD5 __ldg
constexpr int16_t kNeg16 = -16384;  // boundary "-inf": below -open - ext for open <= 16383

// Tile of class R: rows = G*R replayed + 1 halo, columns = G + 32 (halo +
// 32 columns of the first forward lane + G - 1 skew), G = 32 / R.
template <int R>
struct TbSmem {
  static constexpr int G = 32 / R;
  static constexpr int kRows = G * R + 1;
  static constexpr int kX = (G + 32 + 1) / 2 * 2;
  // per cell: H (bits 0-15, 0 <= H <= kTileMax) | (F + open) << 16 (-open <= F <= H).
  // The walk needs F and E only to enter a gap state and, inside a gap run,
  // as entry value + k * ext (a run that has not closed extends: F(i-1) =
  // F(i) + ext); a cell that is neither a diagonal move nor H == F has H == E
  // (H = max(D, E, F, 0)), so E is not stored at all.
  uint32_t H[kRows][kX];  // row 0 / col 0 = halo
  int4 row[32];         // per tile row: E at c_lo, H at c_lo - 1, matrix row, diag above / F_bot
  uint8_t bcode[kX], braw[kX];
  uint8_t acode[32], araw[32];
};

template <int R>
__device__ __forceinline__ int32_t tH(const TbSmem<R> &T, int row, int col) {
  return (int32_t)(T.H[row][col] & 0xFFFFu);
}

// checkpoint words hold two biased u16 values (v + B)
__device__ __forceinline__ int32_t ulo(uint32_t x, int32_t B) { return (int32_t)(x & 0xFFFFu) - B; }
__device__ __forceinline__ int32_t uhi(uint32_t x, int32_t B) { return (int32_t)(x >> 16) - B; }

template <int R>
__device__ __forceinline__ void tb_replay(TbSmem<R> &T, const int8_t *smat, const uint8_t *slut,
                                          const uint32_t *ck,
                                          const uint2 *rowck, int hi,
                                          const CkLayout &CL, int strip, int g, int w, int m,
                                          int n, const RawView &acodes, const RawView &bcodes,
                                          const uint8_t *araw, const uint8_t *braw, int lane,
                                          int32_t OPEN, int32_t EXT, int32_t B, int &trow0,
                                          int &tcmin, const int rho_in, const int kap_in) {
  const int t0 = g * CL.G;
  const int t1 = min(t0 + CL.G, 32) - 1;
  trow0 = strip * 32 * R + t0 * R;
  const int cmin = 32 * w - t1;              // tile column index x = c - cmin + 1
  const int width = 32 + (t1 - t0);
  tcmin = cmin;
  // the walk enters at (rho_in, kap_in) and only moves up/left
  const int qmax = rho_in - trow0;
  const int q = lane;
  const bool row_ok = q <= qmax;
  const int tq = t0 + q / R, rq = q - (q / R) * R;
  const int rho = trow0 + q;
  const bool real_row = row_ok & (rho < m);
  const uint32_t *sbase = ck + (uint64_t)strip * CL.col_words;
  // row checkpoints of boundary b in strip st: (Ho2, F2) u16x2 words per step,
  // this pair's half selected by `hi`
  auto rowp = [&](int st, int b) -> const uint2 * {
    return rowck + ((uint64_t)st * CL.row_words + (uint64_t)b * 2 * CL.spad) / 2;
  };
  // Issue every global load of the set-up first (residue bytes of the tile's
  // columns and rows, this row's column checkpoint, the top halo row) so their
  // latencies overlap, then the LUT lookups, then the shared-memory stores.
  const int c0 = cmin + lane, c1 = cmin + 32 + lane;
  const bool ok0 = (c0 >= 0) & (c0 < n), ok1 = (32 + lane < width) & (c1 >= 0) & (c1 < n);
  const uint8_t rb0 = ok0 ? LD5(braw + c0) : (uint8_t)0;
  const uint8_t rb1 = ok1 ? LD5(braw + c1) : (uint8_t)0;
  const uint8_t ra = real_row ? LD5(araw + rho) : (uint8_t)0;
  uint32_t ckx = 0u, cky = 0u;
  const bool have_ck = (w > 0) & row_ok;
  if (have_ck) {
    const uint32_t *wd = sbase + (uint64_t)w * 32 * ck_words(R) + tq;
    ckx = wd[32 * rq];
    cky = wd[32 * R];
  }
  const uint2 *toprow = nullptr;
  int tsrc = 0;
  if (t0 > 0) {
    toprow = rowp(strip, ck_boundary(t0 - 1, CL));
    tsrc = t0 - 1;
  } else if (strip > 0) {
    toprow = rowp(strip - 1, CL.nb - 1);
    tsrc = 31;
  }
  const int tidx = 32 * w - t0 + lane + tsrc;
  const bool have_top = toprow && tidx >= 0;
  uint2 z = make_uint2(0u, 0u);
  if (have_top) z = toprow[tidx];
  const uint8_t bc0 = ok0 ? slut[rb0] : (uint8_t)kPad;   // shared-memory LUT
  const uint8_t bc1 = ok1 ? slut[rb1] : (uint8_t)kPad;
  const int acode = real_row ? (int)slut[ra] : kPad;
  __syncwarp();
  T.bcode[lane] = bc0;
  T.braw[lane] = rb0;
  if (32 + lane < width) {
    T.bcode[32 + lane] = bc1;
    T.braw[32 + lane] = rb1;
  }
  if (row_ok) {
    T.acode[q] = (uint8_t)acode;
    T.araw[q] = ra;
  }
  int32_t Ho = -OPEN, E = kNeg16, hoUpPrevT = -OPEN, FbotT = kNeg16;
  if (have_ck) {
    Ho = ulo(ckx, B);
    E = uhi(ckx, B);
    hoUpPrevT = ulo(cky, B);
    FbotT = uhi(cky, B);
  }
  // halo: this row's left boundary (column c_lo - 1) and, for the first row of
  // each forward lane, the diagonal above it (column c_lo - 1 of the row above)
  const int x0 = t1 - tq;                    // tile column of c_lo(q) - 1
  if (row_ok) {
    T.H[q + 1][x0] = (uint32_t)(Ho + OPEN);
    if (rq == 0) T.H[q][x0] = (uint32_t)(hoUpPrevT + OPEN);
  }
  // top halo row: H of the row above the tile at columns c_lo(t0) .. +31;
  // lane l also keeps (Ho, F) of column c_lo(t0) + l packed for row 0's feed
  uint32_t topv;
  {
    int32_t tHo = -OPEN, tF = kNeg16;
    if (have_top) {
      tHo = (int32_t)(hi ? (z.x >> 16) : (z.x & 0xFFFFu)) - B;
      tF = (int32_t)(hi ? (z.y >> 16) : (z.y & 0xFFFFu)) - B;
    }
    T.H[0][t1 - t0 + 1 + lane] = (uint32_t)(tHo + OPEN);
    topv = ((uint32_t)tHo & 0xFFFFu) | ((uint32_t)tF << 16);
  }
  // (An L2 prefetch of the checkpoint lines of the tiles the walk can go to
  // next -- left and up -- was 1-2 % slower on configs 2/3 in round 2.)
  // Column-parallel replay: lane l owns column c_lo(row) + l and the warp
  // steps down the tile one row at a time (no wavefront skew).  Per row:
  //   F  = max(F_up - ext, H_up - open)            (vertical, from the row above)
  //   Ht = max(0, H_diag + s, F)                     (H without the horizontal term)
  //   E  = horizontal gap, exactly E[l] = max(E[l-1] - ext, H[l-1] - open), as a
  //        max-plus prefix scan over the lanes: with open >= ext,
  //        E[l] + l*ext = max(E[0], max_{l'<l} Ht[l'] - open + (l'+1)*ext)
  //   H  = max(Ht, E)
  // Rows of forward lane t cover columns 32w - t + [0, 32): entering the next
  // forward lane shifts the columns left by one, so the row above is shifted
  // one lane up; its lane-0 cell and the diagonal come from the checkpoints.
  if (row_ok)
    T.row[q] = make_int4(max(E - EXT, Ho),         // E at c_lo (left boundary)
                         Ho + OPEN,                 // H at c_lo - 1
                         acode * kCodes,            // matrix row of the residue
                         rq == 0 ? hoUpPrevT + OPEN // first row: the diagonal above c_lo - 1
                                 : FbotT);          // (last row: F at c_lo - 1)
  int32_t upH = (int32_t)(int16_t)(topv & 0xFFFFu) + OPEN, upF = (int32_t)topv >> 16;
  int32_t prevHb = 0, prevFb = kNeg16;   // H / F of the previous row at ITS c_lo - 1
  const int32_t Kl = (lane + 1) * EXT - OPEN, lext = lane * EXT;
  __syncwarp();
  for (int tb = t0, qs = 0; qs <= qmax; ++tb, qs += R) {   // forward lanes of the tile
    if (qs > 0) {                           // columns shift left by one: row above one lane up
      const int32_t sh = __shfl_up_sync(0xffffffffu, upH, 1);
      const int32_t sf = __shfl_up_sync(0xffffffffu, upF, 1);
      upH = lane == 0 ? prevHb : sh;
      upF = lane == 0 ? prevFb : sf;
    }
    const int xs = (t1 - tb) + 1 + lane;    // tile column of this lane's cell
    const int8_t *mcol = smat + T.bcode[xs - 1];
    const int nr = min(R, qmax + 1 - qs);   // rows of this forward lane to replay
    auto row_step = [&](const int r) {
      const int qq = qs + r;
      const int4 rw = T.row[qq];             // broadcast
      int32_t dg = __shfl_up_sync(0xffffffffu, upH, 1);
      if (lane == 0) dg = r == 0 ? rw.w : prevHb;
      const int32_t sc = mcol[rw.z];
      const int32_t f = max(upF - EXT, upH - OPEN);
      const int32_t ht = __vimax3_s32_relu(dg + sc, f, 0);
      int32_t z = ht + Kl;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) z = max(z, (int32_t)__shfl_up_sync(0xffffffffu, z, d));
      const int32_t x0e = rw.x;                             // E at c_lo (left boundary)
      int32_t ex = __shfl_up_sync(0xffffffffu, z, 1);
      if (lane == 0) ex = x0e;
      const int32_t e = max(x0e, ex) - lext;
      const int32_t h = max(ht, e);
      T.H[qq + 1][xs] = (uint32_t)(h + (OPEN << 16)) + ((uint32_t)f << 16);   // h | (f + open) << 16
      upH = h;
      upF = f;
      prevHb = rw.y;
      prevFb = rw.w;                         // used after the forward lane's last row
    };
    if (nr == R) {                           // whole forward lane: no per-row exit test
#pragma unroll
      for (int r = 0; r < R; ++r) row_step(r);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (r >= nr) break;
        row_step(r);
      }
    }
  }
  __syncwarp();
}

#ifdef K5_COUNT
__device__ unsigned long long g_k5c[8];   // debug: pairs, j tiles, j rows, walk tiles, walk rows, aln, iters
#define K5C(i, v) do { if (lane == 0) atomicAdd(&g_k5c[i], (unsigned long long)(v)); } while (0)
#else
#define K5C(i, v) do { } while (0)
#endif
// Traceback of one pair whose packed forward pass wrote checkpoints
// (PairState: best, i_end, code_off, box_n, flags & kFlagNeedJ); one warp.
template <int R>
__device__ __forceinline__ void tb_pair(const KArgs &A, TbSmem<R> &T, const int8_t *smat,
                                        const uint8_t *slut, int64_t k, int lane) {
  const int32_t OPEN = A.open_, EXT = A.ext, Bias = A.bias16;
  const sw_pair_t p = A.pairs[k];
  PairState *st = A.st + k;
  const int m = (int)p.a_len, n = (int)p.b_len;
  const CkLayout CL = ck_layout(R, st->box_n);   // layout of the forward pass's checkpoints
  const uint32_t *ck = reinterpret_cast<const uint32_t *>(A.pool + st->code_off);
  const uint2 *rowck = reinterpret_cast<const uint2 *>(A.pool + st->code_off + st->row_delta);
  const int hi = (st->flags & kFlagHi) ? 1 : 0;
  const uint8_t *araw = A.raw + p.a_off, *braw = A.raw + p.b_off;
  const RawView acodes{araw, A.lut}, bcodes{braw, A.lut};
  const int i_end = st->i_end;
  int j_end = st->j_end;
  int cs = -1, cg = -1, cw = -1, trow0 = 0, tcmin = 0, tqmax = -1;
  if (st->flags & kFlagNeedJ) {
    // The packed forward pass knows best and i_end only.  j_end = first
    // column of row i_end with H == best (align.py:124).  The checkpoints
    // hold, per window, the running maximum over the R rows of each lane: the
    // first window where the lane of row i_end reaches best is the earliest
    // row i_end can; the tiles of row i_end are replayed from there until the
    // row reaches best (a second replay only when a later row of the same
    // lane reached best first).
    const int best = st->best;
    const int strip = i_end / (32 * R);
    const int t = (i_end - strip * 32 * R) / R;
    const uint32_t *lmcol = ck + (uint64_t)strip * CL.col_words + 32ull * (R + 1) + t;
    int wstar = CL.nwin - 1;
    for (int w0 = 1; w0 < CL.nwin; w0 += 32) {
      const int w = w0 + lane;
      bool hit = false;
      if (w < CL.nwin) hit = (int32_t)(lmcol[(uint64_t)w * 32 * ck_words(R)] & 0xFFFFu) - Bias >= best;
      const uint32_t hm = __ballot_sync(0xffffffffu, hit);
      if (hm) { wstar = w0 + __ffs(hm) - 1 - 1; break; }
    }
    const int g = t / CL.G;
    for (; wstar < CL.nwin; ++wstar) {
      const int kap_hi = min(32 * wstar - t + 31, n - 1);
      if (32 * wstar - t > kap_hi) continue;
      tb_replay<R>(T, smat, slut, ck, rowck, hi, CL, strip, g, wstar, m, n, acodes, bcodes, araw, braw, lane, OPEN,
                   EXT, Bias, trow0, tcmin, i_end, kap_hi);
      K5C(1, 1); K5C(2, i_end - trow0 + 1);
      cs = strip; cg = g; cw = wstar;
      const int q = i_end - trow0;
      tqmax = q;
      const int c = 32 * wstar - t + lane;
      const bool hit = (c >= 0) && (c <= kap_hi) && (tH(T, q + 1, c - tcmin + 1) >= best);
      const uint32_t hm = __ballot_sync(0xffffffffu, hit);
      if (hm) { j_end = 32 * wstar - t + __ffs(hm) - 1; break; }
    }
  }
  int i = i_end + 1, j = j_end + 1, state = 0, matches = 0, aln = 0;
  int32_t gap = 0;   // state 1/2: F/E of the current cell
  bool lost = j_end < 0;
  for (;;) {
    if (lost) break;
    if (i == 0 || j == 0) {
      lost = state != 0;
      break;
    }
    const int rho = i - 1, kap = j - 1;
    // fast path: still inside the replayed part of the current tile
    int q = rho - trow0;
    const int u = kap - (cw * 32 - (cg * CL.G + q / R));
    if (!(cs >= 0 && q >= 0 && q <= tqmax && u >= 0 && u < 32)) {
      const int strip = rho / (32 * R);
      const int t = (rho - strip * 32 * R) / R;
      const int g = t / CL.G;
      const int w = (kap + t) >> 5;
      tb_replay<R>(T, smat, slut, ck, rowck, hi, CL, strip, g, w, m, n, acodes, bcodes, araw, braw, lane, OPEN,
                   EXT, Bias, trow0, tcmin, rho, kap);
      K5C(3, 1); K5C(4, rho - trow0 + 1);
      cs = strip; cg = g; cw = w;
      q = rho - trow0;
      tqmax = q;
    }
    const int x = kap - tcmin + 1;
    // first tile column of tile row qq (its left halo is at x_first - 1)
    const int t0 = cg * CL.G, tspan = min(t0 + CL.G, 32) - 1 - t0;
    if (state == 0) {                       // align.py:137-151
      // Resolve a diagonal run 32 cells at a time: lane k checks cell
      // (q-k, x-k); the run continues while each cell is an H-state diagonal
      // move (h != 0 and h == H[diag] + s) inside the replayed tile.
      const int qq = q - lane, xx = x - lane;
      bool ok = (qq >= 0) && (kap - lane >= 0);
      ok = ok && (xx >= tspan - qq / R + 1);
      bool dg = false, mt = false;
      if (ok) {
        const int32_t hk = tH(T, qq + 1, xx);
        const int32_t sk = smat[T.acode[qq] * kCodes + T.bcode[xx - 1]];
        dg = (hk != 0) && (hk == tH(T, qq, xx - 1) + sk);
        mt = T.araw[qq] == T.braw[xx - 1];
      }
      const uint32_t run_mask = __ballot_sync(0xffffffffu, dg);
      const uint32_t mt_mask = __ballot_sync(0xffffffffu, mt);
      const int run = (run_mask == 0xffffffffu) ? 32 : __ffs(~run_mask) - 1;
      if (run > 0) {
        const uint32_t sel = run == 32 ? 0xffffffffu : ((1u << run) - 1u);
        matches += __popc(mt_mask & sel);
        aln += run; i -= run; j -= run;
        continue;
      }
      const uint32_t hw = T.H[q + 1][x];
      const int32_t h = (int32_t)(hw & 0xFFFFu);
      if (h == 0) break;
      gap = h;                              // the gap state's value at this cell
      state = h == (int32_t)(hw >> 16) - OPEN ? 1 : 2;   // F first (align.py:145-150), else E
    } else if (state == 1) {                // align.py:152-160: vertical gap run
      const int qq = q - lane;
      const bool ok = (qq >= 0) && (x >= tspan - qq / R + 1);
      const bool close = ok && (gap + lane * EXT == tH(T, qq, x) - OPEN);   // F(qq) == H above - open
      const uint32_t cm = __ballot_sync(0xffffffffu, close);
      const uint32_t vm = __ballot_sync(0xffffffffu, ok);
      const int nvalid = __ffs(~vm) == 0 ? 32 : __ffs(~vm) - 1;
      int steps;
      if (cm) { steps = __ffs(cm); state = 0; }
      else steps = nvalid;
      gap += steps * EXT;
      aln += steps; i -= steps;
    } else {                                // align.py:161-169: horizontal gap run
      const int xx = x - lane;
      const bool ok = (kap - lane >= 0) && (xx >= tspan - q / R + 1);
      const bool close = ok && (gap + lane * EXT == tH(T, q + 1, xx - 1) - OPEN);   // E(xx) == H left - open
      const uint32_t cm = __ballot_sync(0xffffffffu, close);
      const uint32_t vm = __ballot_sync(0xffffffffu, ok);
      const int nvalid = __ffs(~vm) == 0 ? 32 : __ffs(~vm) - 1;
      int steps;
      if (cm) { steps = __ffs(cm); state = 0; }
      else steps = nvalid;
      gap += steps * EXT;
      aln += steps; j -= steps;
    }
  }
  K5C(0, 1); K5C(5, aln);
  if (lane == 0) {
    sw_result_t r;
    r.score = st->best;
    r.i_begin = i; r.i_end = i_end;
    r.j_begin = j; r.j_end = j_end;
    r.matches = matches; r.aln_len = aln;
    r.status = lost ? SW_STATUS_INTERNAL : SW_STATUS_OK;
    A.out[k] = r;
    st->j_end = j_end;
    st->flags |= kFlagDone;
  }
}

// 9 blocks of 4 warps per SM (56 registers, no spills): the replay is latency
// bound, and the u32 tile (no E/F matrices) leaves shared memory for 9 blocks
// at R <= 9.  A/B on B200, config 3 / config 2 full GCUPS: 7 blocks (72
// registers, 3 int16 tiles) 2,447 / 1,850; u32 tile at 7 blocks 2,446 / 1,840;
// 8 blocks 2,531 / 1,892; 9 blocks 2,552 / 1,918; 10 blocks (48 registers,
// spills) 2,493 / 1,892.
#ifndef K5_MIN_BLOCKS
#define K5_MIN_BLOCKS 9
#endif
template <int R>
__global__ void __launch_bounds__(kTbWarps * 32, K5_MIN_BLOCKS)
k_tb(KArgs A, int stage, int cls) {
  struct Shared {
    TbSmem<R> t[kTbWarps];
    int8_t mat[kCodes * kCodes];
    uint8_t lut[256];                   // raw byte -> residue code
  };
  __shared__ __align__(16) Shared sh;   // one shared window base for tiles and matrix
  int8_t *smat = sh.mat;
  for (int i = threadIdx.x; i < kCodes * kCodes; i += blockDim.x) smat[i] = A.mat[i];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sh.lut[i] = A.lut[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  TbSmem<R> &T = sh.t[warp];
  for (;;) {
    const int64_t k = next_item(A, stage, cls, lane);
    if (k < 0) break;
    tb_pair<R>(A, T, smat, sh.lut, k, lane);
  }
}

// K4: traceback walk, one thread per pair (align.py:133-181).
__global__ void k_walk(KArgs A, const uint32_t *only, uint32_t n_only) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t k;
  if (only) {
    if (t >= n_only) return;
    k = only[t];
  } else {
    if (t >= A.n_pairs) return;
    k = t;
  }
  const sw_pair_t p = A.pairs[k];
  PairState *st = A.st + k;
  sw_result_t r;
  r.score = 0; r.i_begin = r.i_end = r.j_begin = r.j_end = -1;
  r.matches = 0; r.aln_len = 0; r.status = SW_STATUS_OK;
  if (A.st[k].flags & kFlagInvalid) {
    r.status = SW_STATUS_INVALID;
    A.out[k] = r;
    return;
  }
  if (p.a_len == 0 || p.b_len == 0) {
    r.status = SW_STATUS_EMPTY;
    A.out[k] = r;
    return;
  }
  const int32_t flags = st->flags;
  if (flags & kFlagDone) return;
  if (flags & kFlagRetry) return;
  if (st->best == 0) {
    A.out[k] = r;
    st->flags = flags | kFlagDone;
    return;
  }
  const int i0 = st->i0, j0 = st->j0;
  const int n = st->box_n;
  const int R = box_rows_of(st->box_cls);
  const int BPL = box_lane_bytes(R);
  const int steps = box_padded_steps(n, R);
  const uint8_t *codes = A.pool + st->code_off;
  const uint8_t *ra = A.raw + p.a_off + i0, *rb = A.raw + p.b_off + j0;
  int i = st->i_end - i0 + 1, j = st->j_end - j0 + 1, state = 0, matches = 0, aln = 0;
  bool lost = false;
  for (;;) {
    if (state == 0) {
      if (i == 0 || j == 0) break;
      const uint32_t nib = code_at(codes, R, BPL, steps, i - 1, j - 1);
      const uint32_t src = nib & 3u;
      if (src == 0u) break;
      if (src == 1u) {
        matches += ra[i - 1] == rb[j - 1];
        ++aln; --i; --j;
      } else {
        state = (int)src - 1;  // 1 F (up), 2 E (left)
      }
    } else if (state == 1) {
      if (i == 0) { lost = true; break; }
      const uint32_t nib = code_at(codes, R, BPL, steps, i - 1, j - 1);
      ++aln; --i;
      if (nib & 4u) state = 0;
    } else {
      if (j == 0) { lost = true; break; }
      const uint32_t nib = code_at(codes, R, BPL, steps, i - 1, j - 1);
      ++aln; --j;
      if (nib & 8u) state = 0;
    }
  }
  r.score = st->best;
  r.i_begin = i0 + i; r.i_end = st->i_end;
  r.j_begin = j0 + j; r.j_end = st->j_end;
  r.matches = matches; r.aln_len = aln;
  r.status = lost ? SW_STATUS_INTERNAL : SW_STATUS_OK;
  A.out[k] = r;
  st->flags = flags | kFlagDone;
}

// Byte -> residue code (align.py:27-30: unknown bytes score as 'X').
// `raw` may sit at any byte address (a caller's device buffer or a slice of
// one); `codes` must have the same address modulo 16 (the caller offsets it),
// so the body moves as aligned 128-bit words and only the unaligned head and
// tail go byte by byte.
__global__ void k_encode(const uint8_t *__restrict__ raw, uint8_t *__restrict__ codes, uint64_t n,
                         const uint8_t *__restrict__ lut) {
  __shared__ uint8_t slut[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) slut[i] = lut[i];
  __syncthreads();
  uint64_t head = (16u - ((uintptr_t)raw & 15u)) & 15u;
  if (head > n) head = n;
  if (blockIdx.x == 0 && threadIdx.x < head) codes[threadIdx.x] = slut[raw[threadIdx.x]];
  raw += head;
  codes += head;
  n -= head;
  const uint64_t n16 = n / 16;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v = reinterpret_cast<const uint4 *>(raw)[i];
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t x = w[q];
      w[q] = (uint32_t)slut[x & 255u] | ((uint32_t)slut[(x >> 8) & 255u] << 8) |
             ((uint32_t)slut[(x >> 16) & 255u] << 16) | ((uint32_t)slut[x >> 24] << 24);
    }
    reinterpret_cast<uint4 *>(codes)[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  for (uint64_t i = n16 * 16 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    codes[i] = slut[raw[i]];
}

// Classify pairs by row count (work list = stage x length class), count the
// lists (warp-aggregated atomics) and emit a sort key per pair:
// (list << 48) | (65535 - m) << 16 | (65535 - n).  A radix sort then orders
// every list by descending shape (largest first; neighbours of the same shape
// for the packed kernel, which aligns two consecutive pairs per warp) and
// k_scatter_lists writes the sorted lists.
constexpr int kNoList = 127;
// sort key = list (7 bits) above the order field: the 32-bit shape order by
// default (a 39-bit key: 5 radix passes), a 48-bit cell count otherwise
__host__ __device__ constexpr int list_key_shift(int sort_cells) { return sort_cells ? 48 : 32; }
__global__ void k_classify(KArgs A, unsigned long long *stats, int allow_ckpt, int packed_ok,
                           unsigned long long *keys, uint32_t *vals, int sort_cells) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned lane = threadIdx.x & 31;
  const bool in = k < A.n_pairs;
  sw_pair_t p;
  p.a_len = 0;
  p.b_len = 0;
  if (in) {
    p = A.pairs[k];
    PairState s;
    s.best = 0; s.i_end = s.j_end = -1; s.flags = 0; s.i0 = s.j0 = 0; s.box_cls = 0;
    s.box_n = 0; s.code_off = 0; s.box_m = 0; s.row_delta = 0;
    // the call's only bounds check (sw_align_batch and the device entry point):
    // a pair outside the arena or longer than 65,000 residues is never
    // scheduled; the call then fails with SW_EINVAL
    if (p.a_off > A.arena_bytes || p.a_len > A.arena_bytes - p.a_off ||   // no u64 wrap
        p.b_off > A.arena_bytes || p.b_len > A.arena_bytes - p.b_off ||
        p.a_off < A.arena_lo || p.b_off < A.arena_lo ||
        p.a_len > 65000u || p.b_len > 65000u) {
      s.flags = kFlagInvalid;
      atomicAdd(&stats[5], 1ull);
      p.a_len = 0;
      p.b_len = 0;
    }
    A.st[k] = s;
  }
  const bool real = in && p.a_len > 0 && p.b_len > 0;
  const uint64_t cells = (uint64_t)p.a_len * p.b_len;
  const bool fused = allow_ckpt && cells <= kFusedMaxCells;
  // short/medium pairs: packed pass, per length class; long pairs: one
  // scalar class (R = 16), so each long-pair phase has a single tail
  const int slot = real ? (fused ? 6 * kNumClasses + packed_class_of((int)p.a_len, (int)p.b_len)
                                   : long_class((int)p.a_len, packed_ok)) : -1;
  const unsigned peers = __match_any_sync(0xffffffffu, slot);
  const int leader = __ffs(peers) - 1;
  if (slot >= 0 && (int)lane == leader) atomicAdd(&A.ctrs[slot], (uint32_t)__popc(peers));
  if (in) {
    // Lists are processed in key order, consecutive pairs sharing a warp (a
    // duo computes max(m) x max(n) of its two pairs).  Packed pairs: by strip
    // count, then n -- duo partners have equal strips and nearly equal n (by
    // m, then n, partners had unrelated n: 2 % more computed cells on config
    // 3, forward -2.4 %); other pairs: by m, then n.
    unsigned long long shape = (((unsigned long long)(0xFFFFu - min(p.a_len, 0xFFFFu)) << 16) |
                                (unsigned long long)(0xFFFFu - min(p.b_len, 0xFFFFu)));
    if (real && fused) {
      const int R = class_rows(packed_class_of((int)p.a_len, (int)p.b_len));
      const uint32_t S = (p.a_len + 32u * R - 1) / (32u * R);
      shape = ((unsigned long long)(0xFFFFu - S) << 16) | (unsigned long long)(0xFFFFu - p.b_len);
    }
    // sort_cells 2 (host-pipelined arenas): the upload slice the pair's bytes
    // end in, then shape -- the packed pass consumes the arena roughly in
    // upload order, so its warps rarely wait for late slices
    unsigned long long order = shape;
    if (sort_cells == 1) order = (0xFFFFFFFFFFFFull - cells) & 0xFFFFFFFFFFFFull;
    if (sort_cells == 2 && A.slice_bytes) {
      const uint64_t end = max(p.a_off + p.a_len, p.b_off + p.b_len);
      const uint64_t chunk = end > A.arena_lo ? (end - A.arena_lo - 1) / A.slice_bytes : 0;
      order = (min(chunk, (uint64_t)0xFFFF) << 32) | shape;
    }
    keys[k] = ((unsigned long long)(slot >= 0 ? slot : kNoList) << list_key_shift(sort_cells)) | order;
    vals[k] = (uint32_t)k;
  }
  unsigned long long c = real ? cells : 0ull;
  unsigned long long mb = real ? p.b_len : 0ull;
  // checkpoint bytes the packed pass will ask for (per pair: its column
  // checkpoints and half of its duo's row checkpoints), so the host can size
  // the pool before the first packed round instead of deferring pairs
  unsigned long long ck = 0ull;
  if (real && fused) {
    const int R = class_rows(packed_class_of((int)p.a_len, (int)p.b_len));
    const CkLayout L = ck_layout(R, (int)p.b_len);
    const unsigned long long strips = (p.a_len + 32u * R - 1) / (32u * R);
    ck = strips * (L.col_words + L.row_words / 2) * 4ull;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    c += __shfl_xor_sync(0xffffffffu, c, o);
    ck += __shfl_xor_sync(0xffffffffu, ck, o);
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, mb, o);
    mb = t > mb ? t : mb;
  }
  if (lane == 0) {
    if (c) atomicAdd(&stats[0], c);
    if (mb) atomicMax(&stats[1], mb);
    if (ck) atomicAdd(&stats[6], ck);
  }
}

// Sorted (key, pair) -> per-list arrays; list offsets are the exclusive
// prefix of the list counts in key order (lists are contiguous in the sort).
__global__ void k_scatter_lists(KArgs A, const unsigned long long *keys, const uint32_t *vals,
                                int key_shift) {
  __shared__ uint32_t off[kStages * kNumClasses];
  if (threadIdx.x == 0) {
    uint32_t acc = 0;
    for (int i = 0; i < kStages * kNumClasses; ++i) {
      off[i] = acc;
      acc += A.ctrs[i];
    }
  }
  __syncthreads();
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < A.n_pairs;
       p += (uint64_t)gridDim.x * blockDim.x) {
    const int slot = (int)(keys[p] >> key_shift);
    if (slot >= kStages * kNumClasses) continue;
    A.lists[(uint64_t)slot * A.n_pairs + (p - off[slot])] = vals[p];
  }
}

// Move retry pairs back into the K3 lists.
__global__ void k_requeue(KArgs A) {
  const uint32_t n = A.ctrs[5 * kNumClasses];
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const uint32_t k = list_of(A, 5, 0)[t];
    list_push(A, 2, class_of(A.st[k].i_end - A.st[k].i0 + 1), k);
  }
}

// Start another packed round: the pairs deferred for lack of checkpoint room
// (stage 8) become the packed input (stage 6) and every other list and cursor
// of the class is emptied.  One block per class.
__global__ void k_packed_round(KArgs A) {
  const int c = blockIdx.x;
  const uint32_t n = A.ctrs[8 * kNumClasses + c];
  const uint32_t *src = list_of(A, 8, c);
  uint32_t *dst = list_of(A, 6, c);
  for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) dst[t] = src[t];
  __syncthreads();
  if (threadIdx.x < kStages) {
    const int stage = threadIdx.x;
    A.ctrs[stage * kNumClasses + c] = stage == 6 ? n : 0u;
    A.ctrs[kStages * kNumClasses + stage * kNumClasses + c] = 0u;
  }
}

}  // namespace pastis
