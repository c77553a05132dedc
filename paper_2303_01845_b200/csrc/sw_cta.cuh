// sw_cta.cuh -- K1c/K2c: one CTA per long pair (north-star item 4).
//
// The scalar score pass of sw_kernels.cuh (k_score: scaled int32, exact
// row-major-first end cell / reverse box) with the strips of ONE pair spread
// over the kCtaWarps warps of a CTA: warp w computes strips w, w+W, w+2W, ...
// and streams the bottom row of every strip to the warp computing the next
// strip, so all warps advance along the pair together (pipelined strips)
// instead of one warp walking all strips.  Links between consecutive warps
// are shared-memory rings with flow control; the wrap-around link (warp W-1
// -> warp 0, strip k+W-1 -> k+W) goes through a per-CTA global row so its
// producer never blocks (a bounded cyclic chain of rings could deadlock).
// Progress counters live in shared memory; all warps of a CTA are
// co-resident, so spinning on them is safe.
#pragma once
#include "sw_kernels.cuh"

namespace pastis {

constexpr int kCtaWarps = 4;
constexpr int kRing = 256;                       // columns per ring (power of 2)
constexpr int kCtaChunk = 32;                    // columns per consumer fetch
constexpr int kSmemCta = kMatBytes + kCtaWarps * (kProfBytes + kRing * 8) + 256;

struct CtaSync {               // per-CTA shared state
  volatile int prod[kCtaWarps];   // columns published into the link leaving warp w
  volatile int cons[kCtaWarps];   // columns consumed from the link leaving warp w
  int64_t item;
  volatile int dead_strip;      // reverse pass: first strip whose bottom row carries no live path
  volatile int stop_col[8];     // reverse pass: strip k's bottom row is dead from column stop_col[k & 7]
  unsigned long long red_fwd[kCtaWarps];
  int red_x[kCtaWarps], red_y[kCtaWarps], red_v[kCtaWarps];
};
static_assert(sizeof(CtaSync) <= 256, "CtaSync must fit the 256 B reserved in kSmemCta");

template <int R, int MODE>
__global__ void __launch_bounds__(kCtaWarps * 32)
k_score_cta(KArgs A, int stage, int cls) {
  extern __shared__ __align__(16) uint8_t smem[];
  int8_t *smat = reinterpret_cast<int8_t *>(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t *prof = smem + kMatBytes + warp * kProfBytes;
  int2 *rings = reinterpret_cast<int2 *>(smem + kMatBytes + kCtaWarps * kProfBytes);
  CtaSync &S = *reinterpret_cast<CtaSync *>(smem + kMatBytes + kCtaWarps * (kProfBytes + kRing * 8));
  load_matrix(smat, A.mat);
  int2 *wrap = A.bnd + (uint64_t)blockIdx.x * A.bnd_stride;   // warp W-1 -> warp 0 row
  const int32_t OPEN = A.open_ << 16, nEXT = -(A.ext << 16);
  // reverse pass (MODE 1): anchored at the end cell, floored, stopped after a
  // round of strips whose bottom row is dead -- see score_pair (sw_kernels.cuh)
  const int32_t FLOOR = (int32_t)max(-32600, -32766 + A.open_ + A.ext) * 65536;
  const int32_t ANC = FLOOR - OPEN;
  const int2 dflt = MODE == 1 ? make_int2(ANC, ANC) : make_int2(-OPEN, kNegInf);
  for (;;) {
    if (threadIdx.x == 0) {
      const uint32_t pos = atomicAdd(&A.ctrs[kStages * kNumClasses + stage * kNumClasses + cls], 1u);
      const uint32_t cnt = *(volatile uint32_t *)&A.ctrs[stage * kNumClasses + cls];
      S.item = pos < cnt ? (int64_t)list_of(A, stage, cls)[pos] : -1;
      for (int w = 0; w < kCtaWarps; ++w) { S.prod[w] = 0; S.cons[w] = 0; }
      S.dead_strip = 0x7fffffff;
    }
    __syncthreads();
    const int64_t k = S.item;
    if (k < 0) break;
    const sw_pair_t p = A.pairs[k];
    PairState *st = A.st + k;
    int m, n;
    View rows, cols;
    int32_t best_known = 0, i_end = 0, j_end = 0;
    if (MODE == 0) {
      m = (int)p.a_len;
      n = (int)p.b_len;
      rows = View{A.codes + p.a_off, 1};
      cols = View{A.codes + p.b_off, 1};
    } else {
      i_end = st->i_end;
      j_end = st->j_end;
      best_known = st->best;
      m = i_end + 1;
      n = j_end + 1;
      rows = View{A.codes + p.a_off + i_end, -1};
      cols = View{A.codes + p.b_off + j_end, -1};
    }
    const int nstrips = (m + 32 * R - 1) / (32 * R);
    ScoreOut res{0ull, 0, 0, 0};
    const int in_link = (warp + kCtaWarps - 1) % kCtaWarps;   // link feeding this warp
    int prod_total = 0, cons_total = 0;   // this warp's counters on its out / in links
    // reverse pass: once a strip is dead (S.dead_strip), every deeper strip
    // is abandoned -- at its start, at each 32-column fetch and inside the
    // ring waits; the dead strip itself has produced all its rows by then,
    // so no producer is left waiting on an abandoned consumer
    auto abandon = [&](int st) {
      return MODE == 1 && __shfl_sync(0xffffffffu, (int)(S.dead_strip < st), 0) != 0;
    };
    for (int strip = warp; strip < nstrips; strip += kCtaWarps) {
      if (abandon(strip)) break;
      const int row0 = strip * 32 * R;
      __syncwarp();
      build_profile<R>(prof, smat, rows, m, row0, lane);
      __syncwarp();
      ScoreLane<R, false> L;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        L.Ho[r] = MODE == 1 ? ANC : -OPEN;
        L.E[r] = MODE == 1 ? ANC : kNegInf;
        L.key[r] = 0;
      }
      L.hoUpPrev = (MODE == 1 && !(strip == 0 && lane == 0)) ? ANC : -OPEN;
      L.botHo = MODE == 1 ? ANC : -OPEN;
      L.botF = MODE == 1 ? ANC : kNegInf;
      bool alive = false;
      L.code_next = lane == 0 ? cols.at(0) : kPad;
      const bool has_above = strip > 0, has_below = strip + 1 < nstrips;
      const bool in_wrap = warp == 0;                  // fed by the global wrap row
      const bool out_wrap = warp == kCtaWarps - 1;     // feeds the global wrap row
      int2 *ring_in = rings + in_link * kRing, *ring_out = rings + warp * kRing;
      int2 cur = dflt;
      const int steps = n + 31;
      const int prod_base = prod_total, cons_base = cons_total;
      // reset by lane 31, the lane that publishes S.prod, before any column is published
      if (MODE == 1 && lane == 31) S.stop_col[strip & 7] = 0x7fffffff;
      for (int s = 0; s < steps; ++s) {
        if constexpr (MODE == 1) {
          // Horizontal stop: every path from the anchor into the columns right
          // of the wavefront crosses it (a lane's cells, the diagonal feed
          // hoUpPrev, the F leaving its bottom row) or enters from the row
          // above right of lane 0.  Once all of those are dead by the dead-
          // strip criterion (H <= 0, E/F <= ext - open; the row above dead
          // from its producer's stop column on), no cell to the right can
          // equal best (score_pair's argument, applied to a column cut), so
          // the strip ends here; its bottom row is dead from column s - 31 on.
          if ((s % kCtaChunk) == 0 && s > 0) {
            bool live = (L.hoUpPrev > -OPEN) | (L.botF > -OPEN - nEXT);
#pragma unroll
            for (int r = 0; r < R; ++r) live |= __viaddmax_s32(L.E[r], nEXT, L.Ho[r]) > -OPEN;
            const bool top_dead = !has_above || S.stop_col[(strip - 1) & 7] <= s;
            if (__all_sync(0xffffffffu, !live && top_dead)) {
              if (has_below) {
                if (lane == 31) S.stop_col[strip & 7] = max(0, s - 31);
                __threadfence_block();
                prod_total = prod_base + n;
                if (lane == 31) S.prod[warp] = prod_total;
              }
              if (has_above) {
                cons_total = cons_base + n;
                if (lane == 0) S.cons[in_link] = cons_total;
              }
              break;
            }
          }
        }
        // ---- top input of lane 0 (column s): fetched 32 columns at a time
        if (has_above && (s % kCtaChunk) == 0) {
          const int need = min(s + kCtaChunk, n);
          if (s < n) {
            const int target = cons_total + (need - s);
            while (S.prod[in_link] < target && !(MODE == 1 && S.dead_strip < strip)) __nanosleep(32);
            if (abandon(strip)) break;
            __syncwarp();
            const int c = s + lane;
            cur = dflt;
            // columns past the producer's stop column were never written: dead
            if (c < n && (MODE == 0 || c < S.stop_col[(strip - 1) & 7]))
              cur = in_wrap ? wrap[c] : ring_in[(cons_total + lane) & (kRing - 1)];
            __syncwarp();
            cons_total = target;
            if (lane == 0) S.cons[in_link] = cons_total;
          }
        }
        int2 top = make_int2(__shfl_sync(0xffffffffu, cur.x, s & 31),
                             __shfl_sync(0xffffffffu, cur.y, s & 31));
        if (!has_above) top = dflt;
        // ---- one wavefront step (same arithmetic as score_step)
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
        if (lane == 0) { upHo = top.x; upF = top.y; }
        int32_t cc = 0;
        if (valid) cc = MODE == 0 ? 65535 - c : c + 1;
        int32_t diag = L.hoUpPrev;
        L.hoUpPrev = upHo;
        int32_t F = upF, hoUp = upHo;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int32_t sc = (int32_t)prmt(word_of(pw, r), 0u, sel_scaled(r & 3));
          L.E[r] = __viaddmax_s32(L.E[r], nEXT, L.Ho[r]);
          const int32_t D = diag + sc + OPEN;
          const int32_t t = MODE == 1 ? __vimax3_s32(D, L.E[r], FLOOR) : __vimax_s32_relu(D, L.E[r]);
          F = __viaddmax_s32(F, nEXT, hoUp);
          const int32_t h = max(t, F);
          diag = L.Ho[r];
          L.Ho[r] = h - OPEN;
          hoUp = t - OPEN;
          L.key[r] = __viaddmax_s32(L.Ho[r], cc + OPEN, L.key[r]);
        }
        L.botHo = L.Ho[R - 1];
        L.botF = F;
        // ---- bottom row of lane 31 (column s - 31) to the next strip's warp
        if (has_below) {
          const int cb = s - 31;
          if (cb >= 0 && cb < n) {
            if (!out_wrap && (cb % kCtaChunk) == 0) {      // flow control on the ring
              const int limit = prod_total + kCtaChunk - kRing;
              while (S.cons[warp] < limit && !(MODE == 1 && S.dead_strip < strip)) __nanosleep(32);
            }
            if (lane == 31) {
              const int2 v = make_int2(L.botHo, L.botF);
              if (out_wrap) wrap[cb] = v;
              else ring_out[(prod_total) & (kRing - 1)] = v;
              if (MODE == 1) alive |= (L.botHo > -OPEN) | (L.botF > -OPEN - nEXT);
            }
            ++prod_total;
            if ((prod_total & 7) == 0 || cb == n - 1) {
              __threadfence_block();
              if (lane == 31) S.prod[warp] = prod_total;
            }
          }
        }
      }
      if (MODE == 1 && has_below && !__shfl_sync(0xffffffffu, (int)alive, 31) && lane == 0)
        atomicMin((int *)&S.dead_strip, strip);
      // strip reduction (as k_score)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int x = row0 + lane * R + r;
        if (x >= m) continue;
        const int32_t v = L.key[r] >> 16, lo = L.key[r] & 0xFFFF;
        res.vmax = v > res.vmax ? v : res.vmax;
        if (MODE == 0) {
          const uint64_t comp = ((uint64_t)(uint32_t)v << 32) | ((uint64_t)(0xFFFF - x) << 16) |
                                (uint64_t)lo;
          res.fwd = comp > res.fwd ? comp : res.fwd;
        } else if (v >= best_known && lo >= 1) {
          res.rev_x = x + 1 > res.rev_x ? x + 1 : res.rev_x;
          res.rev_y = lo > res.rev_y ? lo : res.rev_y;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t f = __shfl_xor_sync(0xffffffffu, res.fwd, o);
      res.fwd = f > res.fwd ? f : res.fwd;
      res.rev_x = max(res.rev_x, __shfl_xor_sync(0xffffffffu, res.rev_x, o));
      res.rev_y = max(res.rev_y, __shfl_xor_sync(0xffffffffu, res.rev_y, o));
      res.vmax = max(res.vmax, __shfl_xor_sync(0xffffffffu, res.vmax, o));
    }
    if (lane == 0) {
      S.red_fwd[warp] = res.fwd;
      S.red_x[warp] = res.rev_x;
      S.red_y[warp] = res.rev_y;
      S.red_v[warp] = res.vmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < kCtaWarps; ++w) {
        res.fwd = S.red_fwd[w] > res.fwd ? S.red_fwd[w] : res.fwd;
        res.rev_x = max(res.rev_x, S.red_x[w]);
        res.rev_y = max(res.rev_y, S.red_y[w]);
        res.vmax = max(res.vmax, S.red_v[w]);
      }
      if (MODE == 0) {
        const int32_t best = (int32_t)(res.fwd >> 32);
        const int32_t ie = 0xFFFF - (int32_t)((res.fwd >> 16) & 0xFFFF);
        const int32_t je = 65535 - (int32_t)(res.fwd & 0xFFFF);
        if (res.vmax >= kScaledLimit) {
          st->flags = kFlagWide;
          list_push(A, 3, 0, (uint32_t)k);
        } else {
          st->best = best;
          st->i_end = best > 0 ? ie : -1;
          st->j_end = best > 0 ? je : -1;
          st->flags = 0;
          if (best > 0) {
            const uint64_t area = (uint64_t)(ie + 1) * (uint64_t)(je + 1);
            if ((uint64_t)best * best * 8ull > 49ull * area) {   // homolog: box = prefix
              st->i0 = 0;
              st->j0 = 0;
              list_push(A, 2, class_of(ie + 1), (uint32_t)k);
            } else {
              list_push(A, 1, long_class(ie + 1), (uint32_t)k);
            }
          }
        }
      } else {
        const int32_t i0 = i_end + 1 - res.rev_x, j0 = j_end + 1 - res.rev_y;
        st->i0 = i0;
        st->j0 = j0;
        list_push(A, 2, class_of(i_end - i0 + 1), (uint32_t)k);
      }
    }
    __syncthreads();
  }
}

}  // namespace pastis
