// sw_engine.cu -- host runtime + C ABI (include/pastis_sw.h) of the B200
// batched Smith-Waterman aligner.
//
// Replaces the reference's batch seam (pastislite.align.align_batch,
// align.py:223-246, and AlignEngine's process-pool lanes, align.py:299-347)
// with: raw-byte arena + pair table on the device -> k_encode -> k_classify
// (length bins) -> K1 forward per bin -> K1 wide re-run of overflowing pairs
// -> K2 reverse per bin -> K3 box per bin -> k_walk.  One CUDA stream per
// device; one host thread per device for multi-GPU sharding.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <queue>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/transform_iterator.h>

#include "sw_kernels.cuh"
#include "sw_packed.cuh"
#include "sw_cta.cuh"
#include "sw_cta_packed.cuh"
#include "sw_fasta.h"
#include "sw_kmer.cuh"

using namespace pastis;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CU(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(SW_ECUDA, std::string(#call " failed: ") + cudaGetErrorString(e_));         \
  } while (0)

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    size_t b = std::max<size_t>(want + want / 8, 4096);
    cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaSuccess) bytes = b;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

constexpr int kSmemScore = kMatBytes + kWarpsPerBlock * kProfBytes;

typedef void (*KernelFn)(KArgs, int, int);

struct KernelInfo {
  KernelFn fn;
  int grid;
  int smem;
};

struct DeviceCtx {
  int device = -1;
  int sms = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  DevBuf arena, codes, pairs, out, st, lists, ctrs, stats, mat, lut, bnd, pool;
  // sharding (sw_align_shard / sw_align_batch_multi): the whole pair table,
  // sort keys, the shard's pair table / indices / lengths / offsets, its arena
  DevBuf sh_cells;
  // gathered host arenas: per-pair ready flags, gather segments, their stream
  DevBuf pready, gseg;
  cudaStream_t gstream = nullptr;
  cudaStream_t fstream = nullptr;   // the packed classes' forward passes, in class order (gathered arena)
  DevBuf skeys, svals, cubtmp;  // work-list sort
  DevBuf km_arena, km_off, km_len, km_base, km_keys, km_runs, km_pairs, km_out, km_small;
  cudaEvent_t ev[16];
  // one stream per length class: the packed forward + tile traceback of each
  // class run concurrently so the tail of one class overlaps the others
  cudaStream_t cstream[kNumClasses];
  cudaEvent_t ev_fork, ev_k1[kNumClasses], ev_tb[kNumClasses];
  KernelInfo fwd[kNumClasses], rev[kNumClasses], box[kNumClasses], ckpt[kNumClasses];
  KernelInfo tb[kNumClasses];
  KernelInfo fwd_wide, rev_wide, fwd_cta, rev_cta, fwd_ctap, jend;
  DevBuf cta_rows;
  int max_warps = 0;
  size_t pool_want = 0;   // checkpoint bytes the last call asked for (pool growth)
  // host path: the arena is uploaded in slices on copy_stream while the packed
  // forward already runs; `ready` counts the slices that have landed
  cudaStream_t copy_stream = nullptr;
  cudaStream_t pstream = nullptr;          // greatest priority: run_device's chain
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaEvent_t ev_pairs = nullptr, ev_arena = nullptr;
  DevBuf readyb;
  uint32_t *slice_vals = nullptr;   // pinned 1..kMaxSlices
  bool ready = false;
};

constexpr int kMaxSlices = 64;

std::mutex g_ctx_mu;
std::vector<DeviceCtx *> g_ctx;

template <typename K>
int setup_kernel(K fn, int sms, KernelInfo &ki, int &max_warps) {
  CU(cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          kSmemScore));
  int nb = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)fn, kWarpsPerBlock * 32,
                                                   kSmemScore));
  if (nb < 1) return fail(SW_ECUDA, "kernel cannot be resident (occupancy 0)");
  ki.fn = (KernelFn)fn;
  ki.grid = nb * sms;
  max_warps = std::max(max_warps, ki.grid * kWarpsPerBlock);
  return SW_OK;
}

template <typename K>
int setup_packed(K fn, int sms, int smem, KernelInfo &ki, int &max_warps) {
  CU(cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int nb = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)fn, kWarpsPerBlockP * 32,
                                                   smem));
  if (nb < 1) return fail(SW_ECUDA, "packed kernel cannot be resident");
  ki.fn = (KernelFn)fn;
  ki.grid = nb * sms;
  ki.smem = smem;
  max_warps = std::max(max_warps, ki.grid * kWarpsPerBlockP);
  return SW_OK;
}

template <typename K>
int setup_cta(K fn, int sms, KernelInfo &ki) {
  CU(cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCta));
  int nb = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)fn, kCtaWarps * 32, kSmemCta));
  if (nb < 1) return fail(SW_ECUDA, "CTA kernel cannot be resident");
  ki.fn = (KernelFn)fn;
  ki.grid = nb * sms;
  ki.smem = kSmemCta;
  return SW_OK;
}

template <typename K>
int setup_tb(K fn, int sms, KernelInfo &ki) {
  int nb = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void *)fn, kTbWarps * 32, 0));
  if (nb < 1) return fail(SW_ECUDA, "k_tb cannot be resident");
  ki.fn = (KernelFn)fn;
  ki.grid = nb * sms;
  return SW_OK;
}

template <int C>
int setup_classes(DeviceCtx *c) {
  if constexpr (C < kNumClasses) {
    constexpr int R = class_rows(C);
    int rc = setup_kernel(k_score<R, 0, false>, c->sms, c->fwd[C], c->max_warps);
    if (rc) return rc;
    rc = setup_kernel(k_score<R, 1, false>, c->sms, c->rev[C], c->max_warps);
    if (rc) return rc;
    rc = setup_kernel(k_box<R, false>, c->sms, c->box[C], c->max_warps);
    if (rc) return rc;
    rc = setup_packed(k_score_packed<R>, c->sms, smem_packed(R), c->ckpt[C], c->max_warps);
    if (rc) return rc;
    rc = setup_tb(k_tb<R>, c->sms, c->tb[C]);
    if (rc) return rc;
    return setup_classes<C + 1>(c);
  } else {
    return SW_OK;
  }
}

int get_ctx(int device, DeviceCtx **out) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= 0)
    return fail(SW_ECUDA, "no CUDA device visible");
  if (device < 0 || device >= n) return fail(SW_EINVAL, "device ordinal out of range");
  std::lock_guard<std::mutex> g(g_ctx_mu);
  if ((int)g_ctx.size() < n) g_ctx.resize(n, nullptr);
  if (!g_ctx[device]) g_ctx[device] = new DeviceCtx();
  DeviceCtx *c = g_ctx[device];
  if (!c->ready) {
    CU(cudaSetDevice(device));
    c->device = device;
    CU(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
    // The call's serial chain (planning, the scalar long-pair kernels, the
    // box traceback, the walk) runs on a greatest-priority stream, the
    // length classes on least-priority streams: pending blocks of the chain
    // are scheduled first whenever a class kernel frees an SM, so the chain
    // is not queued behind the classes' persistent grids.
    int prio_least = 0, prio_greatest = 0;
    CU(cudaDeviceGetStreamPriorityRange(&prio_least, &prio_greatest));
    CU(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, prio_greatest));
    CU(cudaStreamCreateWithPriority(&c->pstream, cudaStreamNonBlocking, prio_greatest));
    CU(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
    for (auto &e : c->ev) CU(cudaEventCreate(&e));
    CU(cudaEventCreate(&c->ev_fork));
    for (int k = 0; k < kNumClasses; ++k) {
      CU(cudaStreamCreateWithPriority(&c->cstream[k], cudaStreamNonBlocking, prio_least));
      CU(cudaEventCreate(&c->ev_k1[k]));
      CU(cudaEventCreate(&c->ev_tb[k]));
    }
    CU(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithPriority(&c->gstream, cudaStreamNonBlocking, prio_greatest));
    CU(cudaStreamCreateWithPriority(&c->fstream, cudaStreamNonBlocking, prio_least));
    CU(cudaEventCreateWithFlags(&c->ev_pairs, cudaEventDisableTiming));
    CU(cudaEventCreate(&c->ev_arena));
    CU(c->readyb.ensure(64));
    CU(cudaHostAlloc((void **)&c->slice_vals, kMaxSlices * sizeof(uint32_t), cudaHostAllocDefault));
    for (int k = 0; k < kMaxSlices; ++k) c->slice_vals[k] = (uint32_t)(k + 1);
    int rc = setup_classes<0>(c);
    if (rc) return rc;
    rc = setup_kernel(k_score<16, 0, true>, c->sms, c->fwd_wide, c->max_warps);
    if (rc) return rc;
    rc = setup_kernel(k_score<16, 1, true>, c->sms, c->rev_wide, c->max_warps);
    if (rc) return rc;
    rc = setup_cta(k_score_cta<kCtaRowsR, 0>, c->sms, c->fwd_cta);
    if (rc) return rc;
    rc = setup_cta(k_score_cta<kCtaRowsR, 1>, c->sms, c->rev_cta);
    if (rc) return rc;
    {
      const void *fn = (const void *)k_score_cta_packed<kCtaPR>;
      const int smem = smem_cta_packed(kCtaPR);
      CU(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      int nb = 0;
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kCtaWarps * 32, smem));
      if (nb < 1) return fail(SW_ECUDA, "packed CTA kernel cannot be resident");
      c->fwd_ctap.fn = (KernelFn)k_score_cta_packed<kCtaPR>;
      c->fwd_ctap.grid = nb * c->sms;
      c->fwd_ctap.smem = smem;
      CU(c->cta_rows.ensure((size_t)c->fwd_ctap.grid * kCtaPSlots * kCtaPRowStride * sizeof(uint2)));
    }
    rc = setup_kernel(k_jend<kCtaPR>, c->sms, c->jend, c->max_warps);
    if (rc) return rc;
    // LUT (align.py:27-30) and matrix buffers
    CU(c->lut.ensure(256));
    uint8_t lut[256];
    const char *alpha = "ARNDCQEGHILKMFPSTWYVBZXU*";
    for (int i = 0; i < 256; ++i) lut[i] = 22;  // 'X'
    for (int k = 0; k < kAlpha; ++k) lut[(uint8_t)alpha[k]] = (uint8_t)k;
    CU(cudaMemcpy(c->lut.p, lut, 256, cudaMemcpyHostToDevice));
    CU(c->mat.ensure(kMatBytes));
    c->ready = true;
  }
  *out = c;
  return SW_OK;
}

int check_params(const sw_params_t *p) {
  if (!p) return fail(SW_EINVAL, "params is NULL");
  if (!(p->gap_open >= p->gap_extend && p->gap_extend >= 0))
    return fail(SW_EINVAL, "need gap_open >= gap_extend >= 0");
  if (p->gap_open > 16383)
    return fail(SW_EINVAL, "gap_open > 16383 is outside the GPU aligner's supported domain");
  for (int i = 0; i < 25; ++i)
    for (int j = 0; j < 25; ++j) {
      const int32_t v = p->matrix[i * 25 + j];
      if (v < -127 || v > 127)
        return fail(SW_EINVAL, "substitution scores must lie in [-127, 127] for the GPU aligner");
      if (v != p->matrix[j * 25 + i]) return fail(SW_EINVAL, "substitution matrix must be symmetric");
    }
  return SW_OK;
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// Core device pipeline.  Caller holds c->mu and has set the device.
// `ready`/`slice_bytes`/`arena_done`: host-pipelined arena (align_host) --
// the packed forward waits per pair for its slices, everything reading the
// encoded arena waits for arena_done; nullptr = the arena is resident.
// `arena_lo`: only arena offsets [arena_lo, arena_bytes) are present;
// d_arena is the virtual base (d_arena + off is valid in that range).
int run_device(DeviceCtx *c, const uint8_t *d_arena, uint64_t arena_bytes,
               const sw_pair_t *d_pairs, uint64_t n_pairs, const sw_params_t *prm,
               sw_result_t *d_out, cudaStream_t s, sw_timing_t *tm,
               const uint32_t *ready = nullptr, uint64_t slice_bytes = 0,
               cudaEvent_t arena_done = nullptr, uint64_t arena_lo = 0,
               const uint8_t *gather_src = nullptr) {
  if (n_pairs == 0) return SW_OK;
  if (n_pairs > 0xFFFFFFF0ull) return fail(SW_EINVAL, "too many pairs in one call");
  // the chain runs on the greatest-priority stream, joined back to `s` at the end
  cudaStream_t user_s = s;
  if (s != c->stream) {
    s = c->pstream;
    CU(cudaEventRecord(c->ev_in, user_s));
    CU(cudaStreamWaitEvent(s, c->ev_in, 0));
  }
  uint32_t launches = 0;
  uint32_t plan_cnt[kStages * kNumClasses];
  unsigned long long plan_ckpt = 0;   // checkpoint bytes the packed pass will need
  const double h0 = now_ms();
  // device buffers
  CU(c->codes.ensure(arena_bytes - arena_lo + 64));
  CU(c->st.ensure(n_pairs * sizeof(PairState)));
  CU(c->lists.ensure((size_t)kStages * kNumClasses * n_pairs * 4));
  CU(c->ctrs.ensure(2 * kStages * kNumClasses * 4));
  CU(c->stats.ensure(8 * 8));
  // int8 matrix incl. the virtual code 25 (-128 everywhere)
  int8_t mat[kMatBytes];
  memset(mat, 0, sizeof(mat));
  for (int i = 0; i < kCodes; ++i)
    for (int j = 0; j < kCodes; ++j)
      mat[i * kCodes + j] =
          (i == kPad || j == kPad) ? (int8_t)-128 : (int8_t)prm->matrix[i * 25 + j];
  CU(cudaMemcpyAsync(c->mat.p, mat, kCodes * kCodes, cudaMemcpyHostToDevice, s));
  CU(cudaMemsetAsync(c->ctrs.p, 0, 2 * kStages * kNumClasses * 4, s));
  CU(cudaMemsetAsync(c->stats.p, 0, 8 * 8, s));

  KArgs A;
  memset(&A, 0, sizeof(A));
  // codes[i] = lut[raw[i]] at the raw arena's address modulo 16, so k_encode
  // moves aligned 128-bit words whatever the caller's pointer alignment
  uint8_t *codes_lo = (uint8_t *)c->codes.p + ((uintptr_t)(d_arena + arena_lo) & 15u);
  uint8_t *codes = codes_lo - arena_lo;       // virtual base, like d_arena
  A.codes = codes;
  A.raw = d_arena;
  A.arena_lo = arena_lo;
  A.pairs = d_pairs;
  A.st = (PairState *)c->st.p;
  A.out = d_out;
  A.mat = (const int8_t *)c->mat.p;
  A.lists = (uint32_t *)c->lists.p;
  A.ctrs = (uint32_t *)c->ctrs.p;
  A.n_pairs = n_pairs;
  A.arena_bytes = arena_bytes;
  A.lut = (const uint8_t *)c->lut.p;
  A.ready = ready;
  A.slice_bytes = slice_bytes;
  // gathered host arena: the pair's bytes are pulled over PCIe by
  // k_gather_arena in consumption order; K1p waits per duo on its flags
  if (gather_src) {
    CU(c->pready.ensure(n_pairs * 4 + 4));
    CU(cudaMemsetAsync(c->pready.p, 0, n_pairs * 4 + 4, s));
    A.pair_ready = (const uint32_t *)c->pready.p;
    A.gather_count = (const uint32_t *)c->pready.p + n_pairs;
    A.gather_src = gather_src;
    A.gather_dst = const_cast<uint8_t *>(d_arena);
  }
  A.cta_rows = (uint2 *)c->cta_rows.p;
  A.open_ = prm->gap_open;
  A.ext = prm->gap_extend;
  int smin = 127, smax = -128;
  for (int i = 0; i < 625; ++i) {
    smin = std::min(smin, (int)prm->matrix[i]);
    smax = std::max(smax, (int)prm->matrix[i]);
  }
  // packed passes: u8 profile u = s + open, so D = Ho_diag + u needs no
  // constant; PAD -> u = 0 (scores -open, never reaches a real cell)
  A.prof_lo = -prm->gap_open;
  A.bias16 = prm->gap_open + prm->gap_extend + 128;
  A.p_bb = (uint32_t)A.bias16 * 0x10001u;
  A.p_open2 = (uint32_t)prm->gap_open * 0x10001u;
  A.p_ext2 = (uint32_t)prm->gap_extend * 0x10001u;
  A.p_ho0 = A.p_bb - A.p_open2;
  A.p_next2 = (uint32_t)((65536 - prm->gap_extend) & 0xFFFF) * 0x10001u;
  A.p_nopen2 = (uint32_t)((65536 - prm->gap_open) & 0xFFFF) * 0x10001u;
  // the packed passes need every u in [0, 127]; other parameter sets
  // (matrix minimum below -open, or maximum above 127 - open) take the
  // scalar int32 paths
  const bool packed_ok = smin >= -prm->gap_open && smax + prm->gap_open <= 127;

  CU(cudaEventRecord(c->ev[0], s));
  if (!arena_done) {   // resident arena: encode first, every kernel reads codes
    const int threads = 256;
    uint64_t blocks = std::min<uint64_t>(((arena_bytes - arena_lo) / 16 + threads) / threads + 1,
                                         (uint64_t)c->sms * 8);
    k_encode<<<(unsigned)blocks, threads, 0, s>>>(d_arena + arena_lo, codes_lo, arena_bytes - arena_lo,
                                                 (const uint8_t *)c->lut.p);
    ++launches;
  }
  {
    // PASTIS_SW_TRACEBACK=box forces the reverse-pass + box traceback for every
    // pair (A/B comparisons); default: checkpoint + tile replay for pairs
    // up to kFusedMaxCells cells.
    static const int env_ckpt = [] {
      const char *e = getenv("PASTIS_SW_TRACEBACK");
      return (e && strcmp(e, "box") == 0) ? 0 : 1;
    }();
    CU(c->skeys.ensure(2 * n_pairs * sizeof(unsigned long long)));
    CU(c->svals.ensure(2 * n_pairs * sizeof(uint32_t)));
    unsigned long long *k_in = (unsigned long long *)c->skeys.p, *k_out = k_in + n_pairs;
    uint32_t *v_in = (uint32_t *)c->svals.p, *v_out = v_in + n_pairs;
    // work lists sorted by shape (m, n descending) by default;
    // PASTIS_SW_SORT=cells sorts by cell count instead (A/B comparisons)
    static const int env_sort = [] {
      const char *e = getenv("PASTIS_SW_SORT");
      return (e && strcmp(e, "cells") == 0) ? 1 : (e && strcmp(e, "chunk") == 0) ? 2 : 0;
    }();
    const int sort_cells = env_sort == 2 ? (ready ? 2 : 0) : env_sort;
    k_classify<<<(unsigned)((n_pairs + 255) / 256), 256, 0, s>>>(
        A, (unsigned long long *)c->stats.p, env_ckpt && packed_ok, packed_ok, k_in, v_in, sort_cells);
    ++launches;
    CU(cudaGetLastError());
    // the one host round trip of the call: which lists the plan filled, so
    // the kernels of empty length classes and of an absent long-pair path are
    // not launched (a persistent grid that finds its list empty still costs a
    // launch and a wave of empty blocks: ~30 of a call's 38 launches on a
    // one-class batch)
    CU(cudaMemcpyAsync(plan_cnt, c->ctrs.p, sizeof(plan_cnt), cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(&plan_ckpt, (unsigned long long *)c->stats.p + 6, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    size_t tmp_bytes = 0;
    CU(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in, k_out, v_in, v_out,
                                       (int)n_pairs, 0, list_key_shift(sort_cells) + 7, s));
    CU(c->cubtmp.ensure(tmp_bytes));
    CU(cub::DeviceRadixSort::SortPairs(c->cubtmp.p, tmp_bytes, k_in, k_out, v_in, v_out,
                                       (int)n_pairs, 0, list_key_shift(sort_cells) + 7, s));
    launches += 4;
    k_scatter_lists<<<(unsigned)std::min<uint64_t>((n_pairs + 255) / 256, (uint64_t)c->sms * 8), 256,
                      0, s>>>(A, k_out, v_out, list_key_shift(sort_cells));
    ++launches;
    CU(cudaGetLastError());
    if (gather_src) {
      // gather order: the packed class lists, then the long-pair lists
      // (whose kernels wait for all of it)
      // the packed classes' forward passes run one after the other on one
      // stream in this mode (below), so the gather follows their lists in
      // that order
      std::vector<GatherSeg> seg;
      uint32_t total = 0;
      for (int cls = 0; cls < kNumClasses; ++cls) {
        const uint32_t cnt = plan_cnt[6 * kNumClasses + cls];
        if (cnt) { seg.push_back({(uint32_t)(6 * kNumClasses + cls), 0u, total}); total += cnt; }
      }
      for (int cls = 0; cls < kNumClasses; ++cls) {
        const uint32_t cnt = plan_cnt[cls];
        if (cnt) { seg.push_back({(uint32_t)cls, 0u, total}); total += cnt; }
      }
      if (total) {
        CU(c->gseg.ensure(seg.size() * sizeof(GatherSeg)));
        CU(cudaMemcpyAsync(c->gseg.p, seg.data(), seg.size() * sizeof(GatherSeg),
                           cudaMemcpyHostToDevice, s));
        CU(cudaEventRecord(c->ev[14], s));
        CU(cudaStreamWaitEvent(c->gstream, c->ev[14], 0));
        static const int env_gb = [] {
          const char *e = getenv("PASTIS_SW_GATHER_BLOCKS");
          return e ? std::max(1, atoi(e)) : 16;
        }();
        k_gather_arena<<<env_gb, 1024, 0, c->gstream>>>(A, gather_src, const_cast<uint8_t *>(d_arena),
                                                    (const GatherSeg *)c->gseg.p, (int)seg.size(),
                                                    total, (uint32_t *)c->pready.p);
        ++launches;
        CU(cudaGetLastError());
      }
      CU(cudaEventRecord(arena_done, c->gstream));
    }
  }
  // No host round trip before the kernels: the strip-boundary scratch is
  // sized for the longest supported sequence and the traceback pool is one
  // cached allocation, grown between calls to what the previous call's
  // checkpoints asked for.  A call that outgrows it runs extra packed rounds
  // on the deferred pairs with the pool recycled (device-side chunking).
  A.bnd_stride = 65000 + 64;
  CU(c->bnd.ensure((size_t)c->max_warps * A.bnd_stride * sizeof(int2)));
  A.bnd = (int2 *)c->bnd.p;
  // PASTIS_SW_POOL_MB pins the pool size (tests use it to force the deferral paths)
  static const long long env_mb = [] {
    const char *e = getenv("PASTIS_SW_POOL_MB");
    return e ? atoll(e) : 0ll;
  }();
  // size the pool for this call's checkpoints up front (k_classify's
  // estimate + 15 %), so the packed pass normally runs in one round; a pool
  // that still overflows defers pairs to further rounds
  if (env_mb == 0)
    c->pool_want = std::max(c->pool_want, (size_t)(plan_ckpt + plan_ckpt / 7) + ((size_t)64 << 20));
  if (c->pool.bytes == 0 || c->pool_want > c->pool.bytes) {
    size_t free_b = 0, total_b = 0;
    CU(cudaMemGetInfo(&free_b, &total_b));
    const size_t limit = (size_t)((double)(free_b + c->pool.bytes) * 0.8);
    size_t target = c->pool.bytes == 0 ? std::min<size_t>(free_b / 2, (size_t)16 << 30) : c->pool.bytes;
    target = std::min(std::max(target, c->pool_want), limit);
    if (env_mb > 0) target = std::min<size_t>(target, (size_t)env_mb << 20);
    target = std::max<size_t>(target, env_mb > 0 ? (size_t)1 << 20 : (size_t)8 << 20);
    if (target > c->pool.bytes) {
      c->pool.release();
      CU(c->pool.ensure(target));
    }
  }
  const double h1 = now_ms();
  A.pool = (uint8_t *)c->pool.p;
  A.pool_cap = c->pool.bytes - 64;  // headroom for the widest vector store
  // pool_top lives in the stats buffer slot 3; slot 4 = bytes the first
  // packed round asked for
  A.pool_top = (unsigned long long *)c->stats.p + 3;
  const double h2 = now_ms();
  CU(cudaEventRecord(c->ev[1], s));

  uint32_t h_cnt[kStages * kNumClasses];
  double fwd_ms = 0.0, rev_ms = 0.0, tb_ms = 0.0, tile_ms = 0.0, tail_ms = 0.0;
  uint64_t wide = 0;
  for (int pround = 0;; ++pround) {
    CU(cudaMemsetAsync(A.pool_top, 0, 8, s));
    if (pround > 0) {
      k_packed_round<<<kNumClasses, 256, 0, s>>>(A);
      ++launches;
    }
    // short/medium pairs: packed forward + checkpoints, then the tile
    // traceback, one stream per length class
    CU(cudaEventRecord(c->ev_fork, s));
    // The packed classes' persistent forward grids each fill the GPU, so they
    // run nearly one after the other anyway; with a gathered arena they run
    // strictly in class order on one stream (the order the gather follows),
    // each class's tile traceback on its own stream behind it.
    static const int env_serial = [] {
      const char *e = getenv("PASTIS_SW_SERIAL_FWD");
      return e ? atoi(e) : -1;
    }();
    const bool serial_fwd = pround == 0 && (env_serial >= 0 ? env_serial == 1 : A.pair_ready != nullptr);
    if (serial_fwd) CU(cudaStreamWaitEvent(c->fstream, c->ev_fork, 0));
    for (int cls = 0; cls < kNumClasses; ++cls) {
      cudaStream_t cs = c->cstream[cls];
      CU(cudaStreamWaitEvent(cs, c->ev_fork, 0));
      // round 0: classes the plan left empty are skipped; deferred rounds
      // refill the lists on the device, so every class runs
      if (pround == 0 && plan_cnt[6 * kNumClasses + cls] == 0) {
        CU(cudaEventRecord(c->ev_k1[cls], cs));
        CU(cudaEventRecord(c->ev_tb[cls], cs));
        continue;
      }
      cudaStream_t fs = serial_fwd ? c->fstream : cs;
      c->ckpt[cls].fn<<<c->ckpt[cls].grid, kWarpsPerBlockP * 32, c->ckpt[cls].smem, fs>>>(A, 6, cls);
      CU(cudaEventRecord(c->ev_k1[cls], fs));
      if (fs != cs) CU(cudaStreamWaitEvent(cs, c->ev_k1[cls], 0));
      c->tb[cls].fn<<<c->tb[cls].grid, kTbWarps * 32, 0, cs>>>(A, 7, cls);
      CU(cudaEventRecord(c->ev_tb[cls], cs));
      launches += 2;
    }
    // long pairs (one CTA per pair, or one warp per pair) exist only if the
    // plan put some there; they all run in round 0
    const bool long_pairs = pround == 0 && (plan_cnt[kCtaClass] + plan_cnt[kLongClass]) > 0;
    if (pround == 0 && arena_done) {
      // host-pipelined arena: the packed pass reads raw bytes through the
      // LUT; the scalar kernels below read the encoded arena once all of it
      // has landed
      CU(cudaStreamWaitEvent(s, arena_done, 0));
      const int threads = 256;
      uint64_t blocks = std::min<uint64_t>(((arena_bytes - arena_lo) / 16 + threads) / threads + 1,
                                           (uint64_t)c->sms * 8);
      k_encode<<<(unsigned)blocks, threads, 0, s>>>(d_arena + arena_lo, codes_lo,
                                                   arena_bytes - arena_lo, (const uint8_t *)c->lut.p);
      ++launches;
    }
    // long pairs: scalar forward concurrently with the packed classes -- one
    // CTA per pair for pairs of >= 4 strips, one warp per pair for the others
    // (their lists are empty after the first round)
    if (long_pairs) {
      c->fwd_ctap.fn<<<c->fwd_ctap.grid, kCtaWarps * 32, c->fwd_ctap.smem, s>>>(A, 0, kCtaClass);
      c->fwd[kLongClass].fn<<<c->fwd[kLongClass].grid, kWarpsPerBlock * 32, kSmemScore, s>>>(
          A, 0, kLongClass);
      launches += 2;
    }
    CU(cudaEventRecord(c->ev[7], s));   // end of the concurrent scalar forward
    // then the packed pass's scalar fallbacks (their own list, complete once
    // every packed class has finished), on the long-pair kernel
    for (int cls = 0; cls < kNumClasses; ++cls) CU(cudaStreamWaitEvent(s, c->ev_k1[cls], 0));
    if (pround == 0)
      CU(cudaMemcpyAsync((unsigned long long *)c->stats.p + 4, A.pool_top, 8,
                         cudaMemcpyDeviceToDevice, s));
    c->fwd[kLongClass].fn<<<c->fwd[kLongClass].grid, kWarpsPerBlock * 32, kSmemScore, s>>>(
        A, 0, kFallbackClass);
    // long pairs the packed CTA kernel had no pool room for, then the j_end
    // replay of those it did
    ++launches;
    if (long_pairs) {
      c->fwd_cta.fn<<<c->fwd_cta.grid, kCtaWarps * 32, kSmemCta, s>>>(A, 0, kCtaScalarClass);
      c->jend.fn<<<c->jend.grid, kWarpsPerBlock * 32, kSmemScore, s>>>(A, 9, 0);
      launches += 2;
    }
    c->fwd_wide.fn<<<c->fwd_wide.grid, kWarpsPerBlock * 32, kSmemScore, s>>>(A, 3, 0);
    ++launches;
    CU(cudaGetLastError());
    CU(cudaEventRecord(c->ev[2], s));
    // stage-1 lists: pairs of the scalar forwards (long pairs, and packed-pass
    // fallbacks, whose end row can reach the CTA class) and of k_jend; wide
    // pairs take the prefix box directly (no reverse pass)
    c->rev_cta.fn<<<c->rev_cta.grid, kCtaWarps * 32, kSmemCta, s>>>(A, 1, kCtaClass);
    ++launches;
    c->rev[kLongClass].fn<<<c->rev[kLongClass].grid, kWarpsPerBlock * 32, kSmemScore, s>>>(
        A, 1, kLongClass);
    ++launches;
    CU(cudaGetLastError());
    CU(cudaEventRecord(c->ev[3], s));
    for (int cls = 0; cls < kNumClasses; ++cls) CU(cudaStreamWaitEvent(s, c->ev_tb[cls], 0));
    CU(cudaEventRecord(c->ev[13], s));   // box traceback starts once every class's K5 is done
    uint32_t last_retry = 0;
    for (int round = 0;; ++round) {
      for (int cls = 0; cls < kNumClasses; ++cls) {
        c->box[cls].fn<<<c->box[cls].grid, kWarpsPerBlock * 32, kSmemScore, s>>>(A, 2, cls);
        ++launches;
      }
      k_walk<<<(unsigned)((n_pairs + 127) / 128), 128, 0, s>>>(A, nullptr, 0);
      ++launches;
      CU(cudaGetLastError());
      CU(cudaEventRecord(c->ev[4], s));
      CU(cudaMemcpyAsync(h_cnt, c->ctrs.p, sizeof(h_cnt), cudaMemcpyDeviceToHost, s));
      CU(cudaStreamSynchronize(s));
      tb_ms += ev_ms(round == 0 ? c->ev[13] : c->ev[5], c->ev[4]);
      const uint32_t n_retry = h_cnt[5 * kNumClasses];
      if (n_retry == 0) break;
      // every retry round starts on an empty pool, so it places at least one
      // box unless a single box is larger than the whole pool
      if (round > 0 && n_retry >= last_retry) {
        // grow the pool (its contents are dead here: every placed box has
        // been walked) unless PASTIS_SW_POOL_MB pins it
        size_t free_b = 0, total_b = 0;
        CU(cudaMemGetInfo(&free_b, &total_b));
        const size_t grown = c->pool.bytes * 2;
        if (env_mb > 0 || grown > (size_t)((double)(free_b + c->pool.bytes) * 0.8))
          return fail(SW_EINTERNAL, "traceback code pool too small for one pair's box");
        c->pool.release();
        CU(c->pool.ensure(grown));
        A.pool = (uint8_t *)c->pool.p;
        A.pool_cap = c->pool.bytes - 64;
      }
      last_retry = n_retry;
      // requeue: reset K3 lists, pool, retry list
      CU(cudaEventRecord(c->ev[5], s));
      uint32_t *ctrs = (uint32_t *)c->ctrs.p;
      CU(cudaMemsetAsync(ctrs + 2 * kNumClasses, 0, kNumClasses * 4, s));
      CU(cudaMemsetAsync(ctrs + kStages * kNumClasses + 2 * kNumClasses, 0, kNumClasses * 4, s));
      CU(cudaMemsetAsync(A.pool_top, 0, 8, s));
      k_requeue<<<64, 256, 0, s>>>(A);
      ++launches;
      CU(cudaMemsetAsync(ctrs + 5 * kNumClasses, 0, 4, s));
      CU(cudaMemsetAsync(ctrs + kStages * kNumClasses + 5 * kNumClasses, 0, 4, s));
    }
    // forward = the forward passes that run concurrently after the fork: the
    // packed classes (their own streams) and the scalar long-pair pass (main
    // stream); the scalar fallback re-run is not included (it is in kernel_ms)
    if (getenv("PASTIS_SW_DEBUG_E2E")) {   // per-class completion times (debug aid)
      fprintf(stderr, "round %d: main-fwd %.2f |", pround, ev_ms(c->ev_fork, c->ev[7]));
      for (int cls = 0; cls < kNumClasses; ++cls)
        fprintf(stderr, " R%d k1 %.2f tb %.2f (n=%u) |", class_rows(cls), ev_ms(c->ev_fork, c->ev_k1[cls]),
                ev_ms(c->ev_fork, c->ev_tb[cls]), h_cnt[6 * kNumClasses + cls]);
      fprintf(stderr, "\n");
    }
    double f = ev_ms(c->ev_fork, c->ev[7]);
    for (int cls = 0; cls < kNumClasses; ++cls) f = std::max(f, (double)ev_ms(c->ev_fork, c->ev_k1[cls]));
    fwd_ms += f;
    {
      // K5 runs on the class streams right after each class's forward: the
      // union of its [ev_k1, ev_tb] intervals, and how far it runs past the
      // forward phase
      std::pair<double, double> iv[kNumClasses];
      double tb_end = 0.0;
      for (int cls = 0; cls < kNumClasses; ++cls) {
        iv[cls] = {ev_ms(c->ev_fork, c->ev_k1[cls]), ev_ms(c->ev_fork, c->ev_tb[cls])};
        tb_end = std::max(tb_end, iv[cls].second);
      }
      std::sort(iv, iv + kNumClasses);
      double cur0 = iv[0].first, cur1 = iv[0].first, uni = 0.0;
      for (auto &x : iv) {
        if (x.first > cur1) { uni += cur1 - cur0; cur0 = x.first; cur1 = x.first; }
        cur1 = std::max(cur1, x.second);
      }
      uni += cur1 - cur0;
      tile_ms += uni;
      tail_ms += std::max(0.0, tb_end - f);
    }
    rev_ms += ev_ms(c->ev[2], c->ev[3]);
    wide += h_cnt[3 * kNumClasses];
    uint32_t deferred = 0;
    for (int cls = 0; cls < kNumClasses; ++cls) deferred += h_cnt[8 * kNumClasses + cls];
    if (deferred == 0) break;
    if (pround >= 1024) return fail(SW_EINTERNAL, "checkpoint pool too small for the batch");
  }
  CU(cudaEventRecord(c->ev[12], s));
  unsigned long long hstats[6] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
  CU(cudaMemcpyAsync(hstats, c->stats.p, sizeof(hstats), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (hstats[4] > c->pool.bytes) c->pool_want = (size_t)hstats[4];   // grow on the next call
  if (hstats[5])
    return fail(SW_EINVAL, std::to_string(hstats[5]) +
                               " pair(s) reference bytes outside the arena or exceed 65000 residues");
  if (tm) {
    tm->forward_ms += fwd_ms;
    tm->reverse_ms += rev_ms;
    tm->traceback_ms += tb_ms;
    tm->kernel_ms += ev_ms(c->ev[0], c->ev[12]);
    tm->cells += hstats[0];
    tm->launches += launches;
    tm->wide_pairs += wide;
    tm->host_plan_ms += h1 - h0;
    tm->host_setup_ms += h2 - h1;
    tm->tile_tb_ms += tile_ms;
    tm->fwd_tail_ms += tail_ms;
  }
  if (s != user_s) {
    CU(cudaEventRecord(c->ev_out, s));
    CU(cudaStreamWaitEvent(user_s, c->ev_out, 0));
  }
  return SW_OK;
}

// Pairs [k0, k1) of a HOST batch on `device`: the range's pair table and the
// arena bytes it references ([lo, hi), the whole arena for a whole batch)
// are uploaded on the copy stream -- the table first (the planning kernels
// need it), then the bytes in slices, each followed by a 4-byte copy that
// bumps `ready`; the packed forward starts as soon as its pairs' slices have
// landed, so the upload overlaps the forward pass.  Results go to `out`
// (pairs k0.. in order): host memory, or device memory when out_on_device.
int align_range(int device, const uint8_t *arena, uint64_t arena_bytes, const sw_pair_t *pairs,
                uint64_t k0, uint64_t k1, bool whole, const sw_params_t *params, sw_result_t *out,
                bool out_on_device, cudaStream_t user_stream, sw_timing_t *tm) {
  const double t0 = now_ms();
  const uint64_t n_pairs = k1 - k0;
  DeviceCtx *c = nullptr;
  int rc = get_ctx(device, &c);
  if (rc) return rc;
  std::lock_guard<std::mutex> g(c->mu);
  CU(cudaSetDevice(device));
  const double t_ctx = now_ms();
  if (tm) memset(tm, 0, sizeof(*tm));
  if (n_pairs == 0) return SW_OK;
  // the byte range the pairs reference (pairs outside the arena are left to
  // the device check: the range is clamped to the arena)
  uint64_t lo = 0, hi = arena_bytes;
  if (!whole) {   // a few threads for large ranges (one pass over the range's table)
    const int T = (int)std::max<uint64_t>(1, std::min<uint64_t>(8, n_pairs / 131072));
    std::vector<uint64_t> tlo(T, ~0ull), thi(T, 0);
    auto scan = [&](int t) {
      uint64_t l = ~0ull, h = 0;
      for (uint64_t k = k0 + n_pairs * t / T, e = k0 + n_pairs * (t + 1) / T; k < e; ++k) {
        const sw_pair_t &p = pairs[k];
        l = std::min(l, std::min(p.a_off, p.b_off));
        h = std::max(h, std::max(p.a_off + p.a_len, p.b_off + p.b_len));
      }
      tlo[t] = l;
      thi[t] = h;
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(scan, t);
    scan(0);
    for (auto &x : th) x.join();
    lo = *std::min_element(tlo.begin(), tlo.end());
    hi = std::min(*std::max_element(thi.begin(), thi.end()), arena_bytes);
    lo = std::min(lo, hi);
  }
  cudaStream_t s = user_stream ? user_stream : c->stream;
  const uint64_t span = hi - lo;
  CU(c->arena.ensure(span + 64));
  CU(c->pairs.ensure(n_pairs * sizeof(sw_pair_t)));
  if (!out_on_device) CU(c->out.ensure(n_pairs * sizeof(sw_result_t)));
  sw_result_t *d_out = out_on_device ? out : (sw_result_t *)c->out.p;
  cudaStream_t cs = c->copy_stream;
  // A pinned (device-mapped) host arena is gathered by the device itself, in
  // the order the packed pass consumes it (k_gather_arena): the forward of
  // the first duos does not wait for bytes it does not need.  Otherwise the
  // arena goes up by DMA in slices, each followed by a `ready` bump.
  static const int env_gather = [] {
    const char *e = getenv("PASTIS_SW_GATHER");
    return e ? atoi(e) : 1;
  }();
  const uint8_t *gsrc = nullptr;
  if (env_gather && span > 0) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, arena + lo) == cudaSuccess && at.type == cudaMemoryTypeHost &&
        at.devicePointer)
      gsrc = (const uint8_t *)at.devicePointer - lo;
    cudaGetLastError();
  }
  const uint64_t slice = std::max<uint64_t>((uint64_t)4 << 20, (span + kMaxSlices - 1) / kMaxSlices);
  const int nslices = gsrc ? 0 : (int)((span + slice - 1) / slice);
  CU(cudaEventRecord(c->ev[8], s));
  CU(cudaStreamWaitEvent(cs, c->ev[8], 0));
  CU(cudaMemsetAsync(c->readyb.p, 0, 4, cs));
  CU(cudaMemcpyAsync(c->pairs.p, pairs + k0, n_pairs * sizeof(sw_pair_t), cudaMemcpyHostToDevice, cs));
  CU(cudaEventRecord(c->ev_pairs, cs));
  for (int k = 0; k < nslices; ++k) {
    const uint64_t b0 = (uint64_t)k * slice, nb = std::min<uint64_t>(slice, span - b0);
    CU(cudaMemcpyAsync((uint8_t *)c->arena.p + b0, arena + lo + b0, nb, cudaMemcpyHostToDevice, cs));
    CU(cudaMemcpyAsync(c->readyb.p, c->slice_vals + k, 4, cudaMemcpyHostToDevice, cs));
  }
  if (!gsrc) CU(cudaEventRecord(c->ev_arena, cs));
  CU(cudaStreamWaitEvent(s, c->ev_pairs, 0));
  rc = run_device(c, (const uint8_t *)c->arena.p - lo, hi, (const sw_pair_t *)c->pairs.p, n_pairs,
                  params, d_out, s, tm, nslices > 0 ? (const uint32_t *)c->readyb.p : nullptr, slice,
                  c->ev_arena, lo, gsrc);
  if (rc) return rc;
  CU(cudaEventRecord(c->ev[10], s));
  if (!out_on_device)
    CU(cudaMemcpyAsync(out, d_out, n_pairs * sizeof(sw_result_t), cudaMemcpyDeviceToHost, s));
  CU(cudaEventRecord(c->ev[11], s));
  const double t_issued = now_ms();
  CU(cudaStreamSynchronize(s));
  if (getenv("PASTIS_SW_DEBUG_E2E")) {
    fprintf(stderr, "e2e: ctx=%.3f host_issue=%.3f pre_kernel(ev8->ev0)=%.3f kernel(ev0->ev10)=%.3f "
            "d2h=%.3f wall=%.3f\n", t_ctx - t0, t_issued - t0, ev_ms(c->ev[8], c->ev[0]),
            ev_ms(c->ev[0], c->ev[10]), ev_ms(c->ev[10], c->ev[11]), now_ms() - t0);
  }
  if (tm) {
    tm->h2d_ms = ev_ms(c->ev[8], c->ev_arena);   // overlaps the forward pass (gathered: incl. the wait)
    tm->d2h_ms = ev_ms(c->ev[10], c->ev[11]);
    tm->h2d_bytes = span + n_pairs * sizeof(sw_pair_t);
    tm->d2h_bytes = out_on_device ? 0 : n_pairs * sizeof(sw_result_t);
    tm->total_ms = now_ms() - t0;
  }
  return SW_OK;
}

int align_host(int device, const uint8_t *arena, uint64_t arena_bytes, const sw_pair_t *pairs,
               uint64_t n_pairs, const sw_params_t *params, sw_result_t *out, sw_timing_t *tm) {
  int rc = check_params(params);
  if (rc) return rc;
  if (n_pairs && (!pairs || !out)) return fail(SW_EINVAL, "NULL pairs/out");
  // pair bounds are checked on the device by k_classify (no host pass over the table)
  return align_range(device, arena, arena_bytes, pairs, 0, n_pairs, true, params, out, false,
                     nullptr, tm);
}

bool is_device_ptr(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Cell-balanced contiguous split of a batch into N ranges (the plan of
// sw_align_shard / sw_align_batch_multi): bounds[s] = the smallest k with
// N * cells(pairs[0, k)) >= s * total (cells = a_len * b_len), bounds[0] = 0,
// bounds[N] = n.  Every range's cells are within one pair's of total / N.
// Host version: per-chunk sums, then each chunk scans for the targets that
// fall inside it (several threads).
void plan_ranges_host(const sw_pair_t *pairs, uint64_t n, int N, uint64_t *bounds) {
  typedef unsigned __int128 u128;
  bounds[0] = 0;
  bounds[N] = n;
  if (N == 1) return;
  const int T = (int)std::max<uint64_t>(1, std::min<uint64_t>(16, n / 65536));
  std::vector<u128> part(T + 1, 0);
  auto cells = [&](uint64_t k) { return (uint64_t)pairs[k].a_len * pairs[k].b_len; };
  auto run = [&](auto &&fn) {
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(fn, t);
    fn(0);
    for (auto &x : th) x.join();
  };
  run([&](int t) {
    u128 acc = 0;
    for (uint64_t k = n * t / T, e = n * (t + 1) / T; k < e; ++k) acc += cells(k);
    part[t + 1] = acc;
  });
  for (int t = 0; t < T; ++t) part[t + 1] += part[t];
  const u128 total = part[T];
  for (int s = 1; s < N; ++s) bounds[s] = total == 0 ? 0 : n;
  if (total == 0) return;
  run([&](int t) {
    u128 acc = part[t];
    int s = 1;
    while (s < N && (u128)s * total <= acc * (u128)N) ++s;   // targets of earlier chunks
    for (uint64_t k = n * t / T, e = n * (t + 1) / T; k < e && s < N; ++k) {
      acc += cells(k);
      for (; s < N && acc * (u128)N >= (u128)s * total; ++s) bounds[s] = k + 1;
    }
  });
}

// The same plan on the device for a device-resident table (one sync).
__global__ void k_range_cells(const sw_pair_t *__restrict__ pairs, uint64_t n, uint64_t *cells) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) cells[k] = (uint64_t)pairs[k].a_len * pairs[k].b_len;
}
__global__ void k_range_bounds(const uint64_t *__restrict__ incl, uint64_t n, int N,
                               uint64_t *bounds) {
  typedef unsigned __int128 u128;
  const int s = threadIdx.x;
  if (s > N) return;
  if (s == 0 || s == N) { bounds[s] = s == 0 ? 0 : n; return; }
  const u128 total = incl[n - 1];
  if (total == 0) { bounds[s] = 0; return; }
  // smallest k with N * prefix(k) >= s * total, prefix(k) = incl[k - 1]
  uint64_t lo = 1, hi = n;
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if ((u128)incl[mid - 1] * (u128)N >= (u128)s * total) hi = mid;
    else lo = mid + 1;
  }
  bounds[s] = lo;
}

// byte span [lo, hi) the pairs of range `shard` reference (lo/hi preset to
// ~0 / 0): the device path encodes only that part of the arena
__global__ void k_range_span(const sw_pair_t *__restrict__ pairs, const uint64_t *__restrict__ bounds,
                             int shard, unsigned long long *span) {
  const uint64_t b = bounds[shard], e = bounds[shard + 1];
  unsigned long long lo = ~0ull, hi = 0ull;
  for (uint64_t k = b + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < e;
       k += (uint64_t)gridDim.x * blockDim.x) {
    const sw_pair_t p = pairs[k];
    lo = min(lo, (unsigned long long)min(p.a_off, p.b_off));
    hi = max(hi, (unsigned long long)max(p.a_off + p.a_len, p.b_off + p.b_len));
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&span[0], lo);
    atomicMax(&span[1], hi);
  }
}

// bounds[0..N] of the plan; with shard >= 0 also span[0..1] = the byte range
// that shard's pairs reference
int plan_ranges_device(DeviceCtx *c, const sw_pair_t *d_pairs, uint64_t n, int N, uint64_t *bounds,
                       cudaStream_t s, int shard = -1, uint64_t *span = nullptr) {
  CU(c->sh_cells.ensure(2 * n * sizeof(uint64_t) + (N + 3) * sizeof(uint64_t)));
  uint64_t *cells = (uint64_t *)c->sh_cells.p, *incl = cells + n, *db = incl + n;
  unsigned long long *dspan = (unsigned long long *)(db + N + 1);
  k_range_cells<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(d_pairs, n, cells);
  CU(cudaGetLastError());
  size_t tmp_bytes = 0;
  CU(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, cells, incl, (int)n, s));
  CU(c->cubtmp.ensure(tmp_bytes));
  CU(cub::DeviceScan::InclusiveSum(c->cubtmp.p, tmp_bytes, cells, incl, (int)n, s));
  k_range_bounds<<<1, 1024, 0, s>>>(incl, n, N, db);
  CU(cudaGetLastError());
  if (shard >= 0) {
    const unsigned long long init[2] = {~0ull, 0ull};
    CU(cudaMemcpyAsync(dspan, init, sizeof(init), cudaMemcpyHostToDevice, s));
    k_range_span<<<c->sms * 2, 256, 0, s>>>(d_pairs, db, shard, dspan);
    CU(cudaGetLastError());
  }
  std::vector<uint64_t> h(N + 3);
  CU(cudaMemcpyAsync(h.data(), db, (N + 3) * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  for (int k = 0; k <= N; ++k) bounds[k] = h[k];
  if (span) { span[0] = h[N + 1]; span[1] = h[N + 2]; }
  return SW_OK;
}

struct Square {
  __host__ __device__ uint64_t operator()(uint32_t c) const { return (uint64_t)c * c; }
};
struct Widen {
  __host__ __device__ uint64_t operator()(uint32_t c) const { return c; }
};
struct Flag {
  uint32_t t;
  __host__ __device__ uint64_t operator()(uint32_t c) const { return c >= t ? 1ull : 0ull; }
};

int bits_for(uint64_t v) {   // smallest b with v <= 2^b
  int b = 0;
  while (b < 64 && (1ull << b) < v) ++b;
  return b;
}

template <typename F>
int cub_call(DeviceCtx *c, F &&f) {   // two-phase CUB call with the shared temp buffer
  size_t bytes = 0;
  CU(f(nullptr, bytes));
  CU(c->cubtmp.ensure(bytes + 16));
  CU(f(c->cubtmp.p, bytes));
  return SW_OK;
}

int kmer_candidates(int device, const uint8_t *arena, uint64_t arena_bytes, const uint64_t *seq_off,
                    const uint32_t *seq_len, uint32_t n_seqs, int k, uint32_t min_shared,
                    sw_candidate_t *out, uint64_t out_cap, sw_kmer_stats_t *st) {
  if (!st) return fail(SW_EINVAL, "stats is NULL");
  memset(st, 0, sizeof(*st));
  if (k < 1) return fail(SW_EINVAL, "k must be >= 1");
  if (n_seqs && (!seq_off || !seq_len)) return fail(SW_EINVAL, "NULL sequence table");
  uint64_t space = 1;
  for (int t = 0; t < k; ++t) {
    if (space > (~0ull) / 25) return fail(SW_EINVAL, "25^k does not fit in 64 bits");
    space *= 25;
  }
  const int code_bits = bits_for(space);
  const int seq_bits = std::max(1, bits_for(n_seqs));
  if (code_bits + seq_bits > 64 || 2 * seq_bits > 64)
    return fail(SW_EINVAL, "k-mer code space and sequence count exceed 64-bit keys");
  std::vector<uint64_t> base(n_seqs + 1, 0);
  uint64_t P = 0;
  for (uint32_t s = 0; s < n_seqs; ++s) {
    if (seq_off[s] + seq_len[s] > arena_bytes) return fail(SW_EINVAL, "sequence outside the arena");
    base[s] = P;
    if (seq_len[s] >= (uint32_t)k) P += seq_len[s] - k + 1;
    else ++st->short_seqs;
  }
  base[n_seqs] = P;
  st->positions = P;
  if (P > 0x7FFFFFF0ull) return fail(SW_EINVAL, "too many k-mer positions in one call");
  DeviceCtx *c = nullptr;
  int rc = get_ctx(device, &c);
  if (rc) return rc;
  std::lock_guard<std::mutex> g(c->mu);
  CU(cudaSetDevice(device));
  cudaStream_t s = c->stream;
  if (P == 0) {
    st->performed = 0;
    return SW_OK;
  }
  CU(cudaEventRecord(c->ev[0], s));
  CU(c->km_arena.ensure(arena_bytes + 16));
  CU(c->km_off.ensure(n_seqs * 8 + 8));
  CU(c->km_len.ensure(n_seqs * 4 + 4));
  CU(c->km_base.ensure((n_seqs + 1) * 8));
  CU(c->km_keys.ensure(2 * P * 8));
  CU(c->km_small.ensure(64));
  CU(cudaMemcpyAsync(c->km_arena.p, arena, arena_bytes, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(c->km_off.p, seq_off, n_seqs * 8, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(c->km_len.p, seq_len, n_seqs * 4, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync(c->km_base.p, base.data(), (n_seqs + 1) * 8, cudaMemcpyHostToDevice, s));
  uint64_t *keys_a = (uint64_t *)c->km_keys.p, *keys_b = keys_a + P;
  // 1. keys of every occurrence
  k_kmer_keys<<<(unsigned)std::min<uint64_t>((n_seqs + 7) / 8, (uint64_t)c->sms * 16), 256, 0, s>>>(
      (const uint8_t *)c->km_arena.p, (const uint64_t *)c->km_off.p, (const uint32_t *)c->km_len.p,
      (const uint64_t *)c->km_base.p, n_seqs, k, seq_bits, (const uint8_t *)c->lut.p, keys_a);
  CU(cudaGetLastError());
  // 2. sort + unique (code, seq)
  const int key_bits = code_bits + seq_bits;
  rc = cub_call(c, [&](void *t, size_t &b) {
    return cub::DeviceRadixSort::SortKeys(t, b, keys_a, keys_b, (int)P, 0, key_bits, s);
  });
  if (rc) return rc;
  uint64_t *nsel = (uint64_t *)c->km_small.p;   // [0] unique, [1] runs, [2] pairs, [3] flops
  rc = cub_call(c, [&](void *t, size_t &b) {
    return cub::DeviceSelect::Unique(t, b, keys_b, keys_a, nsel, (int)P, s);
  });
  if (rc) return rc;
  uint64_t U = 0;
  CU(cudaMemcpyAsync(&U, nsel, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  st->distinct = U;
  // 3. buckets = runs of equal code
  CU(c->km_runs.ensure(U * (8 + 4 + 8 + 8) + 64));
  uint64_t *run_code = (uint64_t *)c->km_runs.p;
  uint32_t *run_cnt = (uint32_t *)(run_code + U);
  uint64_t *run_start = (uint64_t *)(((uintptr_t)(run_cnt + U) + 15) & ~(uintptr_t)15);
  uint64_t *run_emit = run_start + U;
  auto codes_it = thrust::make_transform_iterator(keys_a, KeyShift{seq_bits});
  rc = cub_call(c, [&](void *t, size_t &b) {
    return cub::DeviceRunLengthEncode::Encode(t, b, codes_it, run_code, run_cnt, nsel + 1, (int)U, s);
  });
  if (rc) return rc;
  uint64_t R = 0;
  CU(cudaMemcpyAsync(&R, nsel + 1, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  st->buckets = R;
  auto cnt_it = thrust::make_transform_iterator(run_cnt, Widen{});
  auto emit_it = thrust::make_transform_iterator(run_cnt, PairsOf{});
  auto sq_it = thrust::make_transform_iterator(run_cnt, Square{});
  rc = cub_call(c, [&](void *t, size_t &b) {
    return cub::DeviceScan::ExclusiveSum(t, b, cnt_it, run_start, (int)R, s);
  });
  if (rc) return rc;
  rc = cub_call(c, [&](void *t, size_t &b) {
    return cub::DeviceScan::ExclusiveSum(t, b, emit_it, run_emit, (int)R, s);
  });
  if (rc) return rc;
  rc = cub_call(c, [&](void *t, size_t &b) {
    return cub::DeviceReduce::Sum(t, b, sq_it, nsel + 3, (int)R, s);
  });
  if (rc) return rc;
  uint64_t last_off = 0, flops = 0;
  uint32_t last_cnt = 0;
  CU(cudaMemcpyAsync(&last_off, run_emit + (R - 1), 8, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&last_cnt, run_cnt + (R - 1), 4, cudaMemcpyDeviceToHost, s));
  CU(cudaMemcpyAsync(&flops, nsel + 3, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  const uint64_t E = last_off + (uint64_t)last_cnt * (last_cnt - 1) / 2;
  st->emitted = E;
  st->flops = flops;
  if (E > 0x7FFFFFF0ull) return fail(SW_EINVAL, "too many shared-k-mer pair emissions in one call");
  uint64_t D = 0, C = 0;
  if (E > 0) {
    // 4. pairs of every bucket
    CU(c->km_pairs.ensure(2 * E * 8 + E * 4 + 64));
    uint64_t *pairs_a = (uint64_t *)c->km_pairs.p, *pairs_b = pairs_a + E;
    uint32_t *pcnt = (uint32_t *)(pairs_b + E);   // shared count per distinct pair
    k_bucket_pairs<<<(unsigned)std::min<uint64_t>((R + 7) / 8, (uint64_t)c->sms * 16), 256, 0, s>>>(
        keys_a, run_cnt, run_start, run_emit, R, seq_bits, pairs_a);
    CU(cudaGetLastError());
    // 5. sort pair keys, count runs
    rc = cub_call(c, [&](void *t, size_t &b) {
      return cub::DeviceRadixSort::SortKeys(t, b, pairs_a, pairs_b, (int)E, 0, 2 * seq_bits, s);
    });
    if (rc) return rc;
    // distinct pairs into pairs_a, their counts into pcnt
    rc = cub_call(c, [&](void *t, size_t &b) {
      return cub::DeviceRunLengthEncode::Encode(t, b, pairs_b, pairs_a, pcnt, nsel + 2, (int)E, s);
    });
    if (rc) return rc;
    CU(cudaMemcpyAsync(&D, nsel + 2, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    // threshold + order-preserving compaction
    uint64_t *cursor = pairs_b;   // free now (E >= D)
    auto flag_it = thrust::make_transform_iterator(pcnt, Flag{min_shared});
    rc = cub_call(c, [&](void *t, size_t &b) {
      return cub::DeviceScan::ExclusiveSum(t, b, flag_it, cursor, (int)D, s);
    });
    if (rc) return rc;
    uint64_t last_cur = 0;
    uint32_t last_pc = 0;
    CU(cudaMemcpyAsync(&last_cur, cursor + (D - 1), 8, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(&last_pc, pcnt + (D - 1), 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    C = last_cur + (last_pc >= min_shared ? 1 : 0);
    if (C > 0) {
      CU(c->km_out.ensure(C * sizeof(sw_candidate_t)));
      k_write_candidates<<<(unsigned)std::min<uint64_t>((D + 255) / 256, (uint64_t)c->sms * 16), 256,
                           0, s>>>(pairs_a, pcnt, D, seq_bits, min_shared, cursor,
                                   (sw_candidate_t *)c->km_out.p);
      CU(cudaGetLastError());
    }
  }
  CU(cudaEventRecord(c->ev[1], s));
  CU(cudaStreamSynchronize(s));
  st->discovered = D;
  st->performed = C;
  st->device_ms = ev_ms(c->ev[0], c->ev[1]);
  if (C > out_cap) return fail(SW_ERANGE, "candidate buffer too small (see stats->performed)");
  if (C > 0) {
    if (!out) return fail(SW_EINVAL, "NULL candidate buffer");
    CU(cudaMemcpy(out, c->km_out.p, C * sizeof(sw_candidate_t), cudaMemcpyDeviceToHost));
  }
  return SW_OK;
}

}  // namespace

extern "C" {

int sw_abi_version(void) { return SW_ABI_VERSION; }

int sw_get_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

const char *sw_last_error(void) { return g_err.c_str(); }
#ifdef K5_COUNT
int sw_debug_k5_counters(unsigned long long *out) {   // debug builds only
  cudaMemcpyFromSymbol(out, pastis::g_k5c, sizeof(unsigned long long) * 8);
  static const unsigned long long zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  return (int)cudaMemcpyToSymbol(pastis::g_k5c, zero, sizeof(zero));
}
#endif

int sw_align_batch(int device, const uint8_t *arena, uint64_t arena_bytes, const sw_pair_t *pairs,
                   uint64_t n_pairs, const sw_params_t *params, sw_result_t *out,
                   sw_timing_t *timing) {
  return align_host(device, arena, arena_bytes, pairs, n_pairs, params, out, timing);
}

int sw_align_batch_device(int device, const uint8_t *d_arena, uint64_t arena_bytes,
                          const sw_pair_t *d_pairs, uint64_t n_pairs, const sw_params_t *params,
                          sw_result_t *d_out, void *stream, sw_timing_t *timing) {
  const double t0 = now_ms();
  int rc = check_params(params);
  if (rc) return rc;
  DeviceCtx *c = nullptr;
  rc = get_ctx(device, &c);
  if (rc) return rc;
  std::lock_guard<std::mutex> g(c->mu);
  CU(cudaSetDevice(device));
  if (timing) memset(timing, 0, sizeof(*timing));
  cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
  rc = run_device(c, d_arena, arena_bytes, d_pairs, n_pairs, params, d_out, s, timing);
  if (rc) return rc;
  CU(cudaStreamSynchronize(s));
  if (timing) timing->total_ms = now_ms() - t0;
  return SW_OK;
}

int sw_partition_pairs(const sw_pair_t *pairs, uint64_t n_pairs, int n_shards, int32_t *shard,
                       uint64_t *load) {
  // the plan of sw_align_shard / sw_align_batch_multi, per pair
  if (n_shards < 1) return fail(SW_EINVAL, "n_shards < 1");
  if (n_pairs && (!pairs || !shard)) return fail(SW_EINVAL, "NULL pairs/shard");
  std::vector<uint64_t> b(n_shards + 1);
  plan_ranges_host(pairs, n_pairs, n_shards, b.data());
  for (int s = 0; s < n_shards; ++s) {
    uint64_t ld = 0;
    for (uint64_t k = b[s]; k < b[s + 1]; ++k) {
      shard[k] = s;
      ld += (uint64_t)pairs[k].a_len * pairs[k].b_len;
    }
    if (load) load[s] = ld;
  }
  return SW_OK;
}

int sw_shard_ranges(const sw_pair_t *pairs, uint64_t n_pairs, int n_shards, uint64_t *bounds) {
  if (n_shards < 1 || !bounds) return fail(SW_EINVAL, "bad n_shards / bounds");
  if (n_pairs && !pairs) return fail(SW_EINVAL, "NULL pairs");
  if (n_pairs && is_device_ptr(pairs)) {
    cudaPointerAttributes at;
    CU(cudaPointerGetAttributes(&at, pairs));
    DeviceCtx *c = nullptr;
    int rc = get_ctx(at.device, &c);
    if (rc) return rc;
    std::lock_guard<std::mutex> g(c->mu);
    CU(cudaSetDevice(at.device));
    return plan_ranges_device(c, pairs, n_pairs, n_shards, bounds, c->stream);
  }
  plan_ranges_host(pairs, n_pairs, n_shards, bounds);
  return SW_OK;
}

int sw_align_shard(int device, const uint8_t *arena, uint64_t arena_bytes, const sw_pair_t *pairs,
                   uint64_t n_pairs, int shard, int n_shards, const sw_params_t *params,
                   sw_result_t *d_out, uint64_t *range, void *stream, sw_timing_t *timing) {
  const double t0 = now_ms();
  int rc = check_params(params);
  if (rc) return rc;
  if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(SW_EINVAL, "bad shard / n_shards");
  if (n_pairs && (!arena || !pairs || !d_out)) return fail(SW_EINVAL, "NULL buffer");
  if (timing) memset(timing, 0, sizeof(*timing));
  std::vector<uint64_t> b(n_shards + 1, 0);
  const bool dev_pairs = n_pairs && is_device_ptr(pairs);
  if (dev_pairs != (n_pairs && is_device_ptr(arena)))
    return fail(SW_EINVAL, "arena and pairs must both be device or both be host memory");
  if (dev_pairs) {
    // everything resident on the device: plan there, align the range in place
    DeviceCtx *c = nullptr;
    rc = get_ctx(device, &c);
    if (rc) return rc;
    std::lock_guard<std::mutex> g(c->mu);
    CU(cudaSetDevice(device));
    cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
    const double h0 = now_ms();
    uint64_t span[2] = {0, 0};
    rc = plan_ranges_device(c, pairs, n_pairs, n_shards, b.data(), s, shard, span);
    if (rc) return rc;
    if (timing) timing->host_plan_ms += now_ms() - h0;
    if (range) { range[0] = b[shard]; range[1] = b[shard + 1]; }
    // only the arena bytes this range references are encoded (clamped: pairs
    // outside the arena are rejected by the planning kernel)
    const uint64_t hi = std::min<uint64_t>(span[1], arena_bytes), lo = std::min(span[0], hi);
    rc = run_device(c, arena, hi, pairs + b[shard], b[shard + 1] - b[shard], params, d_out, s,
                    timing, nullptr, 0, nullptr, lo);
    if (rc) return rc;
    CU(cudaStreamSynchronize(s));
  } else {
    const double h0 = now_ms();
    plan_ranges_host(pairs, n_pairs, n_shards, b.data());
    const double h1 = now_ms();
    if (range) { range[0] = b[shard]; range[1] = b[shard + 1]; }
    rc = align_range(device, arena, arena_bytes, pairs, b[shard], b[shard + 1], false, params, d_out,
                     true, (cudaStream_t)stream, timing);
    if (rc) return rc;
    if (timing) timing->host_plan_ms += h1 - h0;
  }
  if (timing) timing->total_ms = now_ms() - t0;
  return SW_OK;
}

int sw_align_batch_multi(int n_devices, const int *devices, const uint8_t *arena,
                         uint64_t arena_bytes, const sw_pair_t *pairs, uint64_t n_pairs,
                         const sw_params_t *params, sw_result_t *out,
                         sw_timing_t *per_device_timing) {
  if (n_devices < 1 || !devices) return fail(SW_EINVAL, "need at least one device");
  int rc = check_params(params);
  if (rc) return rc;
  if (n_devices == 1)
    return align_host(devices[0], arena, arena_bytes, pairs, n_pairs, params, out,
                      per_device_timing);
  if (n_pairs && (!arena || !pairs || !out)) return fail(SW_EINVAL, "NULL buffer");
  const double h0 = now_ms();
  std::vector<uint64_t> b(n_devices + 1);
  plan_ranges_host(pairs, n_pairs, n_devices, b.data());
  const double plan_ms = now_ms() - h0;
  struct Lane {
    int rc = 0;
    std::string err;
  };
  std::vector<Lane> lanes(n_devices);
  std::vector<std::thread> th;
  for (int d = 0; d < n_devices; ++d) {
    th.emplace_back([&, d]() {
      sw_timing_t *tm = per_device_timing ? per_device_timing + d : nullptr;
      Lane &L = lanes[d];
      // each GPU uploads only its range's pairs and the bytes they reference
      // (overlapped with its forward pass) and writes its results straight
      // into the caller's buffer: the ranges are contiguous in input order
      L.rc = align_range(devices[d], arena, arena_bytes, pairs, b[d], b[d + 1], false, params,
                         out + b[d], false, nullptr, tm);
      if (L.rc) L.err = g_err;
      if (tm) tm->host_plan_ms += plan_ms;
    });
  }
  for (auto &t : th) t.join();
  for (int d = 0; d < n_devices; ++d)
    if (lanes[d].rc)
      return fail(lanes[d].rc, "device " + std::to_string(devices[d]) + ": " + lanes[d].err);
  return SW_OK;
}

int sw_fasta_parse(const uint8_t *text, uint64_t text_bytes, uint8_t *arena, uint8_t *headers,
                   sw_fasta_rec_t *recs, uint64_t recs_cap, sw_fasta_info_t *info) {
  if (!info || (text_bytes && (!text || !arena || !headers || (!recs && recs_cap))))
    return fail(SW_EINVAL, "sw_fasta_parse: NULL buffer");
  const int rc = pastis_fasta::parse(text, text_bytes, arena, headers, recs, recs_cap, info);
  if (rc == SW_EINVAL) return fail(SW_EINVAL, "sw_fasta_parse: recs_cap too small");
  if (rc == SW_EFORMAT) return fail(SW_EFORMAT, "malformed FASTA text");
  return rc;
}

int sw_kmer_candidates(int device, const uint8_t *arena, uint64_t arena_bytes,
                       const uint64_t *seq_off, const uint32_t *seq_len, uint32_t n_seqs, int k,
                       uint32_t min_shared, sw_candidate_t *out, uint64_t out_cap,
                       sw_kmer_stats_t *stats) {
  return kmer_candidates(device, arena, arena_bytes, seq_off, seq_len, n_seqs, k, min_shared, out,
                         out_cap, stats);
}

void sw_release(int device) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  for (size_t d = 0; d < g_ctx.size(); ++d) {
    if (device >= 0 && (int)d != device) continue;
    DeviceCtx *c = g_ctx[d];
    if (!c) continue;
    std::lock_guard<std::mutex> g2(c->mu);
    cudaSetDevice((int)d);
    for (DevBuf *b : {&c->arena, &c->codes, &c->pairs, &c->out, &c->st, &c->lists, &c->ctrs,
                      &c->stats, &c->bnd, &c->pool, &c->skeys, &c->svals, &c->cubtmp,
                      &c->km_arena, &c->km_off, &c->km_len, &c->km_base, &c->km_keys, &c->km_runs,
                      &c->km_pairs, &c->km_out, &c->km_small, &c->cta_rows, &c->sh_cells})
      b->release();
    c->pool_want = 0;
  }
}

// Debug aid (not part of the public header): copy the per-pair scratch state
// (PairState, 48 B each) of the last batch run on `device` to host memory.
int sw_debug_pair_state(int device, void *host_out, uint64_t n_pairs) {
  DeviceCtx *c = nullptr;
  int rc = get_ctx(device, &c);
  if (rc) return rc;
  std::lock_guard<std::mutex> g(c->mu);
  CU(cudaSetDevice(device));
  if (n_pairs * sizeof(PairState) > c->st.bytes) return fail(SW_EINVAL, "n_pairs too large");
  CU(cudaMemcpy(host_out, c->st.p, n_pairs * sizeof(PairState), cudaMemcpyDeviceToHost));
  return SW_OK;
}

int sw_debug_pool(int device, void *host_out, uint64_t bytes) {
  DeviceCtx *c = nullptr;
  int rc = get_ctx(device, &c);
  if (rc) return rc;
  std::lock_guard<std::mutex> g(c->mu);
  CU(cudaSetDevice(device));
  if (bytes > c->pool.bytes) return fail(SW_EINVAL, "bytes too large");
  CU(cudaMemcpy(host_out, c->pool.p, bytes, cudaMemcpyDeviceToHost));
  return SW_OK;
}

void *sw_host_alloc(uint64_t bytes) {
  void *p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    g_err = "cudaHostAlloc failed";
    return nullptr;
  }
  return p;
}

void sw_host_free(void *p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
