/*
 * TEST INFRASTRUCTURE ONLY -- the parity oracle for the GPU aligner.
 *
 * Plain-C restatement of the reference CPU aligner
 *   /root/reference/pkg/src/pastislite/align.py:79-181  (_smith_waterman_timed)
 * using the cell-form Gotoh recurrence of the reference's independent oracle
 *   /root/reference/pkg/src/pastislite/oracle.py:60-82  (fill + strict '>' argmax)
 * which align.py:113-121 (prefix-max E) equals exactly whenever
 * gap_open >= gap_extend (enforced by AlignParams, align.py:45-47).
 * The traceback state machine is align.py:133-169 line for line in meaning:
 *   H state: h==0 -> stop; h==H[i-1][j-1]+s -> diag; h==F -> F; h==E -> E
 *   F state: step up; back to H iff F[i][j]==H[i-1][j]-open
 *   E state: step left; back to H iff E[i][j]==H[i][j-1]-open
 * matches compares the raw input BYTES (align.py:142 compares characters),
 * scores use the byte->index LUT of align.py:27-30 (unknown byte -> 'X').
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py -> tests/golden/ fixtures; tests/test_oracle.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path never does.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORC_ALPHABET "ARNDCQEGHILKMFPSTWYVBZXU*"
#define ORC_SIZE 25
#define ORC_X 22
#define ORC_NEG (-(1 << 29)) /* align.py:25 */

typedef struct { /* same layout as include/pastis_sw.h sw_pair_t */
  uint64_t a_off;
  uint64_t b_off;
  uint32_t a_len;
  uint32_t b_len;
} orc_pair_t;

static void build_lut(uint8_t lut[256]) { /* align.py:27-30 */
  for (int c = 0; c < 256; ++c) lut[c] = ORC_X;
  for (int k = 0; k < ORC_SIZE; ++k) lut[(uint8_t)ORC_ALPHABET[k]] = (uint8_t)k;
}

/* out[0..6] = score, i_begin, i_end, j_begin, j_end, matches, aln_len.
 * returns 0 ok, 1 empty input (AlignmentError, align.py:81-82),
 * -1 out of memory, -2 traceback lost (align.py:150/159/168 assertions). */
int orc_align(const uint8_t *a, int64_t m, const uint8_t *b, int64_t n, int32_t open_,
              int32_t ext, const int32_t *matrix, int32_t *out) {
  for (int k = 0; k < 7; ++k) out[k] = 0;
  if (m <= 0 || n <= 0) return 1;
  uint8_t lut[256];
  build_lut(lut);
  const int64_t W = n + 1;
  const size_t cells = (size_t)(m + 1) * (size_t)W;
  int32_t *H = (int32_t *)malloc(cells * sizeof(int32_t));
  int32_t *E = (int32_t *)malloc(cells * sizeof(int32_t));
  int32_t *F = (int32_t *)malloc(cells * sizeof(int32_t));
  uint8_t *bi = (uint8_t *)malloc((size_t)n);
  if (!H || !E || !F || !bi) {
    free(H); free(E); free(F); free(bi);
    return -1;
  }
  for (int64_t j = 0; j < n; ++j) bi[j] = lut[b[j]];
  /* align.py:92-96: H zero boundary, E[:,0] = F[0,:] = _NEG */
  for (int64_t j = 0; j <= n; ++j) { H[j] = 0; F[j] = ORC_NEG; E[j] = ORC_NEG; }
  int32_t best = 0;
  int64_t bi_end = 0, bj_end = 0;
  for (int64_t i = 1; i <= m; ++i) { /* align.py:104-121 / oracle.py:60-82 */
    int32_t *Hi = H + i * W, *Hp = H + (i - 1) * W;
    int32_t *Ei = E + i * W, *Fi = F + i * W, *Fp = F + (i - 1) * W;
    const int32_t *row = matrix + (size_t)lut[a[i - 1]] * ORC_SIZE;
    Hi[0] = 0; Ei[0] = ORC_NEG; Fi[0] = ORC_NEG;
    for (int64_t j = 1; j <= n; ++j) {
      int32_t e = Hi[j - 1] - open_, e2 = Ei[j - 1] - ext;
      if (e2 > e) e = e2;
      int32_t f = Hp[j] - open_, f2 = Fp[j] - ext;
      if (f2 > f) f = f2;
      int32_t h = Hp[j - 1] + row[bi[j - 1]];
      if (e > h) h = e;
      if (f > h) h = f;
      if (h < 0) h = 0;
      Ei[j] = e; Fi[j] = f; Hi[j] = h;
      if (h > best) { best = h; bi_end = i; bj_end = j; } /* row-major first max, align.py:124 */
    }
  }
  int rc = 0;
  if (best == 0) { /* align.py:127-128 */
    out[0] = 0; out[1] = out[2] = out[3] = out[4] = -1; out[5] = out[6] = 0;
    goto done;
  }
  {
    int64_t i = bi_end, j = bj_end;
    int32_t matches = 0, aln_len = 0;
    int state = 0; /* 0 H, 1 F, 2 E  (align.py:135-169) */
    for (;;) {
      if (state == 0) {
        int32_t h = H[i * W + j];
        if (h == 0) break;
        int32_t s = matrix[(size_t)lut[a[i - 1]] * ORC_SIZE + bi[j - 1]];
        if (h == H[(i - 1) * W + j - 1] + s) {
          matches += (a[i - 1] == b[j - 1]);
          aln_len += 1; i -= 1; j -= 1;
        } else if (h == F[i * W + j]) {
          state = 1;
        } else if (h == E[i * W + j]) {
          state = 2;
        } else { rc = -2; goto done; }
      } else if (state == 1) {
        int32_t f = F[i * W + j];
        aln_len += 1;
        int32_t close = H[(i - 1) * W + j] - open_;
        i -= 1;
        if (f == close) state = 0;
        else if (f != F[i * W + j] - ext) { rc = -2; goto done; }
      } else {
        int32_t e = E[i * W + j];
        aln_len += 1;
        int32_t close = H[i * W + j - 1] - open_;
        j -= 1;
        if (e == close) state = 0;
        else if (e != E[i * W + j] - ext) { rc = -2; goto done; }
      }
    }
    out[0] = best; out[1] = (int32_t)i; out[2] = (int32_t)(bi_end - 1);
    out[3] = (int32_t)j; out[4] = (int32_t)(bj_end - 1);
    out[5] = matches; out[6] = aln_len;
  }
done:
  free(H); free(E); free(F); free(bi);
  return rc;
}

/* Score-only forward pass in O(n) memory: best and the row-major-first end
 * cell.  Same recurrence as orc_align; used to check very large pairs. */
int orc_score(const uint8_t *a, int64_t m, const uint8_t *b, int64_t n, int32_t open_,
              int32_t ext, const int32_t *matrix, int32_t *out3) {
  out3[0] = 0; out3[1] = out3[2] = -1;
  if (m <= 0 || n <= 0) return 1;
  uint8_t lut[256];
  build_lut(lut);
  int32_t *Hrow = (int32_t *)malloc((size_t)(n + 1) * 4);
  int32_t *Frow = (int32_t *)malloc((size_t)(n + 1) * 4);
  uint8_t *bi = (uint8_t *)malloc((size_t)n);
  if (!Hrow || !Frow || !bi) { free(Hrow); free(Frow); free(bi); return -1; }
  for (int64_t j = 0; j < n; ++j) bi[j] = lut[b[j]];
  for (int64_t j = 0; j <= n; ++j) { Hrow[j] = 0; Frow[j] = ORC_NEG; }
  int32_t best = 0;
  for (int64_t i = 1; i <= m; ++i) {
    const int32_t *row = matrix + (size_t)lut[a[i - 1]] * ORC_SIZE;
    int32_t hdiag = 0, hleft = 0, eleft = ORC_NEG;
    for (int64_t j = 1; j <= n; ++j) {
      int32_t e = hleft - open_, e2 = eleft - ext;
      if (e2 > e) e = e2;
      int32_t f = Hrow[j] - open_, f2 = Frow[j] - ext;
      if (f2 > f) f = f2;
      int32_t h = hdiag + row[bi[j - 1]];
      if (e > h) h = e;
      if (f > h) h = f;
      if (h < 0) h = 0;
      hdiag = Hrow[j];
      Hrow[j] = h; Frow[j] = f; hleft = h; eleft = e;
      if (h > best) { best = h; out3[1] = (int32_t)(i - 1); out3[2] = (int32_t)(j - 1); }
    }
  }
  out3[0] = best;
  free(Hrow); free(Frow); free(bi);
  return 0;
}

/* Exact alignment of one pair in O(sqrt(m) n) memory -- the independent
 * long-pair checker (pairs up to 65,000 x 65,000 residues, where orc_align's
 * 16 B/cell matrices would need 67 GB).  Same recurrence, end cell and
 * traceback state machine as orc_align (align.py:103-169); only the storage
 * differs:
 *   1. orc_score: best and the row-major-first end cell (align.py:124);
 *   2. a second forward pass over the prefix rows 0..I, cols 0..J (I, J =
 *      end cell + 1: the DP only looks up and left, so these values equal
 *      the full matrix's) keeps the (H, F) rows 0, K, 2K, ... as checkpoints;
 *   3. the traceback walks up the prefix one block of K rows at a time: the
 *      block (cK, (c+1)K] is recomputed from checkpoint row cK into full
 *      H/E/F rows and the state machine runs while i stays inside it.
 * Cost <= 3 m n cell updates.  Returns as orc_align. */
int orc_align_long(const uint8_t *a, int64_t m, const uint8_t *b, int64_t n, int32_t open_,
                   int32_t ext, const int32_t *matrix, int32_t *out) {
  for (int k = 0; k < 7; ++k) out[k] = 0;
  if (m <= 0 || n <= 0) return 1;
  int32_t sc[3];
  int rc = orc_score(a, m, b, n, open_, ext, matrix, sc);
  if (rc) return rc;
  if (sc[0] == 0) {
    out[0] = 0; out[1] = out[2] = out[3] = out[4] = -1; out[5] = out[6] = 0;
    return 0;
  }
  const int32_t best = sc[0];
  const int64_t I = (int64_t)sc[1] + 1, J = (int64_t)sc[2] + 1, W = J + 1;
  int64_t K = 32;
  while (K * K < I && K < 4096) K *= 2;
  const int64_t nck = I / K + 1;
  uint8_t lut[256];
  build_lut(lut);
  uint8_t *bi = (uint8_t *)malloc((size_t)J);
  int32_t *ckH = (int32_t *)malloc((size_t)nck * W * 4), *ckF = (int32_t *)malloc((size_t)nck * W * 4);
  int32_t *H = (int32_t *)malloc((size_t)(K + 1) * W * 4), *E = (int32_t *)malloc((size_t)(K + 1) * W * 4);
  int32_t *F = (int32_t *)malloc((size_t)(K + 1) * W * 4);
  if (!bi || !ckH || !ckF || !H || !E || !F) { rc = -1; goto done; }
  for (int64_t j = 0; j < J; ++j) bi[j] = lut[b[j]];
  /* 2. checkpoint pass: rolling rows in H[0], F[0] */
  {
    int32_t *Hr = H, *Fr = F;
    for (int64_t j = 0; j <= J; ++j) { Hr[j] = 0; Fr[j] = ORC_NEG; }
    memcpy(ckH, Hr, W * 4); memcpy(ckF, Fr, W * 4);
    for (int64_t i = 1; i <= I; ++i) {
      const int32_t *row = matrix + (size_t)lut[a[i - 1]] * ORC_SIZE;
      int32_t hdiag = 0, hleft = 0, eleft = ORC_NEG;
      for (int64_t j = 1; j <= J; ++j) {
        int32_t e = hleft - open_, e2 = eleft - ext;
        if (e2 > e) e = e2;
        int32_t f = Hr[j] - open_, f2 = Fr[j] - ext;
        if (f2 > f) f = f2;
        int32_t h = hdiag + row[bi[j - 1]];
        if (e > h) h = e;
        if (f > h) h = f;
        if (h < 0) h = 0;
        hdiag = Hr[j];
        Hr[j] = h; Fr[j] = f; hleft = h; eleft = e;
      }
      if (i % K == 0) { memcpy(ckH + (i / K) * W, Hr, W * 4); memcpy(ckF + (i / K) * W, Fr, W * 4); }
    }
  }
  /* 3. block-wise traceback */
  {
    int64_t i = I, j = J, blk = -1;
    int32_t matches = 0, aln_len = 0;
    int state = 0;
#define AT(M, ii, jj) (M)[((ii) - blk * K) * W + (jj)]
    for (;;) {
      const int64_t c = (i - 1) / K;       /* block holding row i: rows (cK, (c+1)K] */
      if (i >= 1 && c != blk) {
        blk = c;
        const int64_t r0 = c * K, r1 = (c + 1) * K < I ? (c + 1) * K : I;
        memcpy(H, ckH + c * W, W * 4);
        memcpy(F, ckF + c * W, W * 4);
        for (int64_t jj = 0; jj <= J; ++jj) E[jj] = ORC_NEG;
        for (int64_t ii = r0 + 1; ii <= r1; ++ii) {
          int32_t *Hi = H + (ii - r0) * W, *Hp = Hi - W, *Ei = E + (ii - r0) * W;
          int32_t *Fi = F + (ii - r0) * W, *Fp = Fi - W;
          const int32_t *row = matrix + (size_t)lut[a[ii - 1]] * ORC_SIZE;
          Hi[0] = 0; Ei[0] = ORC_NEG; Fi[0] = ORC_NEG;
          for (int64_t jj = 1; jj <= J; ++jj) {
            int32_t e = Hi[jj - 1] - open_, e2 = Ei[jj - 1] - ext;
            if (e2 > e) e = e2;
            int32_t f = Hp[jj] - open_, f2 = Fp[jj] - ext;
            if (f2 > f) f = f2;
            int32_t h = Hp[jj - 1] + row[bi[jj - 1]];
            if (e > h) h = e;
            if (f > h) h = f;
            if (h < 0) h = 0;
            Ei[jj] = e; Fi[jj] = f; Hi[jj] = h;
          }
        }
      }
      if (state == 0) {
        const int32_t h = AT(H, i, j);
        if (h == 0) break;
        const int32_t s = matrix[(size_t)lut[a[i - 1]] * ORC_SIZE + bi[j - 1]];
        if (h == AT(H, i - 1, j - 1) + s) {
          matches += (a[i - 1] == b[j - 1]);
          aln_len += 1; i -= 1; j -= 1;
        } else if (h == AT(F, i, j)) {
          state = 1;
        } else if (h == AT(E, i, j)) {
          state = 2;
        } else { rc = -2; goto done; }
      } else if (state == 1) {
        const int32_t f = AT(F, i, j);
        aln_len += 1;
        const int32_t close = AT(H, i - 1, j) - open_, ext_from = AT(F, i - 1, j) - ext;
        i -= 1;
        if (f == close) state = 0;
        else if (f != ext_from) { rc = -2; goto done; }
        if (i == 0) { rc = -2; goto done; }
      } else {
        const int32_t e = AT(E, i, j);
        aln_len += 1;
        const int32_t close = AT(H, i, j - 1) - open_;
        const int32_t ext_from = AT(E, i, j - 1) - ext;
        j -= 1;
        if (e == close) state = 0;
        else if (e != ext_from) { rc = -2; goto done; }
      }
      if (i == 0 || j == 0) {   /* H(0, *) = H(*, 0) = 0: the walk stops there */
        if (state != 0) { rc = -2; goto done; }
        break;
      }
    }
#undef AT
    out[0] = best; out[1] = (int32_t)i; out[2] = (int32_t)(I - 1);
    out[3] = (int32_t)j; out[4] = (int32_t)(J - 1);
    out[5] = matches; out[6] = aln_len;
  }
done:
  free(bi); free(ckH); free(ckF); free(H); free(E); free(F);
  return rc;
}

/* ---- threaded batch driver (CPU baseline; same pair table as the C-ABI) ---- */
typedef struct {
  const uint8_t *arena;
  const orc_pair_t *pairs;
  int64_t n_pairs;
  int32_t open_, ext;
  const int32_t *matrix;
  int32_t *out; /* 8 int32 per pair: 7 fields + status */
  int64_t next;
  int long_mode; /* 1: orc_align_long */
  pthread_mutex_t mu;
} orc_job_t;

static void *orc_worker(void *arg) {
  orc_job_t *job = (orc_job_t *)arg;
  for (;;) {
    pthread_mutex_lock(&job->mu);
    int64_t k = job->next;
    job->next += 1;
    pthread_mutex_unlock(&job->mu);
    if (k >= job->n_pairs) break;
    const orc_pair_t *p = job->pairs + k;
    int32_t *o = job->out + 8 * k;
    int rc = (job->long_mode ? orc_align_long : orc_align)(
        job->arena + p->a_off, p->a_len, job->arena + p->b_off, p->b_len, job->open_, job->ext,
        job->matrix, o);
    o[7] = rc;
  }
  return NULL;
}

int orc_align_batch_mode(const uint8_t *arena, const orc_pair_t *pairs, int64_t n_pairs,
                         int32_t open_, int32_t ext, const int32_t *matrix, int32_t *out,
                         int n_threads, int long_mode) {
  if (n_threads < 1) n_threads = 1;
  if (n_threads > 256) n_threads = 256;
  orc_job_t job;
  memset(&job, 0, sizeof(job));
  job.arena = arena; job.pairs = pairs; job.n_pairs = n_pairs;
  job.open_ = open_; job.ext = ext; job.matrix = matrix; job.out = out;
  job.long_mode = long_mode;
  pthread_mutex_init(&job.mu, NULL);
  pthread_t th[256];
  for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, orc_worker, &job);
  for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
  pthread_mutex_destroy(&job.mu);
  return 0;
}

int orc_align_batch(const uint8_t *arena, const orc_pair_t *pairs, int64_t n_pairs,
                    int32_t open_, int32_t ext, const int32_t *matrix, int32_t *out,
                    int n_threads) {
  return orc_align_batch_mode(arena, pairs, n_pairs, open_, ext, matrix, out, n_threads, 0);
}
