/*
 * BENCH/TEST WORKLOADS ONLY -- seeded synthetic protein pair batches of
 * BASELINE.json's configs, written straight into a flat byte arena + pair
 * table (the layout of include/pastis_sw.h's sw_pair_t), multi-threaded.
 *
 * The numpy generators in workloads.py take ~20 s per million config-3
 * pairs; this one takes well under a second, so the bench can build N x 1M
 * pair batches per rank and the tests can check the full benched batch.
 *
 * Model (BASELINE.json configs):
 *   residues   uniform over the 20 standard residues (synth.py:12 of the
 *              reference);
 *   homolog(a) every residue substituted with p = sub_rate; at every position
 *              an indel event with p = indel_rate: half deletions of 1..3
 *              residues starting there, half insertions of 1..3 random
 *              residues before it; then truncated / padded with random
 *              residues to the target length;
 *   config 2   len(a) = len(b) = L; b = homolog(a) with p = 1/2, else uniform;
 *   config 3   len(a) = clip(round(LogNormal(5.5, 0.75)), 30, 2000); with
 *              p = 1/2 b = homolog(a) of length clip(round(len(a) U(0.7, 1.3)),
 *              30, 2000), else an independent draw of the same distribution;
 *   config 5   both lengths U[lo, hi]; b = homolog(a) with p = hom_frac
 *              (0 for the BASELINE config: independent pairs).
 * Random streams: xoshiro256** seeded by splitmix64 from (seed, stream id);
 * lengths come from one stream (pass 1), the residues of each block of 4096
 * pairs from the block's own stream (pass 2, any thread count -> same bytes).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { uint64_t a_off, b_off; uint32_t a_len, b_len; } syn_pair_t;

typedef struct { uint64_t s[4]; } rng_t;

static uint64_t splitmix(uint64_t *x) {
  uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static void rng_seed(rng_t *r, uint64_t seed, uint64_t stream) {
  uint64_t x = seed * 0x2545F4914F6CDD1Dull ^ (stream + 0x632BE59BD9B4E019ull);
  for (int k = 0; k < 4; ++k) r->s[k] = splitmix(&x);
}
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static inline uint64_t next64(rng_t *r) {
  uint64_t *s = r->s;
  const uint64_t res = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
  s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45);
  return res;
}
static inline double unif(rng_t *r) { return (double)(next64(r) >> 11) * (1.0 / 9007199254740992.0); }
static inline uint32_t below(rng_t *r, uint32_t n) { return (uint32_t)(((next64(r) >> 32) * n) >> 32); }
static double normal(rng_t *r) {
  double u = unif(r), v = unif(r);
  if (u < 1e-300) u = 1e-300;
  return sqrt(-2.0 * log(u)) * cos(6.283185307179586 * v);
}

static const char kStd[] = "ARNDCQEGHILKMFPSTWYV";
static inline uint8_t rres(rng_t *r) { return (uint8_t)kStd[below(r, 20)]; }

static uint32_t lognormal_len(rng_t *r) {
  double v = exp(5.5 + 0.75 * normal(r));
  long x = lround(v);
  if (x < 30) x = 30;
  if (x > 2000) x = 2000;
  return (uint32_t)x;
}

typedef struct {
  int kind;             /* 2, 3, 5 */
  uint64_t seed;
  uint32_t length;      /* config 2 */
  uint32_t lo, hi;      /* config 5 */
  double hom_frac, sub_rate, indel_rate;
} syn_cfg_t;

/* pass 1: lengths + homolog flags (one stream) */
int syn_lengths(const syn_cfg_t *c, uint64_t n, uint32_t *la, uint32_t *lb, uint8_t *hom) {
  rng_t r;
  rng_seed(&r, c->seed, 0xFFFFFFFFull);
  for (uint64_t k = 0; k < n; ++k) {
    uint32_t a, b;
    uint8_t h;
    if (c->kind == 2) {
      a = b = c->length;
      h = unif(&r) < c->hom_frac;
    } else if (c->kind == 3) {
      a = lognormal_len(&r);
      h = unif(&r) < c->hom_frac;
      if (h) {
        long x = lround((double)a * (0.7 + 0.6 * unif(&r)));
        if (x < 30) x = 30;
        if (x > 2000) x = 2000;
        b = (uint32_t)x;
      } else {
        b = lognormal_len(&r);
      }
    } else if (c->kind == 5) {
      a = c->lo + below(&r, c->hi - c->lo + 1);
      h = unif(&r) < c->hom_frac;
      b = h ? a : c->lo + below(&r, c->hi - c->lo + 1);
    } else {
      return -1;
    }
    la[k] = a; lb[k] = b; hom[k] = h;
  }
  return 0;
}

/* homolog of a[0..m) fitted to exactly `len` residues written to out */
static void homolog(rng_t *r, const uint8_t *a, uint32_t m, uint8_t *out, uint32_t len,
                    double sub, double indel) {
  uint32_t o = 0, i = 0;
  while (i < m && o < len) {
    const double u = unif(r);
    if (u < indel * 0.5) {                 /* deletion of 1..3 residues starting here */
      i += 1 + below(r, 3);
      continue;
    }
    if (u < indel) {                       /* insertion of 1..3 residues before it */
      uint32_t q = 1 + below(r, 3);
      while (q-- && o < len) out[o++] = rres(r);
      if (o >= len) break;
    }
    out[o++] = unif(r) < sub ? rres(r) : a[i];
    ++i;
  }
  while (o < len) out[o++] = rres(r);      /* pad */
}

typedef struct {
  const syn_cfg_t *c;
  uint64_t n;
  const syn_pair_t *t;
  const uint8_t *hom;
  uint8_t *arena;
  uint64_t next;
  pthread_mutex_t mu;
} job_t;

#define BLOCK 4096

static void *worker(void *arg) {
  job_t *J = (job_t *)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    const uint64_t b0 = J->next;
    J->next += BLOCK;
    pthread_mutex_unlock(&J->mu);
    if (b0 >= J->n) break;
    rng_t r;
    rng_seed(&r, J->c->seed, b0 / BLOCK);
    const uint64_t b1 = b0 + BLOCK < J->n ? b0 + BLOCK : J->n;
    for (uint64_t k = b0; k < b1; ++k) {
      const syn_pair_t *p = J->t + k;
      uint8_t *a = J->arena + p->a_off, *b = J->arena + p->b_off;
      for (uint32_t x = 0; x < p->a_len; ++x) a[x] = rres(&r);
      if (J->hom[k]) homolog(&r, a, p->a_len, b, p->b_len, J->c->sub_rate, J->c->indel_rate);
      else for (uint32_t x = 0; x < p->b_len; ++x) b[x] = rres(&r);
    }
  }
  return NULL;
}

/* pass 2: residues into arena at the table's offsets */
int syn_fill(const syn_cfg_t *c, uint64_t n, const syn_pair_t *t, const uint8_t *hom, uint8_t *arena,
             int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  job_t J;
  J.c = c; J.n = n; J.t = t; J.hom = hom; J.arena = arena; J.next = 0;
  pthread_mutex_init(&J.mu, NULL);
  pthread_t th[256];
  for (int k = 0; k < threads; ++k) pthread_create(&th[k], NULL, worker, &J);
  for (int k = 0; k < threads; ++k) pthread_join(th[k], NULL);
  pthread_mutex_destroy(&J.mu);
  return 0;
}
