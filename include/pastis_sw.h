/*
 * pastis_sw.h -- C ABI of the B200-native batched Smith-Waterman aligner
 * (libpastis_sw.so, built from paper_2303_01845_b200/csrc/).
 *
 * The reference (/root/reference/pkg/src/pastislite, pure Python) has no FFI;
 * its drop-in seam is the Python API of pastislite.align.  Each entry point
 * below replaces one piece of that API; the Python mirror in
 * paper_2303_01845_b200/align.py calls these through ctypes.
 *
 *   sw_align_batch        replaces align.align_batch's per-pair loop
 *                         (align.py:223-246 -> _smith_waterman_timed
 *                         align.py:79-181) for a whole batch at once.
 *   sw_align_batch_multi  replaces AlignEngine's process-pool lanes
 *                         (align.py:299-347, _chunk align.py:265-269) with a
 *                         cell-balanced shard over several GPUs.
 *   sw_align_batch_device same as sw_align_batch on device-resident buffers.
 *   sw_result_t           AlignmentResult (align.py:55-67) minus `cells`
 *                         (= a_len*b_len, computed by the caller) plus a
 *                         per-pair status that maps to AlignmentError
 *                         (align.py:33-34, raised at align.py:81-82).
 *   sw_params_t           AlignParams (align.py:37-52) gap_open, gap_extend,
 *                         matrix (25x25, alphabet order of alphabet.py:8).
 *
 * Sequences are passed as RAW BYTES (what the reference receives as str):
 * the byte->residue mapping of align.py:27-30 (unknown -> 'X') is applied on
 * the device, and `matches` compares raw bytes exactly like align.py:142.
 *
 * Error convention: functions return 0 on success and a negative SW_E* code
 * on a call-level failure; sw_last_error() then describes it (thread-local).
 * Per-pair failures never fail the call: they are reported in
 * sw_result_t.status (align_batch's per-pair isolation, align.py:235-241).
 */
#ifndef PASTIS_SW_H
#define PASTIS_SW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SW_ABI_VERSION 2

/* call-level return codes */
#define SW_OK 0
#define SW_EINVAL (-1)   /* bad arguments / parameters outside the supported domain */
#define SW_ECUDA (-2)    /* CUDA runtime error (no device, OOM, launch failure) */
#define SW_EINTERNAL (-3)
#define SW_EFORMAT (-4)  /* malformed input text (sw_fasta_parse: see info->error) */
#define SW_ERANGE (-5)   /* output buffer too small (sw_kmer_candidates: see stats->performed) */

/* per-pair status codes (sw_result_t.status) */
#define SW_STATUS_OK 0
#define SW_STATUS_EMPTY 1     /* empty sequence: AlignmentError (align.py:81-82) */
#define SW_STATUS_INTERNAL 2  /* traceback lost: AssertionError (align.py:150) */
#define SW_STATUS_INVALID 3   /* pair outside the arena / > 65000 residues: the call returns SW_EINVAL */

typedef struct sw_pair_t { /* one candidate pair; a = rows, b = columns */
  uint64_t a_off;          /* byte offset of sequence a in the arena */
  uint64_t b_off;          /* byte offset of sequence b in the arena */
  uint32_t a_len;
  uint32_t b_len;
} sw_pair_t;               /* 24 bytes */

typedef struct sw_params_t {
  int32_t gap_open;        /* first gap residue costs gap_open */
  int32_t gap_extend;      /* each further residue costs gap_extend */
  int32_t matrix[25 * 25]; /* symmetric, row-major, alphabet ARNDCQEGHILKMFPSTWYVBZXU* */
} sw_params_t;
/* Supported domain (checked, SW_EINVAL otherwise): 0 <= gap_extend <=
 * gap_open <= 16383 and every matrix entry in [-127, 127].  BLOSUM62
 * (entries -4..11) with 11/1 or 11/2 is well inside it. */

typedef struct sw_result_t { /* AlignmentResult fields, 0-based inclusive spans */
  int32_t score;
  int32_t i_begin, i_end;  /* -1 for the empty (score 0) alignment */
  int32_t j_begin, j_end;
  int32_t matches;         /* identical aligned residue pairs */
  int32_t aln_len;         /* alignment columns including gaps */
  int32_t status;          /* SW_STATUS_* */
} sw_result_t;             /* 32 bytes */

typedef struct sw_timing_t { /* filled when non-NULL; device times from CUDA events */
  double forward_ms;       /* K1: forward score + end cell (paper's "forward scoring time") */
  double reverse_ms;       /* K2: reverse pass -> start box */
  double traceback_ms;     /* K3 + walk: box recompute with direction codes + traceback
                              (after the tile traceback K5, which is tile_tb_ms) */
  double kernel_ms;        /* all device work of the call (encode .. walk) */
  double h2d_ms;           /* host->device copies (host-buffer entry points only) */
  double d2h_ms;           /* device->host copy of the results */
  double total_ms;         /* wall time of the call */
  uint64_t cells;          /* sum of a_len*b_len over non-empty pairs */
  uint64_t h2d_bytes;
  uint64_t d2h_bytes;
  uint32_t launches;       /* kernels launched by the call */
  uint32_t wide_pairs;     /* pairs that needed the 32-bit-wide score path */
  uint64_t box_cells;      /* cells recomputed by K3 (sum of box areas) */
  uint64_t rev_cells;      /* cells scored by K2 */
  double host_plan_ms;     /* host time until the length plan is known (one small sync) */
  double host_setup_ms;    /* host time spent sizing / allocating cached device buffers */
  double tile_tb_ms;       /* K5 tile traceback: union of its per-class stream intervals
                              (they overlap the forward pass of the other classes) */
  double fwd_tail_ms;      /* forward phase end -> last K5 done (traceback not hidden
                              behind the forward pass) */
} sw_timing_t;

/* Number of visible CUDA devices (0 when none). */
int sw_get_device_count(void);

/* Human-readable description of the last failure on this thread. */
const char *sw_last_error(void);

/* ABI version of the loaded library (== SW_ABI_VERSION). */
int sw_abi_version(void);

/* Align n_pairs pairs whose bytes live in a HOST arena; results in HOST
 * memory, in input order.  Copies in, runs forward/reverse/traceback
 * kernels on `device`, copies out.  Synchronous.  Pinned host buffers give
 * the fastest copies but any host memory works. */
int sw_align_batch(int device, const uint8_t *arena, uint64_t arena_bytes,
                   const sw_pair_t *pairs, uint64_t n_pairs, const sw_params_t *params,
                   sw_result_t *out, sw_timing_t *timing);

/* Same on DEVICE-resident buffers (arena, pairs and out all on `device`).
 * `stream` is a cudaStream_t (NULL = the library's own stream).  Returns
 * after the work completes.  The arena may start at any byte address. */
int sw_align_batch_device(int device, const uint8_t *d_arena, uint64_t arena_bytes,
                          const sw_pair_t *d_pairs, uint64_t n_pairs,
                          const sw_params_t *params, sw_result_t *d_out, void *stream,
                          sw_timing_t *timing);

/* Shard a HOST batch over n_devices GPUs by cell count and return the
 * results in `out` in input order (replaces AlignEngine's process lanes,
 * align.py:299-335, whose _chunk split align.py:265-269 ignores lengths).
 * The plan (sw_shard_ranges) cuts the batch into contiguous ranges of equal
 * cells; every GPU uploads only its range's pairs and the arena bytes they
 * reference, overlapped with its forward pass, and writes its results
 * straight into its part of `out`; one host thread per GPU.
 * per_device_timing may be NULL or point to n_devices entries. */
int sw_align_batch_multi(int n_devices, const int *devices, const uint8_t *arena,
                         uint64_t arena_bytes, const sw_pair_t *pairs, uint64_t n_pairs,
                         const sw_params_t *params, sw_result_t *out,
                         sw_timing_t *per_device_timing);

/* The cell-balanced plan: bounds[0..n_shards] with bounds[0] = 0,
 * bounds[n_shards] = n_pairs and bounds[s] = the smallest k such that
 * n_shards * cells(pairs[0, k)) >= s * cells(all pairs), cells = a_len*b_len:
 * shard s takes the contiguous range [bounds[s], bounds[s+1]), and every
 * shard's cells are within one pair's of the mean.  `pairs` may be host or
 * device memory (then the plan runs on that device: scan + binary search). */
int sw_shard_ranges(const sw_pair_t *pairs, uint64_t n_pairs, int n_shards, uint64_t *bounds);

/* One shard of that plan on `device` (the unit of the multi-process driver:
 * one process per GPU, each calling this with its rank, then gathering the
 * records over NCCL).  `arena` and `pairs` are both device memory (the plan
 * runs on the device, only the arena bytes the range references are encoded,
 * nothing is copied) or both host memory (the plan runs on the host; the
 * range's pairs and the bytes they reference are uploaded, overlapped with
 * the forward pass).  d_out is a DEVICE buffer receiving the results of
 * pairs range[0] .. range[1]-1, in order; range (2 entries) may be NULL. */
int sw_align_shard(int device, const uint8_t *arena, uint64_t arena_bytes,
                   const sw_pair_t *pairs, uint64_t n_pairs, int shard, int n_shards,
                   const sw_params_t *params, sw_result_t *d_out, uint64_t *range,
                   void *stream, sw_timing_t *timing);

/* The same plan as a per-pair shard id, for host drivers and tests:
 * shard[k] in [0, n_shards); load[s] (may be NULL) receives the cell total
 * of shard s. */
int sw_partition_pairs(const sw_pair_t *pairs, uint64_t n_pairs, int n_shards,
                       int32_t *shard, uint64_t *load);

/* Release cached device buffers of `device` (-1 = all devices). */
void sw_release(int device);

/* Page-locked host memory for arenas / pair tables / results (fast copies).
 * Returns NULL on failure (sw_last_error). */
void *sw_host_alloc(uint64_t bytes);
void sw_host_free(void *p);

/* ---- FASTA ingest (the input side of the path) -----------
 * sw_fasta_parse replaces seqio.read_fasta (seqio.py:42-92) for ASCII text:
 * records in file order; residues concatenated, stripped, upper-cased, bytes
 * outside the alphabet mapped to 'X' (counted in n_mapped: seqio.py:88-89);
 * header = first whitespace-delimited token of the '>' line.  The residues
 * land directly in `arena` (the byte arena sw_align_batch consumes), the
 * header tokens in `headers`.  Capacities: arena and headers >= text_bytes,
 * recs_cap >= number of '>' bytes in the text.  Returns SW_OK, SW_EINVAL
 * (bad arguments / recs_cap too small) or SW_EFORMAT with info->error set to
 * the reference's first error (FastaError, seqio.py:19) or SW_FASTA_NONASCII
 * (Unicode text: the caller applies Python's str semantics itself). */
#define SW_FASTA_NONASCII 1            /* input has bytes >= 0x80 */
#define SW_FASTA_DATA_BEFORE_HEADER 2  /* "residue data before first header" (seqio.py:82-83) */
#define SW_FASTA_EMPTY_HEADER 3        /* "record with empty description line" (seqio.py:78-79) */
#define SW_FASTA_EMPTY_SEQ 4           /* "record ... has an empty sequence" (seqio.py:66-67) */
#define SW_FASTA_NO_RECORDS 5          /* "no FASTA records" (seqio.py:86-87) */

typedef struct sw_fasta_rec_t {
  uint64_t off;       /* residues: arena[off, off + len) */
  uint64_t hdr_off;   /* header token: headers[hdr_off, hdr_off + hdr_len) */
  uint32_t len;
  uint32_t hdr_len;
} sw_fasta_rec_t;     /* 24 bytes */

typedef struct sw_fasta_info_t {
  uint64_t n_recs, arena_bytes, header_bytes, n_mapped;
  int32_t error;      /* 0 or SW_FASTA_* */
  uint32_t error_hdr_len;
  uint64_t error_hdr_off;   /* SW_FASTA_EMPTY_SEQ: the record's header in `headers` */
} sw_fasta_info_t;

int sw_fasta_parse(const uint8_t *text, uint64_t text_bytes, uint8_t *arena, uint8_t *headers,
                   sw_fasta_rec_t *recs, uint64_t recs_cap, sw_fasta_info_t *info);

/* ---- candidate discovery (the caller side of the path) ----
 * sw_kmer_candidates replaces the reference's candidate stage: the overlap
 * semiring product A*A^T of the sequence-by-k-mer matrix (kmer.py:56-126,
 * sparse.local_spgemm sparse.py:236, blocked SUMMA summa.py, symmetry pruning
 * balance.py:98-128) followed by the threshold/orientation filter
 * (pipeline.py:290-303): every unordered pair i < j whose sequences share at
 * least min_shared DISTINCT k-mers (k-mer code = base-25 over alphabet.py:8,
 * first residue most significant, kmer.py:43-53; sequences shorter than k
 * have none), sorted by (i, j), with its shared count.  Sequences are residue
 * bytes in `arena` (seq_off/seq_len per sequence, e.g. from sw_fasta_parse).
 * Requires ceil(log2(25^k)) + ceil(log2(n_seqs)) <= 64.  If out_cap is
 * smaller than the number of candidates, returns SW_ERANGE with
 * stats->performed set (call again with a larger buffer). */
typedef struct sw_candidate_t {
  uint32_t i, j;      /* i < j: a = rows = sequence i, b = columns = sequence j */
  uint32_t count;     /* distinct shared k-mers (OverlapPayload.count, kmer.py:98) */
  uint32_t pad;
} sw_candidate_t;     /* 16 bytes */

typedef struct sw_kmer_stats_t {
  uint64_t positions;      /* k-mer occurrences */
  uint64_t distinct;       /* nnz of A: distinct (sequence, k-mer) entries */
  uint64_t buckets;        /* k-mers present in >= 1 sequence */
  uint64_t emitted;        /* pair emissions = sum over k-mers of c(c-1)/2 */
  uint64_t discovered;     /* unordered pairs sharing >= 1 k-mer (pruned overlap nnz) */
  uint64_t performed;      /* candidates with count >= min_shared */
  uint64_t flops;          /* semiring multiplies of A*A^T = sum over k-mers of c^2 */
  uint32_t short_seqs;     /* sequences shorter than k (kmer.py:87-88) */
  uint32_t pad;
  double device_ms;
} sw_kmer_stats_t;

int sw_kmer_candidates(int device, const uint8_t *arena, uint64_t arena_bytes,
                       const uint64_t *seq_off, const uint32_t *seq_len, uint32_t n_seqs, int k,
                       uint32_t min_shared, sw_candidate_t *out, uint64_t out_cap,
                       sw_kmer_stats_t *stats);

#ifdef __cplusplus
}
#endif

#endif /* PASTIS_SW_H */
