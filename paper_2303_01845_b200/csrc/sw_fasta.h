// sw_fasta.h -- FASTA ingest straight into the aligner's byte arena (host).
//
// Restates seqio.read_fasta (/root/reference/pkg/src/pastislite/seqio.py:42-92)
// for ASCII text, one pass, no per-residue interpreter work:
//   * lines split like Python text mode with universal newlines: "\n",
//     "\r\n" and a lone "\r" each end a line (seqio.py:71 `for line in fh`);
//   * each line stripped of str.strip()'s ASCII whitespace
//     (' ', \t, \n, \r, \v, \f, \x1c-\x1f) and skipped if empty (:72-74);
//   * a '>' line closes the previous record (:75-76), then its header is the
//     first whitespace-delimited token after '>' (:77), empty -> error (:78-79);
//   * other lines before any header -> error (:82-83); else their stripped
//     bytes are appended, upper-cased, bytes outside the 25-letter alphabet
//     (alphabet.py:8) mapped to 'X' and counted (:57-65);
//   * a record with no residues -> error (:66-67); no records at all -> error
//     (:86-87).
// Errors are reported in the order the reference raises them.  Non-ASCII
// input needs Python's Unicode strip/upper semantics: reported as
// SW_FASTA_NONASCII so the caller decodes it as UTF-8 itself.
#pragma once
#include <cstdint>
#include <cstring>

#include "../../include/pastis_sw.h"

namespace pastis_fasta {

// byte classes: bit 0 = line break (\n, \r), bit 1 = str.strip whitespace;
// out[c] = the residue byte c becomes (upper-cased, 'X' outside the
// alphabet), miss[c] = 1 when that counts as "mapped" (seqio.py:60-64)
struct Tables {
  uint8_t cls[256], out[256], miss[256];
  Tables() {
    const char *alpha = "ARNDCQEGHILKMFPSTWYVBZXU*";
    for (int c = 0; c < 256; ++c) {
      cls[c] = 0;
      const bool ws = c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == 0x0b || c == 0x0c ||
                      (c >= 0x1c && c <= 0x1f);
      if (ws) cls[c] |= 2;
      if (c == '\n' || c == '\r') cls[c] |= 1;
      const int u = (c >= 'a' && c <= 'z') ? c - 32 : c;
      bool in = false;
      for (const char *p = alpha; *p; ++p) in |= (uint8_t)*p == u;
      out[c] = in ? (uint8_t)u : (uint8_t)'X';
      miss[c] = in ? 0 : 1;
    }
  }
};

inline bool is_ws(const Tables &T, uint8_t c) { return T.cls[c] & 2; }

inline int parse(const uint8_t *text, uint64_t n, uint8_t *arena, uint8_t *headers,
                 sw_fasta_rec_t *recs, uint64_t recs_cap, sw_fasta_info_t *info) {
  static const Tables T;
  memset(info, 0, sizeof(*info));
  uint8_t any = 0;
  for (uint64_t k = 0; k < n; ++k) any |= text[k];   // vectorised OR: any byte >= 0x80?
  if (any & 0x80) {
    info->error = SW_FASTA_NONASCII;
    return SW_EFORMAT;
  }
  uint64_t apos = 0, hpos = 0, nrec = 0, mapped = 0;
  bool have = false;
  uint64_t cur_hoff = 0, cur_start = 0;
  uint32_t cur_hlen = 0;
  auto fail = [&](int kind) {
    info->error = kind;
    info->n_recs = nrec;
    info->arena_bytes = apos;
    info->header_bytes = hpos;
    info->n_mapped = mapped;
    return SW_EFORMAT;
  };
  // close the open record (seqio.py:55-68)
  auto flush = [&]() -> int {
    if (!have) return 0;
    if (apos == cur_start) {
      info->error_hdr_off = cur_hoff;
      info->error_hdr_len = cur_hlen;
      return SW_FASTA_EMPTY_SEQ;
    }
    if (nrec >= recs_cap) return -1;
    recs[nrec].off = cur_start;
    recs[nrec].hdr_off = cur_hoff;
    recs[nrec].len = (uint32_t)(apos - cur_start);
    recs[nrec].hdr_len = cur_hlen;
    ++nrec;
    return 0;
  };
  uint64_t i = 0;
  while (i < n) {
    // one line: [b, e) up to "\n", "\r\n" or "\r"
    const uint64_t b = i;
    while (i < n && !(T.cls[text[i]] & 1)) ++i;
    uint64_t e = i;
    if (i < n) {
      if (text[i] == '\r' && i + 1 < n && text[i + 1] == '\n') i += 2;
      else i += 1;
    }
    uint64_t s = b;
    while (s < e && is_ws(T, text[s])) ++s;
    while (e > s && is_ws(T, text[e - 1])) --e;
    if (s == e) continue;
    if (text[s] == '>') {
      const int rc = flush();
      if (rc > 0) return fail(rc);
      if (rc < 0) return SW_EINVAL;
      uint64_t t = s + 1;
      while (t < e && is_ws(T, text[t])) ++t;
      uint64_t u = t;
      while (u < e && !is_ws(T, text[u])) ++u;
      if (u == t) return fail(SW_FASTA_EMPTY_HEADER);
      memcpy(headers + hpos, text + t, u - t);
      cur_hoff = hpos;
      cur_hlen = (uint32_t)(u - t);
      hpos += u - t;
      cur_start = apos;
      have = true;
    } else {
      if (!have) return fail(SW_FASTA_DATA_BEFORE_HEADER);
      uint8_t *dst = arena + apos;
      uint32_t miss = 0;
      for (uint64_t k = s; k < e; ++k) {
        const uint8_t c = text[k];
        *dst++ = T.out[c];
        miss += T.miss[c];
      }
      apos += e - s;
      mapped += miss;
    }
  }
  const int rc = flush();
  if (rc > 0) return fail(rc);
  if (rc < 0) return SW_EINVAL;
  if (nrec == 0) return fail(SW_FASTA_NO_RECORDS);
  info->n_recs = nrec;
  info->arena_bytes = apos;
  info->header_bytes = hpos;
  info->n_mapped = mapped;
  return SW_OK;
}

}  // namespace pastis_fasta
