/*
 * vt_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the reference's scalar codec, the normative oracle of
 * arXiv 2109.10433's `vtrans` library.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library.  The CUDA product path in
 * paper_2109_10433_b200/ never links or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * golden vectors in tests/golden/ (made from the reference's own unit tests and
 * from the reference library compiled out of tree into oracle/_ref/), and, when
 * oracle/_ref is present, differentially against the compiled reference itself.
 *
 * Each function cites the reference lines it restates (paths relative to
 * /root/reference/).
 */
#include "vt_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- per-character rules ------------------------------------------------ */

/* proj/src/codec_core.cpp:5-38 (decode_utf8_char).  Returns the code point, or
 * -1 when no valid character starts at `pos`; *len receives the byte length.
 * Order of checks matters for the reported position only through "fail at
 * pos": lead class, then truncation (pos+len > n, :28), then continuation
 * shape (:31), then overlong (:34), cap (:35) and surrogate range (:36). */
int32_t vto_decode_utf8_char(const uint8_t* s, uint64_t n, uint64_t pos, uint32_t* len) {
  uint8_t lead = s[pos];
  uint32_t need, cp, lo;
  if (lead < 0x80) {
    *len = 1;
    return lead;
  }
  if ((lead & 0xE0u) == 0xC0u) {
    need = 2; cp = lead & 0x1Fu; lo = 0x80u;
  } else if ((lead & 0xF0u) == 0xE0u) {
    need = 3; cp = lead & 0x0Fu; lo = 0x800u;
  } else if ((lead & 0xF8u) == 0xF0u) {
    need = 4; cp = lead & 0x07u; lo = 0x10000u;
  } else {
    return -1; /* continuation in lead position, or 0xF8..0xFF */
  }
  if (pos + need > n) return -1; /* truncated: reported at the lead */
  for (uint32_t k = 1; k < need; k++) {
    uint8_t c = s[pos + k];
    if ((c & 0xC0u) != 0x80u) return -1;
    cp = (cp << 6) | (c & 0x3Fu);
  }
  if (cp < lo) return -1;                       /* overlong */
  if (cp > 0x10FFFFu) return -1;                /* above U+10FFFF */
  if (cp >= 0xD800u && cp <= 0xDFFFu) return -1; /* encoded surrogate */
  *len = need;
  return (int32_t)cp;
}

/* proj/src/codec_core.cpp:74-83 (decode_utf16_char). */
int32_t vto_decode_utf16_char(const uint16_t* s, uint64_t n, uint64_t pos, uint32_t* len) {
  uint16_t u = s[pos];
  if (u < 0xD800u || u > 0xDFFFu) {
    *len = 1;
    return u;
  }
  if (u >= 0xDC00u) return -1;       /* low surrogate first */
  if (pos + 1 >= n) return -1;       /* high surrogate at the end */
  uint16_t v = s[pos + 1];
  if (v < 0xDC00u || v > 0xDFFFu) return -1; /* high not followed by low */
  *len = 2;
  return (int32_t)(0x10000u + (((uint32_t)(u - 0xD800u) << 10) | (uint32_t)(v - 0xDC00u)));
}

/* proj/src/codec_core.cpp:40-61 (encode_utf8). */
uint32_t vto_encode_utf8(uint32_t cp, uint8_t out[4]) {
  if (cp < 0x80u) {
    out[0] = (uint8_t)cp;
    return 1;
  }
  if (cp < 0x800u) {
    out[0] = (uint8_t)(0xC0u | (cp >> 6));
    out[1] = (uint8_t)(0x80u | (cp & 0x3Fu));
    return 2;
  }
  if (cp < 0x10000u) {
    out[0] = (uint8_t)(0xE0u | (cp >> 12));
    out[1] = (uint8_t)(0x80u | ((cp >> 6) & 0x3Fu));
    out[2] = (uint8_t)(0x80u | (cp & 0x3Fu));
    return 3;
  }
  out[0] = (uint8_t)(0xF0u | (cp >> 18));
  out[1] = (uint8_t)(0x80u | ((cp >> 12) & 0x3Fu));
  out[2] = (uint8_t)(0x80u | ((cp >> 6) & 0x3Fu));
  out[3] = (uint8_t)(0x80u | (cp & 0x3Fu));
  return 4;
}

/* proj/src/codec_core.cpp:63-72 (encode_utf16). */
uint32_t vto_encode_utf16(uint32_t cp, uint16_t out[2]) {
  if (cp < 0x10000u) {
    out[0] = (uint16_t)cp;
    return 1;
  }
  uint32_t v = cp - 0x10000u;
  out[0] = (uint16_t)(0xD800u + (v >> 10));
  out[1] = (uint16_t)(0xDC00u + (v & 0x3FFu));
  return 2;
}

/* ---- whole-buffer transcoders ------------------------------------------- */

/* proj/src/codec_core.cpp:85-104 (scalar::utf8_to_utf16): greedy decode, stop
 * at the first failure with consumed == error_at.  `out` may be NULL (count
 * only: written is still reported). */
void vto_utf8_to_utf16(const uint8_t* s, uint64_t n, uint16_t* out, vto_result* r) {
  uint64_t p = 0, q = 0;
  r->error_at = -1;
  while (p < n) {
    uint32_t len;
    int32_t cp = vto_decode_utf8_char(s, n, p, &len);
    if (cp < 0) {
      r->error_at = (int64_t)p;
      break;
    }
    uint16_t u[2];
    uint32_t k = vto_encode_utf16((uint32_t)cp, u);
    if (out) {
      out[q] = u[0];
      if (k == 2) out[q + 1] = u[1];
    }
    p += len;
    q += k;
  }
  r->consumed = p;
  r->written = q;
}

/* proj/src/codec_core.cpp:106-125 (scalar::utf16_to_utf8). */
void vto_utf16_to_utf8(const uint16_t* s, uint64_t n, uint8_t* out, vto_result* r) {
  uint64_t p = 0, q = 0;
  r->error_at = -1;
  while (p < n) {
    uint32_t len;
    int32_t cp = vto_decode_utf16_char(s, n, p, &len);
    if (cp < 0) {
      r->error_at = (int64_t)p;
      break;
    }
    uint8_t b[4];
    uint32_t k = vto_encode_utf8((uint32_t)cp, b);
    if (out) memcpy(out + q, b, k);
    p += len;
    q += k;
  }
  r->consumed = p;
  r->written = q;
}

/* Verdict of proj/src/validation.cpp:30-49 (validate_utf8), which by contract
 * (proj/include/vtrans/utf8_to_utf16.hpp:24-28) agrees with the scalar decoder:
 * valid iff the greedy decode reaches the end.  Returns the first error index
 * or -1 (the reference's bool is `result < 0`). */
int64_t vto_validate_utf8(const uint8_t* s, uint64_t n) {
  vto_result r;
  vto_utf8_to_utf16(s, n, NULL, &r);
  return r.error_at;
}

/* proj/src/validation.cpp:51-77 (validate_utf16): index of the first unit that
 * scalar decode_utf16_char rejects, or -1. */
int64_t vto_validate_utf16(const uint16_t* s, uint64_t n) {
  vto_result r;
  vto_utf16_to_utf8(s, n, NULL, &r);
  return r.error_at;
}

/* proj/src/codec_core.cpp:141-150 (count_codepoints_utf8): -1 for nullopt. */
int64_t vto_count_utf8(const uint8_t* s, uint64_t n) {
  uint64_t p = 0, c = 0;
  while (p < n) {
    uint32_t len;
    if (vto_decode_utf8_char(s, n, p, &len) < 0) return -1;
    p += len;
    c++;
  }
  return (int64_t)c;
}

/* proj/src/codec_core.cpp:152-161 (count_codepoints_utf16). */
int64_t vto_count_utf16(const uint16_t* s, uint64_t n) {
  uint64_t p = 0, c = 0;
  while (p < n) {
    uint32_t len;
    if (vto_decode_utf16_char(s, n, p, &len) < 0) return -1;
    p += len;
    c++;
  }
  return (int64_t)c;
}

/* ---- multi-threaded whole-buffer variants -------------------------------
 * Used by the parity tests at BASELINE sizes and by bench.py's cpu_baseline
 * ("port") leg.  Split points follow the character-boundary rule the survey
 * verified against the reference: the UTF-8 cut
 * moves back to the last non-continuation byte within 3 bytes, the UTF-16 cut
 * moves back one unit when it would separate a high from a low surrogate.
 * Per-shard results combine exactly: the first shard with an error decides,
 * and written counts add up over the shards before it. */

static uint64_t split_utf8(const uint8_t* s, uint64_t n, uint64_t cut) {
  if (cut == 0 || cut >= n) return cut;
  for (uint64_t k = 0; k <= 3 && k <= cut; k++) {
    if ((s[cut - k] & 0xC0u) != 0x80u) return cut - k;
  }
  return cut;
}

static uint64_t split_utf16(const uint16_t* s, uint64_t n, uint64_t cut) {
  if (cut == 0 || cut >= n) return cut;
  if (s[cut] >= 0xDC00u && s[cut] <= 0xDFFFu && s[cut - 1] >= 0xD800u && s[cut - 1] <= 0xDBFFu)
    return cut - 1;
  return cut;
}

typedef struct {
  int dir; /* 0: utf8->utf16, 1: utf16->utf8 */
  const void* in;
  uint64_t n;
  void* out; /* NULL: count only; else per-shard scratch */
  vto_result r;
} shard_job;

static void* shard_main(void* arg) {
  shard_job* j = (shard_job*)arg;
  if (j->dir == 0)
    vto_utf8_to_utf16((const uint8_t*)j->in, j->n, (uint16_t*)j->out, &j->r);
  else
    vto_utf16_to_utf8((const uint16_t*)j->in, j->n, (uint8_t*)j->out, &j->r);
  return NULL;
}

/* Runs the scalar transcoder on `threads` shards in parallel and writes the
 * concatenated output to `out` (may be NULL).  Output of shard k is produced in
 * a private buffer and then moved to its combined offset. */
static void mt_run(int dir, const void* in, uint64_t n, void* out, int threads, vto_result* res) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  shard_job jobs[256];
  pthread_t tids[256];
  uint64_t starts[257];
  starts[0] = 0;
  for (int k = 1; k < threads; k++) {
    uint64_t cut = n / (uint64_t)threads * (uint64_t)k;
    uint64_t c = dir == 0 ? split_utf8((const uint8_t*)in, n, cut)
                          : split_utf16((const uint16_t*)in, n, cut);
    if (c < starts[k - 1]) c = starts[k - 1];
    starts[k] = c;
  }
  starts[threads] = n;
  size_t esz_in = dir == 0 ? 1 : 2, esz_out = dir == 0 ? 2 : 1, mult = dir == 0 ? 1 : 3;
  for (int k = 0; k < threads; k++) {
    jobs[k].dir = dir;
    jobs[k].in = (const uint8_t*)in + starts[k] * esz_in;
    jobs[k].n = starts[k + 1] - starts[k];
    jobs[k].out = out ? malloc((jobs[k].n * mult + 16) * esz_out) : NULL;
    pthread_create(&tids[k], NULL, shard_main, &jobs[k]);
  }
  for (int k = 0; k < threads; k++) pthread_join(tids[k], NULL);
  uint64_t written = 0;
  res->error_at = -1;
  res->consumed = n;
  for (int k = 0; k < threads; k++) {
    if (out) memcpy((uint8_t*)out + written * esz_out, jobs[k].out, jobs[k].r.written * esz_out);
    written += jobs[k].r.written;
    if (jobs[k].r.error_at >= 0) {
      res->error_at = (int64_t)starts[k] + jobs[k].r.error_at;
      res->consumed = (uint64_t)res->error_at;
      for (int j = k + 1; j < threads; j++) free(jobs[j].out);
      free(jobs[k].out);
      res->written = written;
      return;
    }
    free(jobs[k].out);
  }
  res->written = written;
}

void vto_utf8_to_utf16_mt(const uint8_t* s, uint64_t n, uint16_t* out, int threads, vto_result* r) {
  mt_run(0, s, n, out, threads, r);
}

void vto_utf16_to_utf8_mt(const uint16_t* s, uint64_t n, uint8_t* out, int threads, vto_result* r) {
  mt_run(1, s, n, out, threads, r);
}

/* Batched validation for the exhaustive sweeps (acceptance C3,
 * proj/tests/acceptance.cpp:138-194): `count` strings packed back to back,
 * string i spans [offsets[i], offsets[i+1]).  Writes the first error index (or
 * -1) per string. */
void vto_validate_utf8_batch(const uint8_t* data, const uint64_t* offsets, uint64_t count,
                             int64_t* first_err) {
  for (uint64_t i = 0; i < count; i++)
    first_err[i] = vto_validate_utf8(data + offsets[i], offsets[i + 1] - offsets[i]);
}

/* Every 1-, 2- and 3-byte input, in the enumeration order of
 * proj/tests/acceptance.cpp:147-167: writes the verdict (1 = valid) of input
 * number i to verdict[i].  Returns the number of inputs (256+65536+16777216). */
uint64_t vto_exhaustive_short_verdicts(uint8_t* verdict) {
  uint64_t k = 0;
  uint8_t b[3];
  for (int a = 0; a < 256; a++) {
    b[0] = (uint8_t)a;
    verdict[k++] = vto_validate_utf8(b, 1) < 0;
  }
  for (int a = 0; a < 256; a++)
    for (int c = 0; c < 256; c++) {
      b[0] = (uint8_t)a;
      b[1] = (uint8_t)c;
      verdict[k++] = vto_validate_utf8(b, 2) < 0;
    }
  for (int a = 0; a < 256; a++)
    for (int c = 0; c < 256; c++)
      for (int d = 0; d < 256; d++) {
        b[0] = (uint8_t)a;
        b[1] = (uint8_t)c;
        b[2] = (uint8_t)d;
        verdict[k++] = vto_validate_utf8(b, 3) < 0;
      }
  return k;
}

/* ---- batched transcoding (the checker for vt_*_batch) ----------------------
 * String i = [offsets[i], offsets[i+1]); output at the same offset (UTF-16
 * units) or 3 * offsets[i] (UTF-8 bytes); one result per string.  The scalar
 * codec per string, as the reference's fuzz driver calls it per case
 * (proj/src/harness.cpp:357-375). */
void vto_utf8_to_utf16_batch(const uint8_t* data, const uint64_t* offsets, uint64_t count,
                             uint16_t* out, vto_result* res) {
  for (uint64_t i = 0; i < count; i++)
    vto_utf8_to_utf16(data + offsets[i], offsets[i + 1] - offsets[i], out + offsets[i], res + i);
}

void vto_utf16_to_utf8_batch(const uint16_t* data, const uint64_t* offsets, uint64_t count,
                             uint8_t* out, vto_result* res) {
  for (uint64_t i = 0; i < count; i++)
    vto_utf16_to_utf8(data + offsets[i], offsets[i + 1] - offsets[i], out + 3 * offsets[i], res + i);
}

/* Differential-fuzz cases shaped like the reference's run_fuzz
 * (proj/src/harness.cpp:388-436, its gen_valid_utf8 at :330-350): case i of
 * kind i % 3 -- 0: random bytes, 1: valid UTF-8 drawn from one of six
 * class mixes, 2: the same with one bit flipped; lengths uniform in
 * [0, max_len].  Our own splitmix64 stream (not the reference's mt19937), so
 * the cases have the reference's shape, not its exact bytes.  Writes
 * offsets[0..count] and the packed bytes; returns the total, or UINT64_MAX if
 * it would exceed `cap`. */
static uint64_t fz_next(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint32_t fz_scalar(uint64_t* s, int cls) {
  switch (cls) {
    case 0: return (uint32_t)(fz_next(s) % 0x80);
    case 1: return 0x80 + (uint32_t)(fz_next(s) % (0x800 - 0x80));
    case 2: {
      uint32_t cp;
      do cp = 0x800 + (uint32_t)(fz_next(s) % (0x10000 - 0x800));
      while (cp >= 0xD800 && cp <= 0xDFFF);
      return cp;
    }
    default: return 0x10000 + (uint32_t)(fz_next(s) % (0x110000 - 0x10000));
  }
}

uint64_t vto_fuzz_cases(uint64_t seed, uint64_t count, uint32_t max_len, uint8_t* data,
                        uint64_t* offsets, uint64_t cap) {
  static const int mixes[6][4] = {{100, 0, 0, 0}, {22, 78, 0, 0}, {1, 0, 99, 0},
                                  {0, 0, 0, 100}, {25, 25, 25, 25}, {50, 0, 50, 0}};
  uint64_t st = seed, pos = 0;
  offsets[0] = 0;
  for (uint64_t i = 0; i < count; i++) {
    const int kind = (int)(i % 3);
    const uint64_t target = max_len ? fz_next(&st) % ((uint64_t)max_len + 1) : 0;
    if (pos + target + 4 > cap) return UINT64_MAX;
    const uint64_t start = pos;
    if (kind == 0) {
      for (uint64_t k = 0; k < target; k++) data[pos++] = (uint8_t)fz_next(&st);
    } else {
      const int* mix = mixes[fz_next(&st) % 6];
      while (pos - start < target) {
        int roll = (int)(fz_next(&st) % 100), cls = 0;
        for (int k = 0; k < 4; k++) {
          if (roll < mix[k]) {
            cls = k;
            break;
          }
          roll -= mix[k];
        }
        pos += vto_encode_utf8(fz_scalar(&st, cls), data + pos);
      }
      if (kind == 2 && pos > start) data[start + fz_next(&st) % (pos - start)] ^= (uint8_t)(1u << (fz_next(&st) % 8));
    }
    offsets[i + 1] = pos;
  }
  return pos;
}
