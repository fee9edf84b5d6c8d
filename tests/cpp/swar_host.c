/*
 * swar_host.c -- TEST HELPER: the device SWAR formula (utf8v_swar.h),
 * compiled for the CPU, driven the way the kernels drive it, and checked
 * against the oracle restatement at volumes Python cannot loop over
 * (all 16,843,009 inputs of length <= 3 at every word alignment).
 */
#include <stdlib.h>
#include <string.h>

#include "utf8_oracle.h"
#include "utf8v_swar.h"
#include "utf8v_bits.h"
#include "utf8v_stream.h"

/* Stream the words of a zero-extended stream [0, n) that starts `off` bytes
 * into an aligned word grid, exactly like k_validate: words in order, lanes
 * up to n+3 included.  Returns the first flagged lane (stream coords), or
 * UINT64_MAX when none. */
static uint32_t word_at(const uint8_t* p, int64_t k, int64_t lo, int64_t hi) {
  uint32_t w = 0;
  for (int j = 0; j < 4; ++j) {
    const int64_t q = 4 * k + j;
    if (q >= lo && q < hi) w |= (uint32_t)p[q - lo] << (8 * j);
  }
  return w;
}

/* K1 drives the lead form (u8v_word_errors_lead: rare pairs flagged at the
 * lead's lane, reading the next word); the batch kernel the lag form. */
uint64_t swar_first_lane(const uint8_t* p, size_t n, unsigned off) {
  const int64_t lo = off, hi = (int64_t)off + (int64_t)n;
  const int64_t words = (hi + 3 + 3) / 4;
  const u8v_consts kc = u8v_make_consts();
  u8v_carry c = u8v_carry_zero();
  uint32_t w = word_at(p, 0, lo, hi);
  for (int64_t k = 0; k < words; ++k) {
    const uint32_t wn = word_at(p, k + 1, lo, hi);
    const uint32_t e = u8v_word_errors_lead(w, wn, &c, kc) & U8V_B7;
    w = wn;
    if (e) {
      for (int j = 0; j < 4; ++j)
        if ((e >> (8 * j + 7)) & 1) return (uint64_t)(4 * k + j - lo);
    }
  }
  return UINT64_MAX;
}

int swar_validate(const uint8_t* p, size_t n, unsigned off) {
  return swar_first_lane(p, n, off) == UINT64_MAX;
}

/* K1's lane-range contract (utf8v_cuda_validate_lanes): nonzero iff some
 * lane in [lane_lo, lane_hi) of the zero-extended stream p[0..n) is
 * flagged.  Used by the multi-process shard tests on the CPU. */
int swar_lanes(const uint8_t* p, size_t n, uint64_t lane_lo, uint64_t lane_hi) {
  const int64_t hi = (int64_t)n;
  const int64_t words = ((int64_t)lane_hi + 3) / 4 + 1;
  const u8v_consts kc = u8v_make_consts();
  u8v_carry c = u8v_carry_zero();
  uint32_t w = word_at(p, 0, 0, hi);
  for (int64_t k = 0; k < words; ++k) {
    const uint32_t wn = word_at(p, k + 1, 0, hi);
    const uint32_t e = u8v_mask_word(u8v_word_errors_lead(w, wn, &c, kc), 4 * k, (int64_t)lane_lo,
                                     (int64_t)lane_hi) & U8V_B7;
    w = wn;
    if (e) return 1;
  }
  return 0;
}

/* The first flagged lane in [lane_lo, lane_hi) of the zero-extended stream
 * p[0..n), or UINT64_MAX: the CPU model of a shard's first-error lane. */
uint64_t swar_first_lane_in(const uint8_t* p, size_t n, uint64_t lane_lo, uint64_t lane_hi) {
  const int64_t hi = (int64_t)n;
  const int64_t words = ((int64_t)lane_hi + 3) / 4 + 1;
  const u8v_consts kc = u8v_make_consts();
  u8v_carry c = u8v_carry_zero();
  uint32_t w = word_at(p, 0, 0, hi);
  for (int64_t k = 0; k < words; ++k) {
    const uint32_t wn = word_at(p, k + 1, 0, hi);
    const uint32_t e = u8v_mask_word(u8v_word_errors_lead(w, wn, &c, kc), 4 * k, (int64_t)lane_lo,
                                     (int64_t)lane_hi) & U8V_B7;
    w = wn;
    for (int j = 0; j < 4; ++j)
      if ((e >> (8 * j + 7)) & 1) return (uint64_t)(4 * k + j);
  }
  return UINT64_MAX;
}

/* Exhaustive agreement for every input of length 0..max_len (<= 3) at word
 * alignment `off`: counts verdict mismatches and first-lane bound violations
 * (E <= L <= E+3).  Mirrors proj/tests/acceptance.cpp:74-113. */
void swar_exhaustive(unsigned off, int max_len, uint64_t* checked, uint64_t* mismatches,
                     uint64_t* bound_violations) {
  uint8_t buf[3];
  uint64_t ck = 0, mm = 0, bv = 0;
  for (int len = 0; len <= max_len; ++len) {
    const uint64_t total = len == 0 ? 1 : (1ull << (8 * len));
    for (uint64_t v = 0; v < total; ++v) {
      for (int i = 0; i < len; ++i) buf[i] = (uint8_t)(v >> (8 * i));
      uint64_t eoff = 0;
      int kind = 0;
      const int ok = orc_validate(buf, (size_t)len, &eoff, &kind);
      const uint64_t L = swar_first_lane(buf, (size_t)len, off);
      ++ck;
      if ((L == UINT64_MAX) != (ok != 0)) ++mm;
      else if (!ok && !(L >= eoff && L <= eoff + 3)) ++bv;
    }
  }
  *checked = ck;
  *mismatches = mm;
  *bound_violations = bv;
}

/* All 65,536 byte pairs embedded at `offset` inside ASCII padding
 * (proj/tests/test_lookup.cpp:287-311), at word alignment `align`. */
uint64_t swar_pairs(size_t offset, unsigned align) {
  uint8_t buf[256];
  const size_t n = offset + 2 + 16;
  memset(buf, 0x41, sizeof buf);
  uint64_t mm = 0;
  for (unsigned b1 = 0; b1 < 256; ++b1)
    for (unsigned b2 = 0; b2 < 256; ++b2) {
      buf[offset] = (uint8_t)b1;
      buf[offset + 1] = (uint8_t)b2;
      uint64_t eo;
      int k;
      const int ok = orc_validate(buf, n, &eo, &k);
      if (swar_validate(buf, n, align) != ok) ++mm;
    }
  return mm;
}

/* K2's decomposition (batch.cu): the UNBOUNDED lane flags of the whole
 * buffer, attributed to the record of each flagged lane except the first
 * three lanes of a record, plus u8v_boundary_errors at every record start
 * (and at the end of the last record).  Must equal per-record validation. */
void swar_batch_decomp(const uint8_t* data, const uint64_t* offsets, size_t n_records, unsigned off,
                       uint8_t* verdicts) {
  if (n_records == 0) return;
  for (size_t r = 0; r < n_records; ++r) verdicts[r] = 1;
  const int64_t lo = (int64_t)off + (int64_t)offsets[0];
  const int64_t hi = (int64_t)off + (int64_t)offsets[n_records];
  if (hi <= lo) return;
  const u8v_consts kc = u8v_make_consts();
  /* 1. unbounded flags over the zero-extended [lo, hi), lanes up to hi+3 */
  const int64_t words = (hi + 3 + 3) / 4;
  u8v_carry c = u8v_carry_zero();
  const uint8_t* p0 = data + offsets[0]; /* word_at indexes from byte lo */
  uint32_t w = word_at(p0, 0, lo, hi);
  for (int64_t k = 0; k < words; ++k) {
    const uint32_t wn = word_at(p0, k + 1, lo, hi);
    const uint32_t e = u8v_word_errors_lead(w, wn, &c, kc) & U8V_B7;
    w = wn;
    for (int j = 0; j < 4; ++j) {
      if (!((e >> (8 * j + 7)) & 1)) continue;
      const int64_t q = 4 * k + j - (int64_t)off; /* data coords */
      if (q < (int64_t)offsets[0] || q >= (int64_t)offsets[n_records]) continue;
      size_t r = 0;
      while (r + 1 < n_records && (int64_t)offsets[r + 1] <= q) ++r;
      if (q - (int64_t)offsets[r] >= 3) verdicts[r] = 0; /* boundary lanes: step 2 */
    }
  }
  /* 2. every boundary */
  for (size_t rr = 0; rr <= n_records; ++rr) {
    const int64_t s0 = (int64_t)offsets[rr];
    int64_t a = rr > 0 ? (int64_t)offsets[rr - 1] : s0;
    int64_t b = rr < n_records ? (int64_t)offsets[rr + 1] : s0;
    if (a > s0) a = s0;
    if (b < s0) b = s0;
    uint64_t w8 = 0;
    for (int k = 0; k < 8; ++k) {
      const int64_t q = s0 - 4 + k;
      if (q >= (int64_t)offsets[0] && q < (int64_t)offsets[n_records]) w8 |= (uint64_t)data[q] << (8 * k);
    }
    int64_t ka = a - (s0 - 4), kb = b - (s0 - 4);
    ka = ka < 0 ? 0 : ka > 4 ? 4 : ka;
    kb = kb < 4 ? 4 : kb > 8 ? 8 : kb;
    const uint32_t f = u8v_boundary_errors(w8, (unsigned)ka, (unsigned)kb, kc);
    if ((f & 1u) && rr > 0) verdicts[rr - 1] = 0;
    if ((f & 2u) && rr < n_records) verdicts[rr] = 0;
  }
}

/* Oracle verdicts for every input of exactly `len` bytes (len <= 3), in the
 * order v = 0 .. 256^len - 1 with byte i = (v >> 8i) & 0xFF. */
void oracle_exhaustive_verdicts(int len, uint8_t* out) {
  uint8_t buf[3];
  const uint64_t total = len == 0 ? 1 : (1ull << (8 * len));
  for (uint64_t v = 0; v < total; ++v) {
    for (int i = 0; i < len; ++i) buf[i] = (uint8_t)(v >> (8 * i));
    uint64_t o;
    int k;
    out[v] = (uint8_t)orc_validate(buf, (size_t)len, &o, &k);
  }
}

/* All inputs of exactly `len` bytes laid out back to back (the batch form). */
void exhaustive_inputs(int len, uint8_t* out) {
  const uint64_t total = len == 0 ? 1 : (1ull << (8 * len));
  for (uint64_t v = 0; v < total; ++v)
    for (int i = 0; i < len; ++i) out[v * len + i] = (uint8_t)(v >> (8 * i));
}

#include <pthread.h>
typedef struct {
  const uint8_t* data;
  const uint64_t* off;
  uint8_t* valid;
  uint64_t* eoff;
  int* kind;
  size_t lo, hi;
} ob_job;

static void* ob_run(void* arg) {
  ob_job* j = (ob_job*)arg;
  for (size_t r = j->lo; r < j->hi; ++r) {
    uint64_t o = 0;
    int k = -1;
    j->valid[r] = (uint8_t)orc_validate(j->data + j->off[r], j->off[r + 1] - j->off[r], &o, &k);
    if (j->eoff) j->eoff[r] = j->valid[r] ? UINT64_MAX : o;
    if (j->kind) j->kind[r] = j->valid[r] ? -1 : k;
  }
  return NULL;
}

/* Oracle verdict (and first error) for every CSR record, on `threads` threads. */
void oracle_batch(const uint8_t* data, const uint64_t* off, size_t n_records, int threads,
                  uint8_t* valid, uint64_t* eoff, int* kind) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  ob_job jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t].data = data;
    jobs[t].off = off;
    jobs[t].valid = valid;
    jobs[t].eoff = eoff;
    jobs[t].kind = kind;
    jobs[t].lo = n_records * (size_t)t / (size_t)threads;
    jobs[t].hi = n_records * (size_t)(t + 1) / (size_t)threads;
    pthread_create(&tid[t], NULL, ob_run, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* Code-point sweep (proj/tests/test_oracle.cpp:106-121, acceptance.cpp:117-175)
 * through the oracle restatement: every scalar accepted, every surrogate
 * rejected as surrogate, every value above U+10FFFF (4-byte shape) rejected
 * as too-large.  Also checks the SWAR lane formula on each encoding. */
void oracle_cp_sweep(uint64_t* accepted, uint64_t* rejected, uint64_t* bad) {
  uint64_t acc = 0, rej = 0, b = 0;
  uint8_t e[4];
  for (uint32_t cp = 0; cp <= 0x1FFFFF; ++cp) {
    const int len = orc_encode(cp, e);
    uint64_t off;
    int kind;
    const int ok = orc_validate(e, (size_t)len, &off, &kind);
    const int swar = swar_validate(e, (size_t)len, cp & 3);
    if (swar != ok) ++b;
    if (cp > 0x10FFFF) {
      if (ok || kind != ORC_TOO_LARGE || off != 0) ++b;
      ++rej;
    } else if (cp >= 0xD800 && cp <= 0xDFFF) {
      if (ok || kind != ORC_SURROGATE || off != 0) ++b;
      ++rej;
    } else {
      if (!ok) ++b;
      ++acc;
    }
  }
  *accepted = acc;
  *rejected = rej;
  *bad = b;
}

/* Bit-sliced chunk form (utf8v_bits.h) vs the SWAR lead form, lane for lane.
 * Every lane's flag depends only on (x[i-3]>=F0, x[i-2]>=E0, x[i-1]>=C0,
 * x[i], bits 5,4 of x[i+1]); all 8192 classes are placed at each of the 32
 * lane positions of a chunk (bytes before/after the chunk come from the
 * prev/next words), the rest of the chunk random.  Then `fuzz` fully random
 * chunks.  Returns the number of lanes that differ. */
static uint64_t bits_rng(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t bits_compare(const uint8_t buf[40]) {
  /* buf[0..4) = prev word, buf[4..36) = chunk, buf[36..40) = next word */
  uint32_t w[8], prev, next;
  memcpy(&prev, buf, 4);
  memcpy(w, buf + 4, 32);
  memcpy(&next, buf + 36, 4);
  const uint32_t planes = u8v_chunk_errors_planes(w, prev, next);
  u8v_carry c = u8v_carry_of(prev);
  const u8v_consts k = u8v_make_consts();
  uint64_t bad = 0;
  for (int j = 0; j < 8; ++j) {
    const uint32_t e = u8v_word_errors_lead(w[j], j < 7 ? w[j + 1] : next, &c, k);
    for (int b = 0; b < 4; ++b) {
      const unsigned sw = (e >> (8 * b + 7)) & 1u;
      const unsigned pl = (planes >> (4 * j + b)) & 1u;
      bad += sw != pl;
    }
  }
  return bad;
}

uint64_t swar_bits_check(uint64_t seed, uint64_t fuzz) {
  static const uint8_t lo_c0[2] = {0x41, 0xC2}, lo_e0[2] = {0x85, 0xE1}, lo_f0[2] = {0x9F, 0xF3};
  static const uint8_t nb[4] = {0x80, 0x90, 0xA0, 0xB0};
  uint8_t buf[40];
  uint64_t s = seed, bad = 0;
  for (int pos = 0; pos < 32; ++pos) {
    const int i = 4 + pos; /* buffer index of the lane */
    for (int cls = 0; cls < 8192; ++cls) {
      for (int q = 0; q < 40; q += 8) {
        const uint64_t r = bits_rng(&s);
        memcpy(buf + q, &r, 8);
      }
      buf[i - 3] = lo_f0[(cls >> 0) & 1];
      buf[i - 2] = lo_e0[(cls >> 1) & 1];
      buf[i - 1] = lo_c0[(cls >> 2) & 1];
      buf[i] = (uint8_t)(cls >> 3);
      buf[i + 1] = nb[(cls >> 11) & 3];
      bad += bits_compare(buf);
    }
  }
  for (uint64_t t = 0; t < fuzz; ++t) {
    const uint64_t mode = bits_rng(&s);
    for (int q = 0; q < 40; ++q) {
      const uint64_t r = bits_rng(&s);
      static const uint8_t hot[] = {0x00, 0x41, 0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF, 0xC0, 0xC1,
                                    0xC2, 0xDF, 0xE0, 0xED, 0xEF, 0xF0, 0xF4, 0xF5, 0xFF};
      buf[q] = (mode & 1) ? (uint8_t)r : hot[r % sizeof hot];
    }
    bad += bits_compare(buf);
  }
  return bad;
}

/* Transpose check: planes match their definition on random chunks. */
uint64_t swar_planes_check(uint64_t seed, uint64_t trials) {
  uint64_t s = seed, bad = 0;
  for (uint64_t t = 0; t < trials; ++t) {
    uint32_t w[8], p[8];
    for (int j = 0; j < 8; ++j) w[j] = (uint32_t)bits_rng(&s);
    u8v_planes(w, p);
    for (int i = 0; i < 32; ++i) {
      const unsigned byte = (w[i / 4] >> (8 * (i % 4))) & 0xFF;
      for (int k2 = 0; k2 < 8; ++k2) bad += ((p[k2] >> i) & 1u) != ((byte >> k2) & 1u);
    }
  }
  return bad;
}

/* A stream fed in pieces (cut at `cuts`, n_cuts ascending inside [0, n]),
 * stitched with utf8v_stream.h exactly as the device session does it (edge
 * lanes from the carry, the rest in place over each piece); returns 1 when
 * the stitched verdict is "valid". */
int swar_stream_split(const uint8_t* p, size_t n, const uint64_t* cuts, size_t n_cuts) {
  uint32_t carry = 0, err = 0;
  uint64_t start = 0;
  for (size_t c = 0; c <= n_cuts; ++c) {
    const uint64_t end = c < n_cuts ? cuts[c] : n;
    const uint8_t* q = p + start;
    const uint64_t m = end - start;
    uint8_t h[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint64_t i = 0; i < m && i < 8; ++i) h[i] = q[i];
    uint32_t h0, h1, tail = 0;
    memcpy(&h0, h, 4);
    memcpy(&h1, h + 4, 4);
    err |= u8v_stream_edge(carry, h0, h1, m, 0);
    if (m > 4) err |= (uint32_t)swar_lanes(q, (size_t)m, 3, m - 1);
    for (uint64_t i = 0; i < 4 && i < m; ++i) {
      const uint64_t src = m >= 4 ? m - 4 + i : i;
      tail |= (uint32_t)q[src] << (8 * i);
    }
    carry = u8v_stream_carry(carry, tail, m);
    start = end;
  }
  err |= u8v_stream_edge(carry, 0, 0, 0, 1);
  return err == 0;
}

/* Permuted-order plane form: error bit pos(i) == natural form's bit i, on
 * random chunks and on every lane class at every position. */
static uint64_t perm_compare(const uint8_t buf[40]) {
  uint32_t w[8], prev, next, h7a, h7b;
  memcpy(&prev, buf, 4);
  memcpy(w, buf + 4, 32);
  memcpy(&next, buf + 36, 4);
  const u8v_consts k = u8v_make_consts();
  const uint32_t nat = u8v_chunk_errors_planes_k(w, prev, next, k, &h7a);
  const uint32_t per = u8v_chunk_errors_planes_perm_k(w, prev, next, k, &h7b);
  uint64_t bad = 0;
  for (unsigned i = 0; i < 32; ++i) {
    bad += ((nat >> i) & 1u) != ((per >> u8v_perm_pos(i)) & 1u);
    bad += ((h7a >> i) & 1u) != ((h7b >> u8v_perm_pos(i)) & 1u);
  }
  return bad;
}

uint64_t swar_bits_perm_check(uint64_t seed, uint64_t fuzz) {
  static const uint8_t lo_c0[2] = {0x41, 0xC2}, lo_e0[2] = {0x85, 0xE1}, lo_f0[2] = {0x9F, 0xF3};
  static const uint8_t nb[4] = {0x80, 0x90, 0xA0, 0xB0};
  uint8_t buf[40];
  uint64_t s = seed, bad = 0;
  for (int pos = 0; pos < 32; ++pos) {
    const int i = 4 + pos;
    for (int cls = 0; cls < 8192; ++cls) {
      for (int q = 0; q < 40; q += 8) {
        const uint64_t r = bits_rng(&s);
        memcpy(buf + q, &r, 8);
      }
      buf[i - 3] = lo_f0[(cls >> 0) & 1];
      buf[i - 2] = lo_e0[(cls >> 1) & 1];
      buf[i - 1] = lo_c0[(cls >> 2) & 1];
      buf[i] = (uint8_t)(cls >> 3);
      buf[i + 1] = nb[(cls >> 11) & 3];
      bad += perm_compare(buf);
    }
  }
  static const uint8_t hot[] = {0x00, 0x41, 0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF, 0xC0, 0xC1,
                                0xC2, 0xDF, 0xE0, 0xED, 0xEF, 0xF0, 0xF4, 0xF5, 0xFF};
  for (uint64_t t = 0; t < fuzz; ++t) {
    const uint64_t mode = bits_rng(&s);
    for (int q = 0; q < 40; ++q) {
      const uint64_t r = bits_rng(&s);
      buf[q] = (mode & 1) ? (uint8_t)r : hot[r % sizeof hot];
    }
    bad += perm_compare(buf);
  }
  return bad;
}

/* The acceptance gate's mutation corpus (proj/tests/acceptance.cpp:263-272):
 * for every seed in [seed_lo, seed_hi), optionally the valid buffer, then one
 * buffer per mutation strategy (kinds {1,2,3,4}, `target` bytes), all
 * concatenated into out (capacity cap) with CSR offsets offs[0..count].
 * Returns the number of buffers, or (size_t)-1 when cap is too small. */
size_t mutation_corpus(uint64_t seed_lo, uint64_t seed_hi, size_t target, int with_valid, uint8_t* out,
                       size_t cap, uint64_t* offs) {
  size_t count = 0, at = 0;
  offs[0] = 0;
  for (uint64_t seed = seed_lo; seed < seed_hi; ++seed) {
    for (int strat = with_valid ? -1 : 0; strat < 6; ++strat) {
      if (cap - at < target + 64) return (size_t)-1;
      const size_t n = strat < 0 ? orc_generate_valid(0xF, target, seed, out + at, cap - at)
                                 : orc_generate_invalid(0xF, target, seed, strat, out + at, cap - at);
      if (n == (size_t)-1) return (size_t)-1;
      at += n;
      offs[++count] = at;
    }
  }
  return count;
}
