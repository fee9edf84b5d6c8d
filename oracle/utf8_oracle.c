/*
 * utf8_oracle.c -- CPU restatement of the reference utf8v algorithms.
 * TEST INFRASTRUCTURE ONLY (see utf8_oracle.h).  Plain C99 + pthreads.
 */
#include "utf8_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ---- oracle_validate: proj/src/oracle.cpp:10-44 ------------------------ */
int orc_validate(const uint8_t* in, size_t n, uint64_t* offset, int* kind) {
  static const uint32_t min_for_len[5] = {0, 0, 0x80, 0x800, 0x10000}; /* :35-36 */
  size_t i = 0;
  while (i < n) {
    const uint8_t lead = in[i];
    if (lead < 0x80) { /* one byte, :15-18 */
      ++i;
      continue;
    }
    if (lead < 0xC0) { *offset = i; *kind = ORC_TOO_LONG; return 0; }     /* :19 */
    if (lead >= 0xF8) { *offset = i; *kind = ORC_HEADER_BITS; return 0; } /* :20 */
    const unsigned len = lead >= 0xF0 ? 4 : lead >= 0xE0 ? 3 : 2;         /* :21 */
    /* structure first, :23-31 */
    uint32_t cp = lead & (0x7Fu >> len);
    for (unsigned k = 1; k < len; ++k) {
      if (i + k >= n) { *offset = i; *kind = ORC_TOO_SHORT; return 0; }
      const uint8_t c = in[i + k];
      if ((c & 0xC0) != 0x80) { *offset = i; *kind = ORC_TOO_SHORT; return 0; }
      cp = (cp << 6) | (c & 0x3F);
    }
    /* range rules in fixed order, :33-40 */
    if (cp < min_for_len[len]) { *offset = i; *kind = ORC_OVERLONG; return 0; }
    if (cp > 0x10FFFF) { *offset = i; *kind = ORC_TOO_LARGE; return 0; }
    if (cp >= 0xD800 && cp <= 0xDFFF) { *offset = i; *kind = ORC_SURROGATE; return 0; }
    i += len;
  }
  return 1;
}

/* ---- multi-threaded oracle with the fsm.cpp:25-34 region rule ---------- */
typedef struct {
  const uint8_t* data;
  size_t lo, hi;
  int valid;
  uint64_t off;
  int kind;
} orc_region;

static void* orc_region_run(void* arg) {
  orc_region* r = (orc_region*)arg;
  uint64_t off = 0;
  int kind = 0;
  r->valid = orc_validate(r->data + r->lo, r->hi - r->lo, &off, &kind);
  r->off = r->lo + off;
  r->kind = kind;
  return NULL;
}

int orc_validate_mt(const uint8_t* data, size_t n, int threads, uint64_t* offset, int* kind) {
  if (threads < 2 || n < (size_t)threads * 1024) return orc_validate(data, n, offset, kind);
  if (threads > 256) threads = 256;
  size_t cut[257];
  cut[0] = 0;
  cut[threads] = n;
  for (int t = 1; t < threads; ++t) {
    size_t p = (size_t)((unsigned __int128)n * (unsigned)t / (unsigned)threads);
    size_t k = 0;
    while (k < 4 && p + k < n && (data[p + k] & 0xC0) == 0x80) ++k;
    if (k == 4) {
      /* four continuation bytes in a row: the text is malformed at or before
       * p+3; fall back to one sequential scan for exact (offset, kind). */
      return orc_validate(data, n, offset, kind);
    }
    cut[t] = p + k;
    if (cut[t] < cut[t - 1]) cut[t] = cut[t - 1];
  }
  orc_region reg[256];
  pthread_t tid[256];
  for (int t = 0; t < threads; ++t) {
    reg[t].data = data;
    reg[t].lo = cut[t];
    reg[t].hi = cut[t + 1];
    pthread_create(&tid[t], NULL, orc_region_run, &reg[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  for (int t = 0; t < threads; ++t) {
    if (!reg[t].valid) {
      /* Let E be the sequential first error.  Every byte before E belongs to
       * a complete character, so a non-continuation cut before E is a
       * character start: the regions before E's region are valid, and E's
       * region, scanned from its cut, retraces the sequential scan up to E.
       * The next cut is a non-continuation byte, so a character at E that
       * runs into it is too-short in both scans, at the same offset. */
      *offset = reg[t].off;
      *kind = reg[t].kind;
      return 0;
    }
  }
  return 1;
}

/* ---- encode_code_point: proj/src/oracle.cpp:46-70 ---------------------- */
int orc_encode(uint32_t cp, uint8_t out[4]) {
  if (cp > 0x1FFFFF) return 0;
  if (cp <= 0x7F) {
    out[0] = (uint8_t)cp;
    return 1;
  }
  if (cp <= 0x7FF) {
    out[0] = (uint8_t)(0xC0 | (cp >> 6));
    out[1] = (uint8_t)(0x80 | (cp & 0x3F));
    return 2;
  }
  if (cp <= 0xFFFF) {
    out[0] = (uint8_t)(0xE0 | (cp >> 12));
    out[1] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
    out[2] = (uint8_t)(0x80 | (cp & 0x3F));
    return 3;
  }
  out[0] = (uint8_t)(0xF0 | (cp >> 18));
  out[1] = (uint8_t)(0x80 | ((cp >> 12) & 0x3F));
  out[2] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
  out[3] = (uint8_t)(0x80 | (cp & 0x3F));
  return 4;
}

/* ---- nibble tables: proj/include/utf8v/tables.hpp:26-99 ---------------- */
static uint16_t nib(unsigned lo, unsigned hi) { /* tables.hpp:52-56 */
  uint16_t m = 0;
  for (unsigned v = lo; v <= hi; ++v) m = (uint16_t)(m | (1u << v));
  return m;
}

void orc_nibble_tables(uint8_t t1[16], uint8_t t2[16], uint8_t t3[16]) {
  /* The eight error patterns {bit, byte1_high, byte1_low, byte2_high},
   * tables.hpp:60-79. */
  const struct { uint8_t bit; uint16_t h1, l1, h2; } pat[8] = {
      {0, nib(0xC, 0xF), 0xFFFF, (uint16_t)(nib(0x0, 0x7) | nib(0xC, 0xF))}, /* too-short */
      {1, nib(0x0, 0x7), 0xFFFF, nib(0x8, 0xB)},                            /* too-long */
      {2, nib(0xE, 0xE), nib(0x0, 0x0), nib(0x8, 0x9)},                     /* overlong-3 */
      {3, nib(0xF, 0xF), nib(0x4, 0xF), nib(0x9, 0xB)},                     /* too-large */
      {4, nib(0xE, 0xE), nib(0xD, 0xD), nib(0xA, 0xB)},                     /* surrogate */
      {5, nib(0xC, 0xC), nib(0x0, 0x1), nib(0x8, 0xB)},                     /* overlong-2 */
      {6, nib(0xF, 0xF), (uint16_t)(nib(0x0, 0x0) | nib(0x5, 0xF)), nib(0x8, 0x8)}, /* ovl-4 */
      {7, nib(0x8, 0xB), 0xFFFF, nib(0x8, 0xB)},                            /* 2 conts */
  };
  memset(t1, 0, 16);
  memset(t2, 0, 16);
  memset(t3, 0, 16);
  for (int p = 0; p < 8; ++p) /* build_nibble_tables, tables.hpp:87-97 */
    for (unsigned n = 0; n < 16; ++n) {
      if (pat[p].h1 & (1u << n)) t1[n] |= (uint8_t)(1u << pat[p].bit);
      if (pat[p].l1 & (1u << n)) t2[n] |= (uint8_t)(1u << pat[p].bit);
      if (pat[p].h2 & (1u << n)) t3[n] |= (uint8_t)(1u << pat[p].bit);
    }
}

/* ---- pair_always_invalid: proj/include/utf8v/tables.hpp:104-124 -------- */
int orc_pair_always_invalid(uint8_t b1, uint8_t b2) {
  const int cont2 = (b2 & 0xC0) == 0x80;
  if ((b1 == 0xC0 || b1 == 0xC1) && cont2) return 1;
  if (b1 == 0xE0 && b2 >= 0x80 && b2 <= 0x9F) return 1;
  if (b1 == 0xF0 && b2 >= 0x80 && b2 <= 0x8F) return 1;
  if (b1 >= 0xC0 && !cont2) return 1;
  if (b1 <= 0x7F && cont2) return 1;
  if (b1 == 0xED && b2 >= 0xA0 && b2 <= 0xBF) return 1;
  if (b1 == 0xF4 && b2 >= 0x90 && b2 <= 0xBF) return 1;
  if (b1 >= 0xF5 && b1 <= 0xF7) return 1;
  if (b1 >= 0xF8) return 1;
  return 0;
}

/* ---- verify_nibble_tables: proj/src/tables.cpp:11-33 ------------------- */
int orc_verify_tables(const uint8_t t1[16], const uint8_t t2[16], const uint8_t t3[16],
                      uint8_t* fb1, uint8_t* fb2, uint8_t* fcls) {
  for (unsigned b1 = 0; b1 < 256; ++b1)
    for (unsigned b2 = 0; b2 < 256; ++b2) {
      const uint8_t c = (uint8_t)(t1[b1 >> 4] & t2[b1 & 0x0F] & t3[b2 >> 4]);
      const int expect_invalid = orc_pair_always_invalid((uint8_t)b1, (uint8_t)b2);
      const int expect_pair = (b1 & 0xC0) == 0x80 && (b2 & 0xC0) == 0x80;
      if (((c & 0x7F) != 0) != expect_invalid || ((c & 0x80) != 0) != expect_pair) {
        if (fb1) *fb1 = (uint8_t)b1;
        if (fb2) *fb2 = (uint8_t)b2;
        if (fcls) *fcls = c;
        return 0;
      }
    }
  return 1;
}

/* ---- Lookup kernels over plain byte lanes ------------------------------- */
static uint8_t g_t1[16], g_t2[16], g_t3[16];
static pthread_once_t g_tables_once = PTHREAD_ONCE_INIT;
static void tables_init(void) { orc_nibble_tables(g_t1, g_t2, g_t3); }

/* prev<N>(previous): proj/include/utf8v/byte_vector.hpp:73-82 */
static inline uint8_t lane_prev(const uint8_t* in, const uint8_t* prev, size_t w, size_t i,
                                size_t n) {
  return i >= n ? in[i - n] : prev[w - n + i];
}

/* classify, lookup_kernel.hpp:21-30 */
void orc_classify_lanes(const uint8_t* in, const uint8_t* prev, uint8_t* out, size_t w) {
  pthread_once(&g_tables_once, tables_init);
  for (size_t i = 0; i < w; ++i) {
    const uint8_t p1 = lane_prev(in, prev, w, i, 1);
    out[i] = (uint8_t)(g_t1[p1 >> 4] & g_t2[p1 & 0x0F] & g_t3[in[i] >> 4]);
  }
}

/* check_multibyte_lengths, lookup_kernel.hpp:38-46 (saturating_sub then OR,
 * AND 0x80, XOR with the classification). */
void orc_length_error_lanes(const uint8_t* in, const uint8_t* prev, uint8_t* out, size_t w) {
  orc_classify_lanes(in, prev, out, w);
  for (size_t i = 0; i < w; ++i) {
    const uint8_t p2 = lane_prev(in, prev, w, i, 2);
    const uint8_t p3 = lane_prev(in, prev, w, i, 3);
    const uint8_t third = p2 > (0xE0 - 0x80) ? (uint8_t)(p2 - (0xE0 - 0x80)) : 0;
    const uint8_t fourth = p3 > (0xF0 - 0x80) ? (uint8_t)(p3 - (0xF0 - 0x80)) : 0;
    const uint8_t expect = (uint8_t)((third | fourth) & 0x80);
    out[i] = (uint8_t)(expect ^ out[i]);
  }
}

/* check_incomplete + incomplete_limits, lookup_kernel.hpp:48-68 */
void orc_incomplete_lanes(const uint8_t* in, uint8_t* out, size_t w) {
  for (size_t i = 0; i < w; ++i) {
    uint8_t lim = 0xFF;
    if (i == w - 3) lim = 0xEF;
    if (i == w - 2) lim = 0xDF;
    if (i == w - 1) lim = 0xBF;
    const uint8_t mx = in[i] > lim ? in[i] : lim;
    out[i] = (uint8_t)(mx ^ lim);
  }
}

/* lookup_checker<vec16_scalar> + validate_with, lookup_kernel.hpp:82-134 */
int orc_lookup_validate(const uint8_t* data, size_t size) {
  enum { W = 16, BLOCK = 64, VEC = BLOCK / W };
  uint8_t prev[W] = {0}, pending[W] = {0}, err = 0;
  uint8_t tmp[W], tail[BLOCK];
  const size_t full = size - size % BLOCK;
  for (size_t pos = 0; pos < size; pos += BLOCK) {
    const uint8_t* blk = data + pos;
    if (pos >= full) { /* zero-padded tail, :128-132 */
      memset(tail, 0, BLOCK);
      memcpy(tail, data + pos, size - pos);
      blk = tail;
    }
    uint8_t combined = 0; /* OR of the vectors, is_all_ascii, :92-96 */
    for (int i = 0; i < BLOCK; ++i) combined |= blk[i];
    if ((combined & 0x80) == 0) {
      for (int i = 0; i < W; ++i) err |= pending[i];
      memset(pending, 0, W);
      memcpy(prev, blk + BLOCK - W, W);
    } else {
      for (int v = 0; v < VEC; ++v) { /* :98-102 */
        orc_length_error_lanes(blk + v * W, prev, tmp, W);
        for (int i = 0; i < W; ++i) err |= tmp[i];
        memcpy(prev, blk + v * W, W);
      }
      orc_incomplete_lanes(blk + BLOCK - W, pending, W); /* :103 */
    }
  }
  for (int i = 0; i < W; ++i) err |= pending[i]; /* valid(), :111 */
  return err == 0;
}

/* ---- corpus: proj/include/utf8v/corpus.hpp:123-146, proj/src/corpus.cpp - */
uint64_t orc_rng_next(orc_rng* r) {
  uint64_t z = (r->state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t orc_rng_below(orc_rng* r, uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const uint64_t x = orc_rng_next(r);
    if (x >= threshold) return x % bound;
  }
}

static uint32_t class_size(int kind) { /* corpus.cpp:58-66 */
  switch (kind) {
    case 1: return 0x80;
    case 2: return 0x800 - 0x80;
    case 3: return 0x10000 - 0x800 - 0x800;
    default: return 0x110000 - 0x10000;
  }
}

uint32_t orc_random_code_point(int kind, orc_rng* r) { /* corpus.cpp:68-82 */
  const uint32_t index = (uint32_t)orc_rng_below(r, class_size(kind));
  switch (kind) {
    case 1: return index;
    case 2: return 0x80 + index;
    case 3: {
      uint32_t cp = 0x800 + index;
      if (cp >= 0xD800) cp += 0x800;
      return cp;
    }
    default: return 0x10000 + index;
  }
}

static int canonical_kinds(unsigned mask, int kinds[4]) { /* corpus.cpp:48-56 */
  int c = 0;
  for (int k = 1; k <= 4; ++k)
    if (mask & (1u << (k - 1))) kinds[c++] = k;
  return c;
}

size_t orc_generate_valid(unsigned mask, size_t target, uint64_t seed, uint8_t* out,
                          size_t cap) { /* corpus.cpp:84-95 */
  int kinds[4];
  const int nk = canonical_kinds(mask, kinds);
  if (nk == 0) return (size_t)-1;
  orc_rng rng = {seed};
  size_t size = 0;
  while (size < target) {
    const int kind = kinds[orc_rng_below(&rng, (uint64_t)nk)];
    uint8_t b[4];
    const int len = orc_encode(orc_random_code_point(kind, &rng), b);
    if (size + (size_t)len > cap) return (size_t)-1;
    memcpy(out + size, b, (size_t)len);
    size += (size_t)len;
  }
  return size;
}

static size_t char_length(uint8_t lead) { /* corpus.cpp:16-21 */
  if (lead < 0x80) return 1;
  if (lead < 0xE0) return 2;
  if (lead < 0xF0) return 3;
  return 4;
}

static int splice(uint8_t* buf, size_t* size, size_t cap, size_t at, const uint8_t* piece,
                  size_t len) { /* corpus.cpp:41-44 */
  if (*size + len > cap) return 0;
  memmove(buf + at + len, buf + at, *size - at);
  memcpy(buf + at, piece, len);
  *size += len;
  return 1;
}

size_t orc_generate_invalid(unsigned mask, size_t target, uint64_t seed, int strategy,
                            uint8_t* bytes, size_t cap) { /* corpus.cpp:107-188 */
  size_t size = orc_generate_valid(mask, target < 1 ? 1 : target, seed, bytes, cap);
  if (size == (size_t)-1) return size;
  orc_rng rng = {seed ^ (0x9E3779B97F4A7C15ull * ((uint64_t)strategy + 1))};
  /* character_boundaries, corpus.cpp:25-35: char starts plus the end */
  size_t nb = 0;
  size_t* bnd = (size_t*)malloc((size + 1) * sizeof(size_t));
  for (size_t i = 0;;) {
    bnd[nb++] = i;
    if (i >= size) break;
    i += char_length(bytes[i]);
  }
#define RANDOM_BOUNDARY() (bnd[orc_rng_below(&rng, nb)])
#define CONT() ((uint8_t)(0x80 + orc_rng_below(&rng, 0x40)))
  size_t result = size;
  switch (strategy) {
    case 0: /* flip, :124-135 */
      for (;;) {
        const size_t pos = (size_t)orc_rng_below(&rng, size);
        const uint8_t value = (uint8_t)orc_rng_below(&rng, 256);
        if (value == bytes[pos]) continue;
        const uint8_t saved = bytes[pos];
        bytes[pos] = value;
        uint64_t o;
        int k;
        if (!orc_validate(bytes, size, &o, &k)) break;
        bytes[pos] = saved;
      }
      break;
    case 1: { /* truncate, :136-152 */
      size_t nm = 0;
      for (size_t i = 0; i < nb; ++i)
        if (bnd[i] < size && char_length(bytes[bnd[i]]) > 1) bnd[nm++] = bnd[i];
      if (nm == 0) {
        const int kind = 2 + (int)orc_rng_below(&rng, 3);
        uint8_t b[4];
        const int len = orc_encode(orc_random_code_point(kind, &rng), b);
        if (size + (size_t)len - 1 > cap) { result = (size_t)-1; break; }
        memcpy(bytes + size, b, (size_t)len - 1);
        result = size + (size_t)len - 1;
        break;
      }
      const size_t start = bnd[orc_rng_below(&rng, nm)];
      const size_t keep = 1 + (size_t)orc_rng_below(&rng, char_length(bytes[start]) - 1);
      result = start + keep;
      break;
    }
    case 2: { /* insert_continuation, :153-155 */
      const uint8_t p[1] = {CONT()};
      const size_t at = RANDOM_BOUNDARY();
      if (!splice(bytes, &result, cap, at, p, 1)) result = (size_t)-1;
      break;
    }
    case 3: { /* overlong, :156-174 */
      const uint64_t which = orc_rng_below(&rng, 3);
      uint8_t p[4];
      size_t len;
      size_t at;
      /* Argument evaluation order in the reference is unspecified, but the
       * initializer list {..} is evaluated left to right ([dcl.init.list]),
       * and random_boundary() is the first function argument -- GCC
       * evaluates splice's arguments right to left, so the piece's draws
       * come before the boundary draw.  Pinned against oracle/_ref. */
      if (which == 0) {
        p[0] = (uint8_t)(0xC0 + orc_rng_below(&rng, 2));
        p[1] = CONT();
        len = 2;
      } else if (which == 1) {
        p[0] = 0xE0;
        p[1] = (uint8_t)(0x80 + orc_rng_below(&rng, 0x20));
        p[2] = CONT();
        len = 3;
      } else {
        p[0] = 0xF0;
        p[1] = (uint8_t)(0x80 + orc_rng_below(&rng, 0x10));
        p[2] = CONT();
        p[3] = CONT();
        len = 4;
      }
      at = RANDOM_BOUNDARY();
      if (!splice(bytes, &result, cap, at, p, len)) result = (size_t)-1;
      break;
    }
    case 4: { /* surrogate, :175-179 */
      uint8_t p[3];
      p[0] = 0xED;
      p[1] = (uint8_t)(0xA0 + orc_rng_below(&rng, 0x20));
      p[2] = CONT();
      const size_t at = RANDOM_BOUNDARY();
      if (!splice(bytes, &result, cap, at, p, 3)) result = (size_t)-1;
      break;
    }
    case 5: { /* too_large, :180-184 */
      uint8_t p[4];
      p[0] = 0xF4;
      p[1] = (uint8_t)(0x90 + orc_rng_below(&rng, 0x30));
      p[2] = CONT();
      p[3] = CONT();
      const size_t at = RANDOM_BOUNDARY();
      if (!splice(bytes, &result, cap, at, p, 4)) result = (size_t)-1;
      break;
    }
    default:
      result = (size_t)-1;
  }
#undef RANDOM_BOUNDARY
#undef CONT
  free(bnd);
  return result;
}
