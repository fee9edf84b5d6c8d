/*
 * gen_host.c -- CPU generator of the BASELINE config streams (C0 / C1 / C4
 * bytes).  TEST AND BENCH INFRASTRUCTURE ONLY: it is compiled into
 * oracle/liboracle.so and, for bench.py's reference arm, into
 * oracle/_ref/libutf8v_ref.so, so that arm builds its input without loading
 * the product library.  tests/test_oracle.py checks that its bytes equal the
 * product's generator (csrc/gen.cu, utf8v_gen_stream / _host).
 *
 * The recipe: the stream is cut into 64 KiB
 * generation chunks; chunk j of a stream with seed S draws from
 * splitmix64(S ^ 0xD1B54A32D192ED03 * (j+1)) (proj/include/utf8v/corpus.hpp:
 * 123-146, with the unbiased below()).  Mix streams append characters while
 * >= 4 bytes of the chunk remain -- kind from below(10): 0-3 one byte, 4-5
 * two, 6-8 three, 9 four; the code point uniform within the kind's class
 * (proj/src/corpus.cpp:68-82), shortest-form encoded
 * (proj/src/oracle.cpp:46-70) -- then pad with 0x20 + below(95).  ASCII
 * streams draw every byte as below(100) < 2 ? 0x0A : 0x20 + below(95).
 */
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>

#define GEN_CHUNK 65536ull

typedef struct {
  uint64_t s;
} gen_rng;

static uint64_t gen_next(gen_rng* r) {
  uint64_t z = (r->s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t gen_below(gen_rng* r, uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const uint64_t x = gen_next(r);
    if (x >= threshold) return x % bound;
  }
}

static uint32_t gen_code_point(int kind, gen_rng* r) {
  uint32_t cp;
  switch (kind) {
    case 1:
      return (uint32_t)gen_below(r, 0x80);
    case 2:
      return 0x80 + (uint32_t)gen_below(r, 0x780);
    case 3:
      cp = 0x800 + (uint32_t)gen_below(r, 0x10000 - 0x800 - 0x800); /* surrogates skipped */
      return cp >= 0xD800 ? cp + 0x800 : cp;
    default:
      return 0x10000 + (uint32_t)gen_below(r, 0x100000);
  }
}

static int gen_encode(uint32_t cp, uint8_t* o) {
  if (cp < 0x80) {
    o[0] = (uint8_t)cp;
    return 1;
  }
  if (cp < 0x800) {
    o[0] = (uint8_t)(0xC0 | (cp >> 6));
    o[1] = (uint8_t)(0x80 | (cp & 0x3F));
    return 2;
  }
  if (cp < 0x10000) {
    o[0] = (uint8_t)(0xE0 | (cp >> 12));
    o[1] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
    o[2] = (uint8_t)(0x80 | (cp & 0x3F));
    return 3;
  }
  o[0] = (uint8_t)(0xF0 | (cp >> 18));
  o[1] = (uint8_t)(0x80 | ((cp >> 12) & 0x3F));
  o[2] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
  o[3] = (uint8_t)(0x80 | (cp & 0x3F));
  return 4;
}

/* [lo, hi) of the stream, valid and exactly sized, drawn from r. */
static void gen_fill(uint8_t* out, uint64_t lo, uint64_t hi, gen_rng* r, int ascii_only) {
  uint64_t p = lo;
  if (ascii_only) {
    while (p < hi) out[p++] = gen_below(r, 100) < 2 ? 0x0A : (uint8_t)(0x20 + gen_below(r, 95));
    return;
  }
  while (hi - p >= 4) {
    const uint64_t k = gen_below(r, 10);
    const int kind = k < 4 ? 1 : k < 6 ? 2 : k < 9 ? 3 : 4;
    p += (uint64_t)gen_encode(gen_code_point(kind, r), out + p);
  }
  while (p < hi) out[p++] = (uint8_t)(0x20 + gen_below(r, 95));
}

/* Fixed bytes at a position; a chunk's fill skips them (config 4's edges). */
typedef struct {
  uint64_t pos;
  uint32_t len;
  uint8_t bytes[12];
} gen_patch;

/* Chunk j: its fill ranges around the (sorted) patches share one RNG. */
static void gen_chunk(uint8_t* out, uint64_t n, uint64_t seed, uint64_t j, int ascii_only, const gen_patch* pt,
                      int npt) {
  const uint64_t cs = j * GEN_CHUNK;
  const uint64_t ce = cs + GEN_CHUNK < n ? cs + GEN_CHUNK : n;
  gen_rng r = {seed ^ (0xD1B54A32D192ED03ull * (j + 1))};
  uint64_t p = cs;
  for (int k = 0; k < npt; ++k) {
    const uint64_t ps = pt[k].pos, pe = ps + pt[k].len;
    if (pe <= cs || ps >= ce) continue;
    if (ps > p) gen_fill(out, p, ps, &r, ascii_only);
    p = pe;
  }
  if (p < ce) gen_fill(out, p, ce, &r, ascii_only);
}

typedef struct {
  uint8_t* out;
  uint64_t n, seed, j0, j1;
  int ascii_only;
  const gen_patch* pt;
  int npt;
} gen_job;

static void* gen_worker(void* arg) {
  const gen_job* g = (const gen_job*)arg;
  for (uint64_t j = g->j0; j < g->j1; ++j) gen_chunk(g->out, g->n, g->seed, j, g->ascii_only, g->pt, g->npt);
  return NULL;
}

static int gen_run(uint8_t* out, uint64_t n, uint64_t seed, int ascii_only, int threads, const gen_patch* pt,
                   int npt) {
  enum { kMaxThreads = 256 };
  const uint64_t chunks = (n + GEN_CHUNK - 1) / GEN_CHUNK;
  if (threads < 1) threads = 1;
  if (threads > kMaxThreads) threads = kMaxThreads;
  if ((uint64_t)threads > chunks) threads = chunks ? (int)chunks : 1;
  pthread_t th[kMaxThreads];
  gen_job jobs[kMaxThreads];
  for (int t = 0; t < threads; ++t) {
    jobs[t].out = out;
    jobs[t].n = n;
    jobs[t].seed = seed;
    jobs[t].ascii_only = ascii_only;
    jobs[t].pt = pt;
    jobs[t].npt = npt;
    jobs[t].j0 = chunks * (uint64_t)t / (uint64_t)threads;
    jobs[t].j1 = chunks * (uint64_t)(t + 1) / (uint64_t)threads;
  }
  for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, gen_worker, &jobs[t]);
  gen_worker(&jobs[0]);
  for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
  for (int k = 0; k < npt; ++k)
    for (uint32_t i = 0; i < pt[k].len; ++i) out[pt[k].pos + i] = pt[k].bytes[i];
  return 0;
}

/* The n-byte config stream with `seed` (ascii_only: the C0 recipe) into
 * out[0..n), over `threads` threads.  Returns 0. */
int orc_gen_stream(uint8_t* out, uint64_t n, uint64_t seed, int ascii_only, int threads) {
  return gen_run(out, n, seed, ascii_only, threads, NULL, 0);
}

static gen_patch gen_make_patch(uint64_t pos, const uint8_t* b, int len) {
  gen_patch p;
  p.pos = pos;
  p.len = (uint32_t)len;
  for (int i = 0; i < 12; ++i) p.bytes[i] = i < len ? b[i] : 0;
  return p;
}

/* Config 4 (utf8v_gen_c4 in csrc/gen.cu): the mix stream with every k*n/8
 * edge (k = 1..7) inside a 3- or 4-byte character; variant 1 (B) puts an
 * overlong E0 80..9F 80..BF 1 byte after n/2, variant 2 (C) ends the stream
 * with 3 bytes of a 4-byte character.  *err_offset: the first error (~0 for
 * A).  n % 8 == 0, n >= 8 * 64 KiB.  Returns 0, or 2 on a bad n. */
int orc_gen_c4(uint8_t* out, uint64_t n, uint64_t seed, int variant, int threads, uint64_t* err_offset) {
  static const int kLen[8] = {0, 3, 4, 3, 4, 3, 4, 3};
  static const int kBefore[8] = {0, 1, 1, 2, 2, 1, 3, 2};
  if (n < 8 * GEN_CHUNK || n % 8 != 0) return 2;
  gen_rng plan = {seed ^ (0xA24BAED4963EE407ull * 5)};
  gen_patch pt[9];
  int npt = 0;
  uint64_t err_at = ~0ull;
  for (int k = 1; k < 8; ++k) {
    const uint64_t b = (uint64_t)k * (n / 8);
    uint8_t enc[12];
    const int len = gen_encode(gen_code_point(kLen[k], &plan), enc);
    if (variant == 1 && k == 4) {
      const int l3 = gen_encode(gen_code_point(3, &plan), enc);
      enc[l3 + 0] = 0xE0;
      enc[l3 + 1] = (uint8_t)(0x80 + gen_below(&plan, 0x20));
      enc[l3 + 2] = (uint8_t)(0x80 + gen_below(&plan, 0x40));
      pt[npt++] = gen_make_patch(b - 2, enc, l3 + 3);
      err_at = b + 1;
      continue;
    }
    pt[npt++] = gen_make_patch(b - (uint64_t)kBefore[k], enc, len);
  }
  if (variant == 2) {
    uint8_t enc[4];
    gen_encode(gen_code_point(4, &plan), enc);
    pt[npt++] = gen_make_patch(n - 3, enc, 3);
    err_at = n - 3;
  }
  if (err_offset) *err_offset = err_at;
  return gen_run(out, n, seed, 0, threads, pt, npt);  /* patches are already in position order */
}
