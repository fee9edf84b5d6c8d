/*
 * utf8_oracle.h -- CPU restatement of the reference utf8v algorithms.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2010_03090_b200/ links, loads or
 * calls this code; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may, and there only as the checker.  The product path is
 * the CUDA library (libutf8v_cuda.so) and fails loudly when that is missing.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * the reference checkout, proj/...).  Parity of this restatement is pinned two
 * ways (see tests/test_oracle.py):
 *   1. against the reference's own known-answer vectors (tests/golden/), and
 *   2. against the unmodified reference library compiled from its sources
 *      into oracle/_ref/ (oracle/Makefile) -- same inputs, same outputs.
 */
#ifndef UTF8_ORACLE_H
#define UTF8_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error_kind, proj/include/utf8v/verdict.hpp:20-27 (same numbering). */
enum {
  ORC_HEADER_BITS = 0,
  ORC_TOO_SHORT = 1,
  ORC_TOO_LONG = 2,
  ORC_OVERLONG = 3,
  ORC_TOO_LARGE = 4,
  ORC_SURROGATE = 5
};

/* oracle_validate, proj/src/oracle.cpp:10-44.  Returns 1 when valid; else 0
 * and writes the offset of the offending sequence's lead byte and its kind. */
int orc_validate(const uint8_t* data, size_t n, uint64_t* offset, int* kind);

/* Same verdict, run on `threads` host threads.  Cuts at floor(k*n/T) moved
 * forward (at most 3 bytes) to a non-continuation byte -- the region_start
 * rule of proj/src/fsm.cpp:25-34.  The first failing region gives the global
 * first error (everything before it is valid text ending on a boundary). */
int orc_validate_mt(const uint8_t* data, size_t n, int threads, uint64_t* offset, int* kind);

/* encode_code_point, proj/src/oracle.cpp:46-70.  Returns byte count, 0 when
 * cp > 0x1FFFFF (the reference throws std::out_of_range). */
int orc_encode(uint32_t cp, uint8_t out[4]);

/* Nibble tables, proj/include/utf8v/tables.hpp:60-99 (built from the eight
 * error patterns exactly as build_nibble_tables does). */
void orc_nibble_tables(uint8_t t1[16], uint8_t t2[16], uint8_t t3[16]);

/* pair_always_invalid, proj/include/utf8v/tables.hpp:104-124. */
int orc_pair_always_invalid(uint8_t b1, uint8_t b2);

/* verify_nibble_tables, proj/src/tables.cpp:11-33.  Returns 1 when the tables
 * pass the 65,536-pair audit; else 0 and writes the first failing pair. */
int orc_verify_tables(const uint8_t t1[16], const uint8_t t2[16], const uint8_t t3[16],
                      uint8_t* fail_b1, uint8_t* fail_b2, uint8_t* fail_classified);

/* Lane entry points of proj/src/lookup_backend_detail.hpp:16-43 over a
 * vector of `width` bytes (classify: lookup_kernel.hpp:21-30; length check:
 * :38-46; incomplete: :48-68). */
void orc_classify_lanes(const uint8_t* in, const uint8_t* prev, uint8_t* out, size_t width);
void orc_length_error_lanes(const uint8_t* in, const uint8_t* prev, uint8_t* out, size_t width);
void orc_incomplete_lanes(const uint8_t* in, uint8_t* out, size_t width);

/* validate_with<vec16_scalar>, proj/include/utf8v/lookup_kernel.hpp:82-134:
 * 64-byte blocks, ASCII skip with the pending-incomplete carry, zero-padded
 * tail.  Returns 1 when valid. */
int orc_lookup_validate(const uint8_t* data, size_t n);

/* splitmix64, proj/include/utf8v/corpus.hpp:123-146. */
typedef struct { uint64_t state; } orc_rng;
uint64_t orc_rng_next(orc_rng* r);
uint64_t orc_rng_below(orc_rng* r, uint64_t bound);

/* random_code_point, proj/src/corpus.cpp:58-82. */
uint32_t orc_random_code_point(int kind, orc_rng* r);

/* generate_valid, proj/src/corpus.cpp:84-95.  kinds: bitmask over {1,2,3,4}
 * (bit k-1 set => kind k allowed).  Writes at most cap bytes; returns the
 * generated size (target_size .. target_size+3), or (size_t)-1 when cap is
 * too small. */
size_t orc_generate_valid(unsigned kinds_mask, size_t target_size, uint64_t seed,
                          uint8_t* out, size_t cap);

/* generate_invalid, proj/src/corpus.cpp:107-188 (strategies numbered as
 * mutation_strategy, proj/include/utf8v/corpus.hpp:175-182). */
size_t orc_generate_invalid(unsigned kinds_mask, size_t target_size, uint64_t seed,
                            int strategy, uint8_t* out, size_t cap);

/* gen_host.c: the n-byte BASELINE config stream (C0 recipe when ascii_only,
 * else the C1/C4 mix) of `seed`, byte-identical to csrc/gen.cu. */
int orc_gen_stream(uint8_t* out, uint64_t n, uint64_t seed, int ascii_only, int threads);
/* gen_host.c: config 4 (variant 0/1/2 = A/B/C), byte-identical to
 * utf8v_gen_c4; *err_offset = the first error (~0 for A). */
int orc_gen_c4(uint8_t* out, uint64_t n, uint64_t seed, int variant, int threads, uint64_t* err_offset);

#ifdef __cplusplus
}
#endif

#endif
