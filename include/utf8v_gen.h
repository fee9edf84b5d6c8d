/*
 * utf8v_gen.h -- synthetic input generators for the BASELINE configs
 * (bench / test tooling; NOT part of the drop-in validation boundary).
 *
 * All functions write DEVICE memory, are deterministic for a given seed on
 * any B200, return 0 on success, 1 on a CUDA error, 2 on a bad argument, and
 * synchronize `stream` (a cudaStream_t, 0 = legacy default) before returning.
 * The generation rules are pinned in DESIGN.md ("Synthetic inputs").
 */
#ifndef UTF8V_GEN_H
#define UTF8V_GEN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define kGenChunk 65536ull

/* Error classes injected into configs 2 and 3 (BASELINE.json configs[2]). */
enum {
  kErrOverlong = 0,     /* 2/3/4-byte overlong, subtype uniform */
  kErrSurrogate = 1,    /* ED A0..BF xx */
  kErrTooLarge = 2,     /* F4 90..BF xx xx */
  kErrBadLead = 3,      /* C0, C1, F5..FF with continuation bytes */
  kErrMissingCont = 4,  /* lead byte then ASCII */
  kErrStrayCont = 5,    /* continuation byte at a character boundary */
  kErrTruncatedEnd = 6, /* region ends inside a multi-byte character */
  kErrClasses = 7
};

/* Valid stream of exactly n bytes: ascii_only=1 -> config 0 bytes
 * (0x20..0x7E + 2% 0x0A), 0 -> the config-1 length mix. */
int utf8v_gen_stream(uint8_t* d_out, uint64_t n, uint64_t seed, int ascii_only, void* stream);

/* Bytes [lo, hi) of the n-byte stream utf8v_gen_stream(n, seed, ...) would
 * produce, written to d_out[0 .. hi-lo) (lo % 4 == 0): the shard a rank of
 * a multi-GPU run holds, without generating the rest. */
int utf8v_gen_stream_range(uint8_t* d_out, uint64_t n, uint64_t lo, uint64_t hi, uint64_t seed,
                           int ascii_only, void* stream);

/* Host (CPU) twin of utf8v_gen_stream writing host memory -- identical
 * bytes; used where no GPU may be touched (bench.py --impl reference). */
int utf8v_gen_stream_host(uint8_t* out, uint64_t n, uint64_t seed, int ascii_only, int threads);

/* Config 2: n_seg segments of seg_len bytes; n_seg/2 of them (chosen by the
 * seed) get one injected error.  Host outputs (may be NULL): per-segment
 * expected verdict and the injected error's segment-relative offset. */
int utf8v_gen_c2(uint8_t* d_out, uint64_t seg_len, uint32_t n_seg, uint64_t seed,
                 uint8_t* h_expected_valid, uint64_t* h_error_offset, void* stream);

/* Config 3 record lengths: lognormal(median, sigma) rounded, clipped to
 * [min_len, max_len]; writes h_offsets[0..n_records] (host, CSR). */
int utf8v_gen_c3_offsets(uint64_t n_records, uint64_t seed, double sigma, uint64_t median,
                         uint64_t min_len, uint64_t max_len, uint64_t* h_offsets);

/* Config 3 contents: every record its own mix stream; 10% of records (of
 * length >= 16) get one injected error.  d_offsets/h_offsets: same CSR array
 * on device and host. */
int utf8v_gen_c3(uint8_t* d_out, const uint64_t* d_offsets, const uint64_t* h_offsets,
                 uint64_t n_records, uint64_t seed, uint8_t* h_expected_valid, void* stream);

/* Config 4: n bytes (n % 8 == 0, n >= 8*64KiB) of the mix with every k*n/8
 * edge inside a 3- or 4-byte character.  variant 0 (A): valid; 1 (B): an
 * overlong whose lead is 1 byte after n/2; 2 (C): ends with 3 bytes of a
 * 4-byte character.  *h_error_offset = the first error's offset (~0 if A). */
int utf8v_gen_c4(uint8_t* d_out, uint64_t n, uint64_t seed, int variant, uint64_t* h_error_offset,
                 void* stream);

#ifdef __cplusplus
}
#endif

#endif
