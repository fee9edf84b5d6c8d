// locate.cuh -- first-error position from a flagged chunk: the reference
// decode (proj/src/oracle.cpp:10-44) over the <= 42-byte window around the
// first flagged 32-byte chunk.  Shared by K3 (validate.cu, over HBM) and the
// small-call server (serve.cu, over shared memory): `s` is any generic
// address of the stream's byte 0.
#pragma once
#include <stdint.h>

#include "kernels.cuh"

namespace u8v {

// The reference decode of oracle.cpp:10-44 run over [from, to) of the stream;
// `from` is a character boundary and the first error lies inside the window.
__device__ __forceinline__ int decode_window(const uint8_t* s, uint64_t from, uint64_t to, uint64_t* off) {
  uint64_t i = from;
  while (i < to) {
    const uint8_t lead = s[i];
    if (lead < 0x80) {
      ++i;
      continue;
    }
    *off = i;
    if (lead < 0xC0) return kTooLong;
    if (lead >= 0xF8) return kHeaderBits;
    const unsigned len = lead >= 0xF0 ? 4 : lead >= 0xE0 ? 3 : 2;
    uint32_t cp = lead & (0x7Fu >> len);
    for (unsigned k = 1; k < len; ++k) {
      if (i + k >= to) return kTooShort;
      const uint8_t c = s[i + k];
      if ((c & 0xC0) != 0x80) return kTooShort;
      cp = (cp << 6) | (c & 0x3F);
    }
    const uint32_t min_cp = len == 2 ? 0x80 : len == 3 ? 0x800 : 0x10000;
    if (cp < min_cp) return kOverlong;
    if (cp > 0x10FFFF) return kTooLarge;
    if (cp >= 0xD800 && cp <= 0xDFFF) return kSurrogate;
    i += len;
  }
  return -1;
}

// Turn the first flagged chunk into (offset, kind).  Every flagged lane L
// satisfies E <= L <= E + 3 for the sequential first error E (proven for the
// lane formula by tests/test_swar.py), so E lies in [chunk_start - 3,
// chunk_end) and the decode needs bytes up to E + 3.  The window starts at
// the character boundary at or before chunk_start - 3 (at most 3
// continuation bytes back; if there are more, E is at that point).
// For a lane range [lane_lo, ...) the chunk may start before lane_lo, in
// bytes another shard owns: the window then starts at lane_lo - 3 (still at
// or before E, as E >= L - 3 >= lane_lo - 3), so it never decodes from the
// middle of a character at the start of a shard's head.
__device__ __forceinline__ void locate_chunk(const uint8_t* __restrict__ s, uint64_t n, int64_t off,
                                             int64_t lane_lo, unsigned long long c,
                                             unsigned long long* __restrict__ out_offset,
                                             int* __restrict__ out_kind) {
  const int64_t lmin = (int64_t)c * kChunkBytes - off;  // first lane of the chunk
  int64_t b0 = (lmin > lane_lo ? lmin : lane_lo) - 3;
  if (b0 < 0) b0 = 0;
  if ((uint64_t)b0 > n) b0 = (int64_t)n;
  int64_t b = b0;
  for (int k = 0; k < 3 && b > 0 && (uint64_t)b < n && (s[b] & 0xC0) == 0x80; ++k) --b;
  if ((uint64_t)b < n && (s[b] & 0xC0) == 0x80 && b > 0) b = b0;
  uint64_t to = (uint64_t)(lmin + kChunkBytes + 4);
  if (to > n) to = n;
  uint64_t o = 0;
  const int kind = decode_window(s, (uint64_t)b, to, &o);
  *out_kind = kind;
  *out_offset = kind < 0 ? ~0ull : o;
}

}  // namespace u8v
