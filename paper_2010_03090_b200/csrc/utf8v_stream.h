// utf8v_stream.h -- stitching a stream validated in pieces (SURVEY §8(f) 4:
// the reference's fsm_state threading, proj/include/utf8v/fsm.hpp:15-20,
// restated for the Lookup lane predicate).
//
// A session has seen T bytes.  Lanes [0, T-1) are evaluated; lane T-1 is
// pending (it reads byte T, lead form).  The carry is the stream's last four
// bytes (bytes T-4..T-1, zero before the stream start), little-endian in one
// word.  Feeding a piece of n bytes evaluates
//   * lanes T-1 .. min(T+3, T+n-1)-1 here, from the carry and the piece's
//     first 8 bytes (the "edge"), and
//   * lanes T+3 .. T+n-2 in place over the piece (piece-local lanes
//     [3, n-1): every byte they read lies inside the piece),
// and leaves lane T+n-1 pending.  finish() evaluates lanes T-1 .. T+2 with
// zeros past the end (the end-of-input check, lookup_kernel.hpp:48-68).
// Compiled into the device edge kernel and, by gcc, into the CPU test that
// checks random splits against whole-stream validation.
#pragma once
#include <stdint.h>

#include "utf8v_swar.h"

// Error bits (bit i = lane T-1+i, i < 4) of the edge lanes.  `head` holds
// the piece's first min(n, 8) bytes (zero beyond), n the piece length
// (n = 0 with finish = 1 evaluates the end of the stream).
U8V_HD uint32_t u8v_stream_edge(uint32_t carry, uint32_t head0, uint32_t head1, uint64_t n,
                                int finish) {
  // Edge lanes: T-1 (byte 3 of the carry word) and T, T+1, T+2 (bytes 0..2
  // of head0), the first m of them: all four at finish, else the ones
  // before the new pending lane T+n-1.
  const uint64_t m = finish ? 4 : (n < 4 ? n : 4);
  const u8v_consts k = u8v_make_consts();
  // Lane T-1 reads bytes T-4..T (the carry word and head byte 0); the
  // carry's other lanes would need earlier bytes and are not wanted, so the
  // word before it is taken as zero and only its lane 3 kept.
  u8v_carry c0 = u8v_carry_zero();
  const uint32_t e0 = u8v_word_errors_lead(carry, head0, &c0, k) & 0x80000000u;
  const uint32_t e1 = u8v_word_errors_lead(head0, head1, &c0, k) & U8V_B7;
  uint32_t bits = e0 ? 1u : 0u;
  for (int b = 0; b < 3; ++b)
    if ((e1 >> (8 * b + 7)) & 1u) bits |= 1u << (b + 1);
  const uint32_t keep = m >= 4 ? 0xFu : ((1u << m) - 1u);
  return bits & keep;
}

// The carry after appending n bytes whose last min(n, 4) are in `tail`
// (little-endian, the last byte in the top byte when n >= 4).
U8V_HD uint32_t u8v_stream_carry(uint32_t carry, uint32_t tail, uint64_t n) {
  if (n >= 4) return tail;
  if (n == 0) return carry;
  const unsigned s = 8u * (unsigned)n;
  return (carry >> s) | (tail << (32u - s));
}
