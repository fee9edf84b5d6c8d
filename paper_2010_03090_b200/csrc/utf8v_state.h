// utf8v_state.h -- the composable state of a segment validated on its own
// (SURVEY §8(f) 4).  The reference threads an fsm_state through
// validate_fsm(piece, state) and notes the fold is associative
// (proj/include/utf8v/fsm.hpp:15-20); this is the Lookup counterpart that
// lets segments validated independently -- in any order, on any device --
// be merged afterwards with an associative combine().
//
// A segment covers bytes [s, e) of a stream.  Its state holds
//   len    e - s
//   flag   nonzero iff one of its interior lanes [s+3, e-1) is flagged -- the
//          lanes that read only the segment's own bytes (lane i reads bytes
//          i-3 .. i+1, utf8v_swar.h)
//   head   its first min(len, 4) bytes (byte k at head[k], zeros after)
//   tail   its last min(len, 4) bytes, right-aligned (byte e-1 at tail[3],
//          zeros before)
// combine(A, B) evaluates the lanes whose 5-byte window crosses the seam
// m = e_A and lies inside A ++ B: lanes i in [m-1, m+3) with i >= s_A + 3 and
// i < e_B - 1.  Their bytes lie in A's last 4 and B's first 4, so each lane
// of the whole stream is evaluated exactly once: inside the leaf segment that
// holds its window, or at the first combine whose result does.  The final
// verdict adds the lanes that read outside the stream: [0, 3) from the head
// with zeros before, [n-1, n+3) from the tail with zeros after.
//
// Compiled into the device kernels (segment and batch states, the in-order
// reduction) and into the host C-ABI (utf8v_state_combine/_valid); the CPU
// tests check random splits and combine orders against the oracle.
#pragma once
#include <stdint.h>

#include "utf8v_swar.h"

// Layout shared with include/utf8v_cuda.h (utf8v_state, 24 bytes).
typedef struct {
  uint64_t len;
  uint32_t flag;
  uint8_t head[4];
  uint8_t tail[4];
  uint32_t reserved;
} u8v_state;

U8V_HD u8v_state u8v_state_empty(void) {
  u8v_state s;
  s.len = 0;
  s.flag = 0;
  s.reserved = 0;
  for (int k = 0; k < 4; ++k) s.head[k] = s.tail[k] = 0;
  return s;
}

U8V_HD uint32_t u8v_word_of(const uint8_t b[4]) {
  return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
}

// Lane flags (bit j = lane j of the window, j = 0..7) of the 8-byte window
// lo|hi (lo = bytes 0..3, hi = bytes 4..7) with zeros before and after;
// lanes 0..2 and 7 are only right when those zeros are the stream's.
U8V_HD uint32_t u8v_window_lanes(uint32_t lo, uint32_t hi) {
  const u8v_consts k = u8v_make_consts();
  u8v_carry c = u8v_carry_zero();
  const uint32_t e0 = u8v_word_errors_lead(lo, hi, &c, k) & U8V_B7;
  const uint32_t e1 = u8v_word_errors_lead(hi, 0, &c, k) & U8V_B7;
  uint32_t bits = 0;
  for (int b = 0; b < 4; ++b) {
    if ((e0 >> (8 * b + 7)) & 1u) bits |= 1u << b;
    if ((e1 >> (8 * b + 7)) & 1u) bits |= 1u << (b + 4);
  }
  return bits;
}

U8V_HD u8v_state u8v_state_combine(u8v_state a, u8v_state b) {
  if (a.len == 0) return b;
  if (b.len == 0) return a;
  u8v_state r = u8v_state_empty();
  r.len = a.len + b.len;
  // Window lane j is stream lane m-4+j (m = the seam); the seam lanes are
  // j = 3 .. 6.  Lane m-1+t (t = 0..3) reads bytes m-4+t .. m+t: inside
  // A ++ B iff len_A >= 4 - t and len_B >= t + 1.
  const uint32_t lanes = u8v_window_lanes(u8v_word_of(a.tail), u8v_word_of(b.head));
  uint32_t seam = 0;
  for (unsigned t = 0; t < 4; ++t)
    if (a.len >= 4 - t && b.len >= t + 1 && ((lanes >> (3 + t)) & 1u)) seam = 1;
  r.flag = (a.flag | b.flag | seam) ? 1u : 0u;
  // head: the first 4 bytes of A ++ B; tail: the last 4.
  for (unsigned k = 0; k < 4; ++k) {
    if (k < a.len) r.head[k] = a.head[k];
    else if (k - a.len < b.len && k - a.len < 4) r.head[k] = b.head[k - a.len];
    const unsigned from_end = 3 - k;  // tail[k] is byte e-1-from_end
    if (from_end < b.len) r.tail[k] = b.tail[k];
    else if (from_end - b.len < a.len && from_end - b.len < 4) r.tail[k] = a.tail[k + (unsigned)b.len];
  }
  return r;
}

// Nonzero iff the stream whose whole state is s is invalid: its interior and
// seam lanes (s.flag) plus the lanes that read before the start or past the
// end of the zero-extended stream.
U8V_HD uint32_t u8v_state_errors(u8v_state s) {
  if (s.flag) return 1;
  // lanes 0..2 read bytes -3 .. 3: zeros then the head (zeros past n)
  const uint32_t start = u8v_window_lanes(0, u8v_word_of(s.head)) & 0x70u;
  // lanes n-1 .. n+2 read bytes n-4 .. n+3: the tail (zeros before the
  // stream when n < 4) then zeros
  const uint32_t end = u8v_window_lanes(u8v_word_of(s.tail), 0) & 0x78u;
  return (start | end) ? 1u : 0u;
}
