// stream_edge.cuh -- the per-piece step of a stream session (utf8v_stream.h)
// as one device thread: evaluate the <= 4 lanes straddling the previous piece
// and advance the carry.  Run by k_stream_edge (finish, and pieces too short
// for K1) and by K1's first thread for the piece it validates, which saves a
// dependent launch per feed.
#pragma once
#include <stdint.h>

#include "utf8v_stream.h"

namespace u8v {

// state[0] = carry (the stream's last four bytes), state[1] = error flag.
__device__ __forceinline__ void stream_edge_piece(uint32_t* state, const uint8_t* piece, uint64_t n,
                                                  int finish) {
  uint32_t h0 = 0, h1 = 0, tail = 0;
  for (uint64_t i = 0; i < n && i < 8; ++i) {
    const uint32_t b = piece[i];
    if (i < 4) h0 |= b << (8 * i);
    else h1 |= b << (8 * (i - 4));
  }
  const uint32_t carry = state[0];
  if (u8v_stream_edge(carry, h0, h1, n, finish)) atomicOr(state + 1, 1u);
  if (finish) {
    state[0] = 0;  // ready for the next stream (the flag is read, then reset)
    return;
  }
  for (uint64_t i = 0; i < 4 && i < n; ++i) {
    const uint64_t src = n >= 4 ? n - 4 + i : i;
    tail |= (uint32_t)piece[src] << (8 * i);
  }
  state[0] = u8v_stream_carry(carry, tail, n);
}

}  // namespace u8v
