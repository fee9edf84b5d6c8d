// stream.cu -- a stream validated in pieces: the session's
// device state and the one-thread edge kernel of utf8v_stream.h.  Each fed
// piece is validated in place by K1 (lanes [3, n-1) of the piece); only the
// <= 4 lanes that straddle the previous piece run here.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"
#include "utf8v_stream.h"

namespace u8v {

// state[0] = carry (the stream's last four bytes), state[1] = error flag.
__global__ void k_stream_edge(uint32_t* state, const uint8_t* __restrict__ piece, uint64_t n,
                              int finish) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t h0 = 0, h1 = 0, tail = 0;
  for (uint64_t i = 0; i < n && i < 8; ++i) {
    const uint32_t b = piece[i];
    if (i < 4) h0 |= b << (8 * i);
    else h1 |= b << (8 * (i - 4));
  }
  const uint32_t carry = state[0];
  if (u8v_stream_edge(carry, h0, h1, n, finish)) state[1] = 1u;
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

void launch_stream_edge(uint32_t* d_state, const uint8_t* d_piece, uint64_t n, int finish,
                        cudaStream_t st) {
  k_stream_edge<<<1, 32, 0, st>>>(d_state, d_piece, n, finish);
}

}  // namespace u8v
