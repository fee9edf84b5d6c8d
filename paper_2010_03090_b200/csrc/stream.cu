// stream.cu -- a stream validated in pieces: the session's
// device state and the one-thread edge kernel of utf8v_stream.h.  Each fed
// piece is validated in place by K1 (lanes [3, n-1) of the piece), whose
// first thread also evaluates the <= 4 lanes that straddle the previous piece
// (stream_edge.cuh); this one-thread kernel runs them for finish() and for
// pieces too short to hold a K1 lane.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"
#include "stream_edge.cuh"

namespace u8v {

__global__ void k_stream_edge(uint32_t* state, const uint8_t* __restrict__ piece, uint64_t n,
                              int finish) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  stream_edge_piece(state, piece, n, finish);
}

void launch_stream_edge(uint32_t* d_state, const uint8_t* d_piece, uint64_t n, int finish,
                        cudaStream_t st) {
  k_stream_edge<<<1, 32, 0, st>>>(d_state, d_piece, n, finish);
}

}  // namespace u8v
