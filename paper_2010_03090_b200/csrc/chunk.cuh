// chunk.cuh -- 32-byte lane chunks shared by K1/K3 (validate.cu) and K2
// (batch.cu): 256-bit streaming loads, zero-masked edge loads, and the
// per-chunk lead-form evaluation of utf8v_swar.h.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"
#include "utf8v_bits.h"
#include "utf8v_swar.h"

namespace u8v {

struct Chunk {
  uint32_t w[kChunkWords];
};

// One 32-byte chunk, one LDG.E.ENL2.256 (no L1 allocation: every byte is
// read once; the halo travels by SHFL).
__device__ __forceinline__ Chunk ld_chunk(const uint8_t* p) {
  Chunk c;
  asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(c.w[0]), "=r"(c.w[1]), "=r"(c.w[2]), "=r"(c.w[3]), "=r"(c.w[4]), "=r"(c.w[5]),
        "=r"(c.w[6]), "=r"(c.w[7])
      : "l"(p));
  return c;
}

// w = the 32-bit word at p when pred, else w unchanged: one predicated LDG
// (the halo and lookahead words of a step are loaded by one lane each; an
// `if` there compiles to a branch with convergence barriers).
__device__ __forceinline__ void ld_word_if(bool pred, const uint8_t* p, uint32_t& w) {
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.nc.u32 %0, [%1];\n\t}"
      : "+r"(w)
      : "l"(p), "r"((unsigned)pred));
}

__device__ __forceinline__ Chunk zero_chunk() {
  Chunk r;
#pragma unroll
  for (int j = 0; j < kChunkWords; ++j) r.w[j] = 0;
  return r;
}

// One chunk with every byte outside [lo, hi) replaced by zero; only bytes
// inside the range are touched (edge chunks only).
__device__ __forceinline__ Chunk ld_chunk_masked(const uint8_t* base, int64_t c, int64_t lo,
                                                 int64_t hi) {
  const int64_t b0 = c * kChunkBytes;
  if (b0 >= lo && b0 + kChunkBytes <= hi) return ld_chunk(base + b0);
  Chunk r = zero_chunk();
  for (int k = 0; k < kChunkBytes; ++k) {
    const int64_t q = b0 + k;
    if (q >= lo && q < hi) r.w[k >> 2] |= (uint32_t)base[q] << (8 * (k & 3));
  }
  return r;
}

__device__ __forceinline__ uint32_t ld_word_masked(const uint8_t* base, int64_t pos, int64_t lo,
                                                   int64_t hi) {
  uint32_t w = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t q = pos + k;
    if (q >= lo && q < hi) w |= (uint32_t)base[q] << (8 * k);
  }
  return w;
}

// One 32-bit word, zero outside [lo, hi); a single LDG when fully inside.
__device__ __forceinline__ uint32_t ld_word_guarded(const uint8_t* base, int64_t pos, int64_t lo,
                                                    int64_t hi) {
  if (pos >= lo && pos + 4 <= hi) return __ldg(reinterpret_cast<const uint32_t*>(base + pos));
  return ld_word_masked(base, pos, lo, hi);
}

__device__ __forceinline__ uint32_t chunk_hibits(const Chunk& v) {
  uint32_t h = 0;
#pragma unroll
  for (int j = 0; j < kChunkWords; ++j) h |= v.w[j];
  return h;
}

// Error lanes of one chunk given the word before it and the word after it:
// the bit-sliced form of utf8v_bits.h.  Unranged (K1/K3 interior): the
// permuted-order form -- the result is nonzero iff some lane of the chunk is
// flagged, bit pos(i) = lane p0 + i.  kRanged (edge steps): natural order,
// bit i = lane p0 + i, lanes outside [L0, L1) dropped.
// *hi7: plane 7 of the chunk (zero iff all its bytes are ASCII).
template <bool kRanged>
__device__ __forceinline__ uint32_t chunk_errors(const Chunk& v, uint32_t prev, uint32_t next,
                                                 u8v_consts k, int64_t p0, int64_t L0, int64_t L1,
                                                 uint32_t* hi7) {
  if (!kRanged) return u8v_chunk_errors_planes_perm_k(v.w, prev, next, k, hi7);
  uint32_t e = u8v_chunk_errors_planes_k(v.w, prev, next, k, hi7);
  const int64_t a = L0 - p0, b = L1 - p0;  // wanted lanes: bits [a, b)
  const uint32_t lo = a <= 0 ? 0xFFFFFFFFu : (a >= 32 ? 0u : (0xFFFFFFFFu << a));
  const uint32_t hi = b >= 32 ? 0xFFFFFFFFu : (b <= 0 ? 0u : (0xFFFFFFFFu >> (32 - b)));
  return e & lo & hi;
}

}  // namespace u8v
