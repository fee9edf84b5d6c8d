// lanes.cu -- the lane-level entry points of the "cuda" lookup_backend.
//
// The reference exposes, per backend, classify_lanes / length_error_lanes /
// incomplete_lanes over exactly `width` bytes and a vector-operation self
// test (proj/include/utf8v/lookup.hpp:18-28, proj/src/lookup_backend_detail.hpp
// :16-43, proj/include/utf8v/lookup_kernel.hpp:139-216) so tests can compare
// backends lane by lane.  Here the "vector" is kLaneWidth = 64 bytes held as
// 16 32-bit words, one word per thread, and the byte_vector operations are
// SWAR device functions:
//   prev<N>        funnel shift across the word boundary (SHF.L.W)
//   shift_right<4> SHR + AND 0x0F per byte
//   lookup16       two PRMT 8-entry byte selects + a per-byte select on bit 3
//   saturating_sub __vsubus4,  unsigned_max __vmaxu4
// The tables are the reference's nibble tables (proj/include/utf8v/tables.hpp
// :60-99), built on the host exactly as the reference builds them and frozen
// against proj/tests/test_tables.cpp:26-34 by the test suite.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace u8v {

// Table 1/2/3 as 4 words each (byte k of word j = entry 4j+k).
__constant__ uint32_t c_tables[3][4];

__device__ __forceinline__ uint32_t v_prev(uint32_t cur, uint32_t before, int n) {
  return __funnelshift_l(before, cur, 8 * n);
}

__device__ __forceinline__ uint32_t v_shr4(uint32_t w) { return (w >> 4) & 0x0F0F0F0Fu; }

// lookup16 over four nibble lanes (each byte of x in 0..15).
__device__ __forceinline__ uint32_t v_lookup16(uint32_t x, const uint32_t t[4]) {
  const uint32_t idx = x & 0x07070707u;
  const uint32_t packed = idx | (idx >> 4);             // n1n0 in byte 0, n3n2 in byte 2
  const uint32_t sel = __byte_perm(packed, 0, 0x3320);  // 4 selector nibbles in bits 0..15
  const uint32_t lo = __byte_perm(t[0], t[1], sel);     // entries 0..7
  const uint32_t hi = __byte_perm(t[2], t[3], sel);     // entries 8..15
  const uint32_t m = ((x >> 3) & 0x01010101u) * 0xFFu;  // byte mask: nibble >= 8
  return (hi & m) | (lo & ~m);
}

__device__ __forceinline__ uint32_t v_classify(uint32_t in, uint32_t prev1) {
  return v_lookup16(v_shr4(prev1), c_tables[0]) & v_lookup16(prev1 & 0x0F0F0F0Fu, c_tables[1]) &
         v_lookup16(v_shr4(in), c_tables[2]);
}

// mode 0: classify (lookup_kernel.hpp:21-30); 1: check_multibyte_lengths
// (:38-46); 2: check_incomplete (:48-68).
__global__ void k_lanes(const uint8_t* __restrict__ in, const uint8_t* __restrict__ prev,
                        uint8_t* __restrict__ out, int mode) {
  const int j = threadIdx.x;  // word index 0..15
  constexpr int kWords = kLaneWidth / 4;
  if (j >= kWords) return;
  const uint32_t* iw = reinterpret_cast<const uint32_t*>(in);
  const uint32_t* pw = reinterpret_cast<const uint32_t*>(prev);
  const uint32_t w = iw[j];
  const uint32_t before = j > 0 ? iw[j - 1] : pw[kWords - 1];
  uint32_t r;
  if (mode == 2) {
    // max(v, L) ^ L with L = FF.. except the last three lanes EF DF BF.
    const uint32_t lim = j == kWords - 1 ? 0xBFDFEFFFu : 0xFFFFFFFFu;
    r = __vmaxu4(w, lim) ^ lim;
  } else {
    const uint32_t p1 = v_prev(w, before, 1);
    r = v_classify(w, p1);
    if (mode == 1) {
      const uint32_t p2 = v_prev(w, before, 2);
      const uint32_t p3 = v_prev(w, before, 3);
      const uint32_t third = __vsubus4(p2, 0x60606060u);   // prev2 - (E0 - 80), saturating
      const uint32_t fourth = __vsubus4(p3, 0x70707070u);  // prev3 - (F0 - 80)
      r ^= (third | fourth) & 0x80808080u;
    }
  }
  reinterpret_cast<uint32_t*>(out)[j] = r;
}

// vector_ops_self_test<V> (lookup_kernel.hpp:139-216) for the 64-byte SWAR
// vector: every operation against plain per-byte arithmetic, 64 rounds of the
// same xorshift stream.  One thread; a test entry point, not a hot path.
__global__ void k_ops_self_test(uint64_t seed, int* __restrict__ result) {
  constexpr int W = kLaneWidth, NW = W / 4;
  uint64_t state = seed ? seed : 1;
  auto next_byte = [&state]() {
    state ^= state << 13;
    state ^= state >> 7;
    state ^= state << 17;
    return (uint8_t)state;
  };
  auto word = [](const uint8_t* b, int j) {
    return (uint32_t)b[4 * j] | ((uint32_t)b[4 * j + 1] << 8) | ((uint32_t)b[4 * j + 2] << 16) |
           ((uint32_t)b[4 * j + 3] << 24);
  };
  int ok = 1;
  for (int round = 0; round < 64 && ok; ++round) {
    uint8_t a[W], b[W], e[W], nib[W];
    uint8_t tb[16];
    for (int i = 0; i < W; ++i) a[i] = next_byte();
    for (int i = 0; i < W; ++i) b[i] = next_byte();
    for (int i = 0; i < 16; ++i) tb[i] = next_byte();
    const uint8_t s = next_byte();
    uint32_t t[4];
    for (int j = 0; j < 4; ++j) t[j] = word(tb, j);
    for (int i = 0; i < W; ++i) nib[i] = a[i] & 0x0F;
    const uint32_t ss = 0x01010101u * s;
    bool all_ascii = true, nonzero = false;
    uint32_t orw = 0;
    for (int j = 0; j < NW; ++j) {
      const uint32_t wa = word(a, j), wb = word(b, j);
      const uint32_t wa_before = j > 0 ? word(a, j - 1) : word(b, NW - 1);
      uint32_t got[12];
      got[0] = wa & wb;
      got[1] = wa | wb;
      got[2] = wa ^ wb;
      got[3] = wa & ~wb;
      got[4] = wa & ss;
      got[5] = v_prev(wa, wa_before, 1);
      got[6] = v_prev(wa, wa_before, 2);
      got[7] = v_prev(wa, wa_before, 3);
      got[8] = v_shr4(wa);
      got[9] = v_lookup16(word(nib, j), t);
      got[10] = __vsubus4(wa, ss);
      got[11] = __vmaxu4(wa, wb);
      orw |= wa;
      for (int k = 0; k < 4; ++k) {
        const int i = 4 * j + k;
        uint8_t want[12];
        want[0] = a[i] & b[i];
        want[1] = a[i] | b[i];
        want[2] = a[i] ^ b[i];
        want[3] = a[i] & (uint8_t)~b[i];
        want[4] = a[i] & s;
        want[5] = i >= 1 ? a[i - 1] : b[W - 1 + i];
        want[6] = i >= 2 ? a[i - 2] : b[W - 2 + i];
        want[7] = i >= 3 ? a[i - 3] : b[W - 3 + i];
        want[8] = a[i] >> 4;
        want[9] = tb[nib[i]];
        want[10] = a[i] > s ? (uint8_t)(a[i] - s) : 0;
        want[11] = a[i] > b[i] ? a[i] : b[i];
        for (int op = 0; op < 12; ++op)
          if ((uint8_t)(got[op] >> (8 * k)) != want[op]) ok = 0;
        all_ascii = all_ascii && a[i] < 0x80;
        nonzero = nonzero || a[i] != 0;
      }
      (void)e;
    }
    if (((orw & 0x80808080u) == 0) != all_ascii) ok = 0;
    if ((orw != 0) != nonzero) ok = 0;
    // zero / splat identities (lookup_kernel.hpp:212-215)
    if ((0u & 0x80808080u) != 0) ok = 0;
    if ((0x80808080u & 0x80808080u) == 0) ok = 0;
    if ((0x7F7F7F7Fu & 0x80808080u) != 0) ok = 0;
  }
  *result = ok;
}

void set_tables(const uint8_t t1[16], const uint8_t t2[16], const uint8_t t3[16]) {
  uint32_t h[3][4];
  const uint8_t* src[3] = {t1, t2, t3};
  for (int t = 0; t < 3; ++t)
    for (int j = 0; j < 4; ++j)
      h[t][j] = (uint32_t)src[t][4 * j] | ((uint32_t)src[t][4 * j + 1] << 8) |
                ((uint32_t)src[t][4 * j + 2] << 16) | ((uint32_t)src[t][4 * j + 3] << 24);
  cudaMemcpyToSymbol(c_tables, h, sizeof h);
}

void launch_classify_lanes(const uint8_t* in, const uint8_t* prev, uint8_t* out, int mode,
                           cudaStream_t st) {
  k_lanes<<<1, kLaneWidth / 4, 0, st>>>(in, prev, out, mode);
}

void launch_ops_self_test(uint64_t seed, int* result, cudaStream_t st) {
  k_ops_self_test<<<1, 1, 0, st>>>(seed, result);
}

}  // namespace u8v
