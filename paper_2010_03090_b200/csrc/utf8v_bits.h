// utf8v_bits.h -- the per-lane Lookup check on bit planes (bit-sliced form).
//
// Same lane predicate as u8v_word_errors_lead (utf8v_swar.h), evaluated for a
// whole 32-byte chunk at once: the chunk is transposed into 8 planes (plane k,
// bit i = bit k of byte i), so every LOP3 of the check covers 32 byte lanes
// instead of the 4 of the SWAR form, and the look-back/lookahead becomes a
// one-bit funnel shift per plane.  K1 is bound by the ALU pipe; per 4-byte
// word this form issues ~10 ALU + ~6 FMA instructions against ~15 + ~13 for
// the SWAR form (tools/kbench.cu: 3592 -> 4476 GB/s on C1).
//
// Transpose: a 4x4 byte transpose by PRMT lines up row q of the four 8x8 bit
// blocks in one register, then three cross-register stages transpose all four
// blocks at once (2 shifts + 2 LOP3 per register pair and stage: 16 PRMT +
// 24 LOP3 + 24 IMAD per chunk).  Shifts are issued as IMAD / IMAD.HI with
// runtime multipliers (FMA pipe); the logic stays on LOP3.
//
// Compiled into the sm_100a kernels and, by gcc, into the CPU test helper
// that checks the transpose and every lane class at every chunk position
// against the SWAR form (tests/test_swar.py).
#pragma once
#include <stdint.h>

#include "utf8v_swar.h"

U8V_HD uint32_t u8v_prmt(uint32_t x, uint32_t y, uint32_t s) {
#if defined(__CUDA_ARCH__)
  return __byte_perm(x, y, s);
#else
  const uint64_t v = ((uint64_t)y << 32) | x;
  uint32_t r = 0;
  for (int n = 0; n < 4; ++n) r |= (uint32_t)((v >> (8 * ((s >> (4 * n)) & 7))) & 0xFF) << (8 * n);
  return r;
#endif
}

// x << s and x >> s on the FMA pipe: a multiply by an immediate power of two
// (IMAD.SHL) and a multiply-high (IMAD.HI).  Inline PTX keeps ptxas from
// turning them into SHF/LEA on the ALU pipe, and immediates need no
// registers (no per-chunk rematerialisation under register pressure).
#if defined(__CUDA_ARCH__)
template <unsigned kMul>
__device__ __forceinline__ uint32_t u8v_mul_imm(uint32_t x) {
  uint32_t d;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "n"(kMul));
  return d;
}
template <unsigned kMul>
__device__ __forceinline__ uint32_t u8v_mulhi_imm(uint32_t x) {
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(x), "n"(kMul));
  return d;
}
// x * kMul + y (kMul an immediate; IMAD).
template <unsigned kMul>
__device__ __forceinline__ uint32_t u8v_mad_imm(uint32_t x, uint32_t y) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(x), "n"(kMul), "r"(y));
  return d;
}
#define U8V_SHL(x, s, k) u8v_mul_imm<(1u << (s))>(x)
#define U8V_SHR(x, s, k) u8v_mulhi_imm<(1u << (32 - (s)))>(x)
#define U8V_SHLADD(x, s, y, k) u8v_mad_imm<(1u << (s))>((x), (y))
#else
#define U8V_SHLADD(x, s, y, k) ((((uint32_t)(x)) << (s)) + (uint32_t)(y))
#define U8V_SHL(x, s, k) ((uint32_t)(x) << (s))
#define U8V_SHR(x, s, k) ((uint32_t)(x) >> (s))
#endif

// (x & m) | (y & ~m) in one LOP3 with m an immediate (ptxas splits the
// expression in two when m appears in both polarities).
#if defined(__CUDA_ARCH__)
#define U8V_BITSEL(m, x, y)                                                        \
  ([](uint32_t xx, uint32_t yy) {                                                  \
    uint32_t d;                                                                    \
    asm("lop3.b32 %0, %1, " #m ", %2, 0xE2;" : "=r"(d) : "r"(xx), "r"(yy));        \
    return d;                                                                      \
  }((x), (y)))
#else
#define U8V_BITSEL(m, x, y) ((((uint32_t)(x)) & (uint32_t)(m)) | (((uint32_t)(y)) & ~(uint32_t)(m)))
#endif

// One stage of the 8x8 bit transpose across a register pair (x = row a,
// y = row a + s, per byte lane): the bits of x at columns with bit log2(s)
// set trade places with the bits of y s columns lower.  Two shifts (FMA
// pipe) and two LOP3 per pair.
#define U8V_XSTAGE(x, y, s, mhi, mlo, k)                                  \
  do {                                                                    \
    const uint32_t _x = (x), _y = (y);                                    \
    (x) = U8V_BITSEL(mhi, U8V_SHL(_y, s, k), _x);                          \
    (y) = U8V_BITSEL(mlo, U8V_SHR(_x, s, k), _y);                          \
  } while (0)

// Planes of a 32-byte chunk w[0..8): p[c] bit i = bit c of byte i.
// 1. Two 4x4 byte transposes (PRMT) make r[q] = byte q of each 8-byte block
//    (r[q] byte j = byte 8j+q): row q of the four 8x8 bit blocks, side by side.
// 2. Three cross-register stages (s = 1, 2, 4) transpose every 8x8 block at
//    once: afterwards r[c] byte j bit q = bit c of byte 8j+q, i.e. plane c.
U8V_HD void u8v_planes_k(const uint32_t w[8], uint32_t p[8], u8v_consts k) {
  // rows 0..3 come from the even words (bytes 8j..8j+3), rows 4..7 from the odd.
  uint32_t A = u8v_prmt(w[0], w[2], 0x5140), B = u8v_prmt(w[0], w[2], 0x7362);
  uint32_t C = u8v_prmt(w[4], w[6], 0x5140), D = u8v_prmt(w[4], w[6], 0x7362);
  uint32_t r0 = u8v_prmt(A, C, 0x5410), r1 = u8v_prmt(A, C, 0x7632);
  uint32_t r2 = u8v_prmt(B, D, 0x5410), r3 = u8v_prmt(B, D, 0x7632);
  A = u8v_prmt(w[1], w[3], 0x5140);
  B = u8v_prmt(w[1], w[3], 0x7362);
  C = u8v_prmt(w[5], w[7], 0x5140);
  D = u8v_prmt(w[5], w[7], 0x7362);
  uint32_t r4 = u8v_prmt(A, C, 0x5410), r5 = u8v_prmt(A, C, 0x7632);
  uint32_t r6 = u8v_prmt(B, D, 0x5410), r7 = u8v_prmt(B, D, 0x7632);
  U8V_XSTAGE(r0, r1, 1, 0xAAAAAAAA, 0x55555555, k);
  U8V_XSTAGE(r2, r3, 1, 0xAAAAAAAA, 0x55555555, k);
  U8V_XSTAGE(r4, r5, 1, 0xAAAAAAAA, 0x55555555, k);
  U8V_XSTAGE(r6, r7, 1, 0xAAAAAAAA, 0x55555555, k);
  U8V_XSTAGE(r0, r2, 2, 0xCCCCCCCC, 0x33333333, k);
  U8V_XSTAGE(r1, r3, 2, 0xCCCCCCCC, 0x33333333, k);
  U8V_XSTAGE(r4, r6, 2, 0xCCCCCCCC, 0x33333333, k);
  U8V_XSTAGE(r5, r7, 2, 0xCCCCCCCC, 0x33333333, k);
  U8V_XSTAGE(r0, r4, 4, 0xF0F0F0F0, 0x0F0F0F0F, k);
  U8V_XSTAGE(r1, r5, 4, 0xF0F0F0F0, 0x0F0F0F0F, k);
  U8V_XSTAGE(r2, r6, 4, 0xF0F0F0F0, 0x0F0F0F0F, k);
  U8V_XSTAGE(r3, r7, 4, 0xF0F0F0F0, 0x0F0F0F0F, k);
  p[0] = r0;
  p[1] = r1;
  p[2] = r2;
  p[3] = r3;
  p[4] = r4;
  p[5] = r5;
  p[6] = r6;
  p[7] = r7;
}

U8V_HD void u8v_planes(const uint32_t w[8], uint32_t p[8]) { u8v_planes_k(w, p, u8v_make_consts()); }

// Bit 7 of each byte of x gathered into bits 28..31 (byte 0 -> bit 28): the
// top four lanes of a plane, from a SWAR flag word.  One IMAD.
U8V_HD uint32_t u8v_movemask_top(uint32_t x, u8v_consts k) {
  (void)k;
#if defined(__CUDA_ARCH__)
  return u8v_mul_imm<0x00204081u>(x & U8V_B7);
#else
  return (x & U8V_B7) * 0x00204081u;
#endif
}

// The rare lead pairs on planes (utf8v_swar.h u8v_rare_key restated), lead
// lanes l1/l2/l3 (>= C0/E0/F0), the lead's low bits p5..p0, the follower's
// bits 5 and 4 (n5, n4; meaningful when the follower is a continuation, else
// S fires anyway).  Factored so every line is one 3-input LOP3:
//   C0/C1  l1 & ~p5 & ~p4 & lo=0|1               (z = ~(p3|p2|p1))
//   E0/F0  z & ~p0 & ~n5 & l2 & ~(p4 & n4)       (E0: b<A0; F0: b<90)
//   ED     l2 & ~p4 & (p3 & p2 & ~p1) & p0 & n5  (b >= A0)
//   F4     l3 & (~p3 & p2 & ~p1) & ~p0 & (n5|n4) (b >= 90)
//   F5..FF l3 & (p3 | p2 & (p1 | p0))
U8V_HD uint32_t u8v_rare_planes(uint32_t l1, uint32_t l2, uint32_t l3, uint32_t p5, uint32_t p4,
                                uint32_t p3, uint32_t p2, uint32_t p1, uint32_t p0, uint32_t n5,
                                uint32_t n4) {
  const uint32_t z = ~(p3 | p2 | p1);
  const uint32_t rc = (l1 & ~p5 & ~p4) & z;
  const uint32_t x = z & ~p0 & ~n5;
  const uint32_t y = l2 & ~(p4 & n4);
  const uint32_t ed = (p3 & p2 & ~p1) & (p0 & n5);
  const uint32_t red = (l2 & ~p4) & ed;
  const uint32_t f4 = (~p3 & p2 & ~p1) & (~p0 & (n5 | n4));
  const uint32_t rf5 = l3 & (p3 | (p2 & (p1 | p0)));
  return rc | (x & y) | red | (l3 & f4) | rf5;
}

// Error plane (bit i = lane i of the chunk flagged) of one chunk.
//   prev: the word before the chunk (bytes -4..-1), next: the word after it.
// Lane i: S_i = cont(x_i) ^ (x_{i-1}>=C0 | x_{i-2}>=E0 | x_{i-3}>=F0), and the
// rare pair (x_i, x_{i+1}) tested at its lead (lead form, utf8v_swar.h).
// *hi7 receives plane 7 (the bytes >= 0x80): zero iff the chunk is ASCII.
U8V_HD uint32_t u8v_chunk_errors_planes_k(const uint32_t w[8], uint32_t prev, uint32_t next,
                                          u8v_consts k, uint32_t* hi7) {
  uint32_t p[8];
  u8v_planes_k(w, p, k);
  *hi7 = p[7];
  // Lead flags of this chunk's bytes.
  const uint32_t l1 = p[7] & p[6];  // >= C0
  const uint32_t l2 = l1 & p[5];    // >= E0
  const uint32_t l3 = l2 & p[4];    // >= F0
  // The same flags of the 4 bytes before the chunk, as the top plane lanes.
  const uint32_t q1 = prev & U8V_SHL(prev, 1, k);
  const uint32_t q2 = q1 & U8V_SHL(prev, 2, k);
  const uint32_t q3 = q2 & U8V_SHL(prev, 3, k);
  const uint32_t e1 = u8v_fsl(u8v_movemask_top(q1, k), l1, 1);
  const uint32_t e2 = u8v_fsl(u8v_movemask_top(q2, k), l2, 2);
  const uint32_t e3 = u8v_fsl(u8v_movemask_top(q3, k), l3, 3);
  const uint32_t S = (p[7] & ~p[6]) ^ (e1 | e2 | e3);
  // Follower bits 5 and 4 (byte i+1) at lane i.
  const uint32_t n5 = u8v_fsr(p[5], next >> 5, 1);
  const uint32_t n4 = u8v_fsr(p[4], next >> 4, 1);
  // Rare pairs (utf8v_swar.h u8v_rare_key, restated on planes).
  return S | u8v_rare_planes(l1, l2, l3, p[5], p[4], p[3], p[2], p[1], p[0], n5, n4);
}

U8V_HD uint32_t u8v_chunk_errors_planes(const uint32_t w[8], uint32_t prev, uint32_t next) {
  uint32_t hi7;
  return u8v_chunk_errors_planes_k(w, prev, next, u8v_make_consts(), &hi7);
}

// ---- permuted-order form (K1, K2, K3) -------------------------------------
// Without the PRMT row gather the eight words of a chunk already are the
// rows of four 8x8 bit blocks -- block b = bytes {b, b+4, ..., b+28} -- so the
// three cross-register stages alone give the planes, in the order
//   pos(i) = 8 * (i mod 4) + (i div 4)       (byte i = 4q + b  ->  bit 8b + q).
// K1/K3 only need "some lane of the chunk is flagged", so only the shifted
// planes must follow the permutation:
//   look-back by k (k = 1..3):  byte i-k is at pos(i) - 8k when b >= k, else at
//     pos(i) + 31 - 8k (word q-1), or in the previous chunk when q = 0:
//     lag_k(P) = (P << 8k) + ((P >> (31-8k)) & M_k | carry_k),
//     M_k = bits [0, 8k) without {0, 8, 16}, carry_k = the flags of the
//     previous word's bytes 4-k..3 landing on bits 0, 8, 16: one IMAD.HI of
//     the bit-7 flag word, (f >> (39 - 8k)).
//   lookahead (byte i+1): pos(i) + 8 when b <= 2, else pos(i) - 23 (word
//     q+1), or the next chunk's byte 0 for i = 31: a funnel shift by 8 of
//     ((P >> 1) & 0x7F | next-byte bit << 7 : P).
// 16 PRMT fewer per chunk than u8v_chunk_errors_planes_k; same lane flags
// (tests/test_swar.py maps the bits back and compares).
U8V_HD uint32_t u8v_perm_pos(unsigned i) { return 8u * (i & 3u) + (i >> 2); }

U8V_HD uint32_t u8v_chunk_errors_planes_perm_k(const uint32_t w[8], uint32_t prev, uint32_t next,
                                               u8v_consts k, uint32_t* hi7) {
  uint32_t r0 = w[0], r1 = w[1], r2 = w[2], r3 = w[3], r4 = w[4], r5 = w[5], r6 = w[6], r7 = w[7];
  U8V_XSTAGE(r0, r1, 1, 0xAAAAAAAA, 0x55555555, k);
  U8V_XSTAGE(r2, r3, 1, 0xAAAAAAAA, 0x55555555, k);
  U8V_XSTAGE(r4, r5, 1, 0xAAAAAAAA, 0x55555555, k);
  U8V_XSTAGE(r6, r7, 1, 0xAAAAAAAA, 0x55555555, k);
  U8V_XSTAGE(r0, r2, 2, 0xCCCCCCCC, 0x33333333, k);
  U8V_XSTAGE(r1, r3, 2, 0xCCCCCCCC, 0x33333333, k);
  U8V_XSTAGE(r4, r6, 2, 0xCCCCCCCC, 0x33333333, k);
  U8V_XSTAGE(r5, r7, 2, 0xCCCCCCCC, 0x33333333, k);
  U8V_XSTAGE(r0, r4, 4, 0xF0F0F0F0, 0x0F0F0F0F, k);
  U8V_XSTAGE(r1, r5, 4, 0xF0F0F0F0, 0x0F0F0F0F, k);
  U8V_XSTAGE(r2, r6, 4, 0xF0F0F0F0, 0x0F0F0F0F, k);
  U8V_XSTAGE(r3, r7, 4, 0xF0F0F0F0, 0x0F0F0F0F, k);
  const uint32_t p0 = r0, p1 = r1, p2 = r2, p3 = r3, p4 = r4, p5 = r5, p6 = r6, p7 = r7;
  *hi7 = p7;
  const uint32_t l1 = p7 & p6;  // >= C0
  const uint32_t l2 = l1 & p5;  // >= E0
  const uint32_t l3 = l2 & p4;  // >= F0
  // Bit-7 flags of the previous word's bytes.
  const uint32_t q1 = prev & U8V_SHL(prev, 1, k) & U8V_B7;
  const uint32_t q2 = q1 & U8V_SHL(prev, 2, k);
  const uint32_t q3 = q2 & U8V_SHL(prev, 3, k);
  const uint32_t t1 = U8V_BITSEL(0x000000FE, U8V_SHR(l1, 23, k), U8V_SHR(q1, 31, k));
  const uint32_t t2 = U8V_BITSEL(0x0000FEFE, U8V_SHR(l2, 15, k), U8V_SHR(q2, 23, k));
  const uint32_t t3 = U8V_BITSEL(0x00FEFEFE, U8V_SHR(l3, 7, k), U8V_SHR(q3, 15, k));
  const uint32_t e1 = U8V_SHLADD(l1, 8, t1, k);
  const uint32_t e2 = U8V_SHLADD(l2, 16, t2, k);
  const uint32_t e3 = U8V_SHLADD(l3, 24, t3, k);
  const uint32_t S = (p7 & ~p6) ^ (e1 | e2 | e3);
  // Follower bits 5 and 4 at the lead's position.
  const uint32_t nx5 = U8V_SHL(next, 2, k);  // bit 7 = next byte 0's bit 5
  const uint32_t nx4 = U8V_SHL(next, 3, k);  // bit 7 = next byte 0's bit 4
  const uint32_t n5 = u8v_fsr(p5, U8V_BITSEL(0x7F, U8V_SHR(p5, 1, k), nx5), 8);
  const uint32_t n4 = u8v_fsr(p4, U8V_BITSEL(0x7F, U8V_SHR(p4, 1, k), nx4), 8);
  return S | u8v_rare_planes(l1, l2, l3, p5, p4, p3, p2, p1, p0, n5, n4);
}

// Byte index of permuted position pos (inverse of u8v_perm_pos).
U8V_HD unsigned u8v_perm_byte(unsigned pos) { return 4u * (pos & 7u) + (pos >> 3); }
