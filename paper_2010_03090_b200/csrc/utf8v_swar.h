// utf8v_swar.h -- the per-word Lookup check, 4 byte lanes per 32-bit register.
//
// Compiled by nvcc into the sm_100a kernels (validate.cu, batch.cu) and, for
// exhaustive verification only, by gcc into a test helper (tests/cpp): the same
// source is checked on the CPU against the oracle for every input of length
// <= 3 and against fuzz corpora, so what runs on the GPU is what was proven.
//
// Semantics (the reference's Lookup verdict, proj/include/utf8v/lookup_kernel.hpp
// :21-134, restated per lane over the zero-extended stream x, x[i] = 0 outside
// [0,n)).  The input is invalid iff some lane i in [0, n+3) has
//
//   S_i = cont(x[i]) XOR (x[i-1] >= C0 | x[i-2] >= E0 | x[i-3] >= F0)
//       -- the classification's too-short / too-long bits plus the 2/3/4-byte
//          continuation cross-check (lookup_kernel.hpp:38-46: bit 7 of the
//          three-table AND is "two continuations", XORed with prev2>=E0 |
//          prev3>=F0), folded into one structural test;
//   R_i = x[i-1] in {C0,C1} | x[i-1] >= F5 | (x[i-1]=E0 & x[i]<A0)
//       | (x[i-1]=ED & x[i]>=A0) | (x[i-1]=F0 & x[i]<90) | (x[i-1]=F4 & x[i]>=90)
//       -- the nibble-table bits 2..6 (tables.hpp:60-79: overlong-3, too-large,
//          surrogate, overlong-2, overlong-4/5+), restated on the pair.
//
// Lanes n..n+2 reduce to check_incomplete (lookup_kernel.hpp:48-68) and an
// all-ASCII block contributes exactly the pending incomplete check (:94-96).
// The equivalence with the nibble-table formulation is proven exhaustively for
// all 65,536 byte pairs at every lane of a word and every input of length <= 3
// by tests/test_swar.py (CPU), and on the GPU by tests/test_gpu_parity.py.
//
// Bit layout: byte k of a word is bits 8k..8k+7 (little-endian memory order);
// all per-lane flags live in bit 7 of their byte.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define U8V_HD __host__ __device__ __forceinline__
#else
#define U8V_HD static inline
#endif

// Upper 32 bits of ((hi:lo) << s), 0 < s < 32.  SHF.L.W on sm_100a.
U8V_HD uint32_t u8v_fsl(uint32_t lo, uint32_t hi, unsigned s) {
#if defined(__CUDA_ARCH__)
  return __funnelshift_l(lo, hi, s);
#else
  return (hi << s) | (lo >> (32 - s));
#endif
}

#define U8V_B7 0x80808080u

// Integer multiply-add / multiply-high routed to the FMA pipe.  On sm_100a
// LOP3/SHF/IADD3/VIADD share the ALU pipe (16 lanes/clk/SMSP), which the
// per-byte logic saturates; IMAD runs on the FMA pipe at the same rate.
// The multipliers come from kernel arguments (u8v_consts) so ptxas cannot
// strength-reduce "x*1+K" back into an ALU add or "mulhi(x, 2^k)" into a
// shift.  Host builds (the CPU checker) compute the same values in C.
typedef struct {
  uint32_t one;    // 1
  uint32_t m256;   // 1 << 8
  uint32_t mshr4;  // 1 << 28: mulhi(x, 1<<28) == x >> 4
} u8v_consts;

U8V_HD u8v_consts u8v_make_consts(void) {
  u8v_consts k;
  k.one = 1u;
  k.m256 = 256u;
  k.mshr4 = 1u << 28;
  return k;
}

U8V_HD uint32_t u8v_mad(uint32_t a, uint32_t b, uint32_t c) {
#if defined(__CUDA_ARCH__)
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
#else
  return a * b + c;
#endif
}

U8V_HD uint32_t u8v_mulhi(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

// Lane flags of the word before the current one.  p is the raw word; f1/f2/f3
// hold, in bit 7 of each byte, byte >= C0 / >= E0 / >= F0.
typedef struct {
  uint32_t p, f1, f2, f3;
  uint32_t ph;  // p >> 24: the byte that precedes the current word
} u8v_carry;

U8V_HD u8v_carry u8v_carry_of(uint32_t p) {
  u8v_carry c;
  c.p = p;
  c.f1 = p & (p << 1);
  c.f2 = c.f1 & (p << 2);
  c.f3 = c.f2 & (p << 3);
  c.ph = p >> 24;
  return c;
}

U8V_HD u8v_carry u8v_carry_zero(void) {
  u8v_carry c;
  c.p = 0;
  c.f1 = 0;
  c.f2 = 0;
  c.f3 = 0;
  c.ph = 0;
  return c;
}

// R: the rare lead pairs, for the pair (a = x[i-1], b = x[i]) in every lane.
// Key zl = a4 a3 a2 a1 a0 b5 b4 (7 bits); bit 7 of a*4 is a5.
//   a in C0..DF (a5 = 0): error iff a4 a3 a2 a1 = 0 (C0/C1)  <=>  zl < 08
//   a >= E0 (a5 = 1; E row a4 = 0, F row a4 = 1; b is a continuation or S
//   fires): E0 & b<A0 -> zl in {00,01}, ED & b>=A0 -> zl in {36,37},
//           F0 & b<90 -> zl == 40, F4 & b>=90 or F5..FF -> zl >= 51.
// Each threshold is one add into bit 7 (zl < 0x80, addend <= 0x7E: no carry
// leaves a lane), issued as IMAD on the FMA pipe.  `a`, the word of previous
// bytes, is w*256 + (byte before w), also on the FMA pipe.  Gated by e1
// (x[i-1] >= C0); flags in bit 7, garbage elsewhere.
U8V_HD uint32_t u8v_rare_key(uint32_t a4, uint32_t zl, uint32_t e1, u8v_consts k) {
  const uint32_t ge08 = u8v_mad(zl, k.one, 0x78787878u);  // bit7: zl >= 0x08
  const uint32_t ge02 = u8v_mad(zl, k.one, 0x7E7E7E7Eu);  // zl >= 0x02
  const uint32_t ge36 = u8v_mad(zl, k.one, 0x4A4A4A4Au);  // zl >= 0x36
  const uint32_t ge38 = u8v_mad(zl, k.one, 0x48484848u);  // zl >= 0x38
  const uint32_t ge40 = u8v_mad(zl, k.one, 0x40404040u);  // zl >= 0x40
  const uint32_t ge41 = u8v_mad(zl, k.one, 0x3F3F3F3Fu);  // zl >= 0x41
  const uint32_t ge51 = u8v_mad(zl, k.one, 0x2F2F2F2Fu);  // zl >= 0x51
  const uint32_t bad_ef = ~ge02 | (ge36 & ~ge38) | (ge40 & ~ge41) | ge51;
  return e1 & ((a4 & bad_ef) | (~a4 & ~ge08));
}

// Upper 32 bits of ((hi:lo) >> s), 0 < s < 32.  SHF.R.W on sm_100a.
U8V_HD uint32_t u8v_fsr(uint32_t lo, uint32_t hi, unsigned s) {
#if defined(__CUDA_ARCH__)
  return __funnelshift_r(lo, hi, s);
#else
  return (lo >> s) | (hi << (32 - s));
#endif
}

// Lead form (K1's hot loop): the same S, but each rare pair (a, b) is tested
// at the lane of its lead a, from w itself and the next word wn -- w << 2 is
// already needed by S and the lead flag f1 is unshifted, so the pair key
// costs one funnel shift instead of four IMADs.  The flag of pair (j, j+1)
// sits at lane j; lane j therefore reads byte j+1 (zero past the stream end).
// Position bound: a flagged lead j is at or after the sequential first
// error E (a bad pair at a character start is E itself; a lead inside
// another character's continuation region also fails S there), so the first
// flagged lane still satisfies E <= L <= E+3 (tests/test_swar.py).
//
// The lead flags are threshold adds on h = (w >> 1) & 0x7F..: bit 7 of
// h + 0x20 / 0x10 / 0x08 is byte >= C0 / E0 / F0 (h < 0x80: no carry leaves a
// lane).  One mask on the ALU pipe plus four IMADs replaces three LOP3s and
// two shifts -- the loop is bound by the ALU pipe, so this is a measured
// +4% (tools/kbench.cu, V6 vs V4).  Only bit 7 of f1/f2/f3 is meaningful,
// as with the AND form.
U8V_HD uint32_t u8v_word_errors_lead(uint32_t w, uint32_t wn, u8v_carry* c, u8v_consts k) {
  const uint32_t s1 = w << 1, s2 = w << 2;
  const uint32_t h = u8v_mulhi(w, 0x80000000u) & 0x7F7F7F7Fu;  // w >> 1, lanes kept apart
  const uint32_t f1 = u8v_mad(h, k.one, 0x20202020u);            // >= C0
  const uint32_t f2 = u8v_mad(h, k.one, 0x10101010u);            // >= E0
  const uint32_t f3 = u8v_mad(h, k.one, 0x08080808u);            // >= F0
  const uint32_t e1 = u8v_fsl(c->f1, f1, 8);
  const uint32_t e2 = u8v_fsl(c->f2, f2, 16);
  const uint32_t e3 = u8v_fsl(c->f3, f3, 24);
  const uint32_t S = (e1 | e2 | e3) ^ (w & ~s1);
  const uint32_t t = u8v_fsr(w, wn, 12);  // bits 1,0 of lane j = bits 5,4 of byte j+1
  const uint32_t zl = (s2 & 0x7C7C7C7Cu) | (t & 0x03030303u);
  const uint32_t R = u8v_rare_key(s2, zl, f1, k);
  c->p = w;
  c->f1 = f1;
  c->f2 = f2;
  c->f3 = f3;
  return S | R;
}

// A record boundary at byte s, for K2's unbounded sweep (batch.cu).  w8
// holds bytes s-4 .. s+3 (byte k of w8 = byte s-4+k).  A = the record ending
// at s owns bytes k in [ka, 4), B = the record starting at s owns bytes k in
// [4, kb) (ka = 4: no A bytes, kb = 4: no B bytes); every other byte is
// dropped, so each record is its own zero-extended stream.  Returns bit 0 if
// A's end-of-stream lanes (n_A .. n_A+2, lookup_kernel.hpp:48-68, :111)
// flag, bit 1 if one of B's first three lanes (look-back within B only,
// from the zero prev vector of lookup_kernel.hpp:115) flags.  These are the
// only lanes whose record-bounded flag can differ from the unbounded one.
// The rare pair needs no bound in the lead form: a flagged pair (j, j+1)
// that crosses into the next record means byte j is a lead that ends its
// record, which is invalid anyway (its end check fires too), and the flag
// sits on that record's lane.
U8V_HD uint32_t u8v_boundary_errors(uint64_t w8, unsigned ka, unsigned kb, u8v_consts k) {
  const uint64_t keep_a = ka >= 4 ? 0ull : (0xFFFFFFFFull & ~((1ull << (8 * ka)) - 1ull));
  const uint64_t keep_b = kb <= 4 ? 0ull : ((kb >= 8 ? ~0ull : (1ull << (8 * kb)) - 1ull) & ~0xFFFFFFFFull);
  const uint32_t xa = (uint32_t)(w8 & keep_a);
  const uint32_t xb = (uint32_t)((w8 & keep_b) >> 32);
  // A's lanes n_A .. n_A+2 read zeros from n_A on: they flag iff a lead in
  // A's last three bytes wants more bytes than A has (byte 3 of xa >= C0,
  // byte 2 >= E0, byte 1 >= F0) -- bit 7 of each byte of t1/t2/t3 is
  // "byte >= C0/E0/F0".
  const uint32_t t1 = xa & (xa << 1);
  const uint32_t t2 = t1 & (xa << 2);
  const uint32_t t3 = t2 & (xa << 3);
  const uint32_t ea = (t1 & 0x80000000u) | (t2 & 0x00800000u) | (t3 & 0x00008000u);
  u8v_carry z = u8v_carry_zero();
  const uint32_t eb = u8v_word_errors_lead(xb, 0, &z, k) & 0x00808080u;  // B's lanes 0 .. 2
  return (ea ? 1u : 0u) | (eb ? 2u : 0u);
}

// Spread 4 bits (bit k = byte k) to bit 7 of each byte.
U8V_HD uint32_t u8v_spread4(uint32_t x) { return ((x & 0xFu) * 0x10204080u) & U8V_B7; }

// Errors contributed by a word of all-ASCII bytes (no leads, no
// continuations): only the continuation expected from the previous word's
// last three bytes -- the pending incomplete check of lookup_kernel.hpp:94-96.
U8V_HD uint32_t u8v_ascii_word_errors(uint32_t w, u8v_carry* c) {
  const uint32_t e = u8v_fsl(c->f1, 0, 8) | u8v_fsl(c->f2, 0, 16) | u8v_fsl(c->f3, 0, 24);
  c->p = w;
  c->f1 = 0;
  c->f2 = 0;
  c->f3 = 0;
  c->ph = w >> 24;
  return e;
}

// Bytes outside [lo, hi) of word at byte position `pos` replaced by zero --
// the zero-extended stream the reference builds with its zeroed tail block
// (lookup_kernel.hpp:128-132) and all-zero initial prev vector (:115).
U8V_HD uint32_t u8v_mask_word(uint32_t w, int64_t pos, int64_t lo, int64_t hi) {
  uint32_t keep = 0;
  for (int k = 0; k < 4; ++k) {
    const int64_t q = pos + k;
    if (q >= lo && q < hi) keep |= 0xFFu << (8 * k);
  }
  return w & keep;
}
