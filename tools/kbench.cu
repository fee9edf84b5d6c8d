// tools/kbench.cu -- DEVELOPMENT HARNESS (not product code): times variants of
// the K1 inner loop (word formulation x occupancy x chunks-per-step) on the
// same device buffer, so formulation choices are made on measurements.
// Interior-only skeleton: n must be a multiple of 2 KiB and 32-byte aligned.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../paper_2010_03090_b200/csrc/utf8v_swar.h"
#include "../paper_2010_03090_b200/csrc/utf8v_bits.h"

namespace kb {

// Historical lag form (round-1 v0..v3; removed from utf8v_swar.h): the rare
// pair ending at each lane is tested at the follower's lane.
__device__ __forceinline__ uint32_t lag_rare_pairs(uint32_t w, uint32_t ph, uint32_t e1, u8v_consts k) {
  const uint32_t a = u8v_mad(w, k.m256, ph);
  const uint32_t a4 = a << 2;
  const uint32_t zl = (a4 & 0x7C7C7C7Cu) | (u8v_mulhi(w, k.mshr4) & 0x03030303u);
  return u8v_rare_key(a4, zl, e1, k);
}
__device__ __forceinline__ uint32_t u8v_word_errors_k(uint32_t w, u8v_carry* c, u8v_consts k) {
  const uint32_t s1 = w << 1, s2 = w << 2, s3 = w << 3;
  const uint32_t f1 = w & s1, f2 = f1 & s2, f3 = f2 & s3;
  const uint32_t e1 = u8v_fsl(c->f1, f1, 8), e2 = u8v_fsl(c->f2, f2, 16), e3 = u8v_fsl(c->f3, f3, 24);
  const uint32_t S = (e1 | e2 | e3) ^ (w & ~s1);
  const uint32_t R = lag_rare_pairs(w, c->ph, e1, k);
  c->p = w; c->f1 = f1; c->f2 = f2; c->f3 = f3; c->ph = u8v_mulhi(w, k.m256);
  return S | R;
}


struct Cfg {
  uint32_t one, m256, mshr4, m2_16, m2_24, m2_8;
};

__device__ __forceinline__ uint32_t mad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint64_t madw(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

struct Carry {
  uint32_t p, f1, f2, f3, ph, h1, h2, h3;
  uint64_t cin;
};

__device__ __forceinline__ Carry carry_of(uint32_t p) {
  Carry c;
  c.p = p;
  c.f1 = p & (p << 1);
  c.f2 = c.f1 & (p << 2);
  c.f3 = c.f2 & (p << 3);
  c.ph = p >> 24;
  c.h1 = c.f1 >> 24;
  c.h2 = c.f2 >> 16;
  c.h3 = c.f3 >> 8;
  const uint32_t g1 = c.f1 & 0x80808080u, g2 = c.f2 & 0x80808080u, g3 = c.f3 & 0x80808080u;
  c.cin = (uint64_t)((g1 >> 24) + (g2 >> 16) + (g3 >> 8));
  return c;
}

// R with the gate as a separate input (shared by all variants).
__device__ __forceinline__ uint32_t rare(uint32_t a4, uint32_t zl, uint32_t gate, const Cfg& k) {
  const uint32_t ge08 = mad(zl, k.one, 0x78787878u);
  const uint32_t ge02 = mad(zl, k.one, 0x7E7E7E7Eu);
  const uint32_t ge36 = mad(zl, k.one, 0x4A4A4A4Au);
  const uint32_t ge38 = mad(zl, k.one, 0x48484848u);
  const uint32_t ge40 = mad(zl, k.one, 0x40404040u);
  const uint32_t ge41 = mad(zl, k.one, 0x3F3F3F3Fu);
  const uint32_t ge51 = mad(zl, k.one, 0x2F2F2F2Fu);
  const uint32_t bad_ef = ~ge02 | (ge36 & ~ge38) | (ge40 & ~ge41) | ge51;
  return gate & ((a4 & bad_ef) | (~a4 & ~ge08));
}

// V0: production formula (utf8v_swar.h u8v_word_errors_k).
// V1: e-terms via IMAD (no SHF funnels).
// V2: e-sum via IMAD.WIDE chain on clean flags; R gated by a7&a6.
// V3: v1 all-ALU formula (for reference).
template <int V>
__device__ __forceinline__ uint32_t word(uint32_t w, Carry& c, const Cfg& k) {
  if (V == 0) {
    u8v_carry cc;
    cc.p = c.p; cc.f1 = c.f1; cc.f2 = c.f2; cc.f3 = c.f3; cc.ph = c.ph;
    u8v_consts kk;
    kk.one = k.one; kk.m256 = k.m256; kk.mshr4 = k.mshr4;
    const uint32_t e = u8v_word_errors_k(w, &cc, kk);
    c.p = cc.p; c.f1 = cc.f1; c.f2 = cc.f2; c.f3 = cc.f3; c.ph = cc.ph;
    return e;
  } else if (V == 1) {
    const uint32_t s1 = w << 1, s2 = w << 2, s3 = w << 3;
    const uint32_t f1 = w & s1, f2 = f1 & s2, f3 = f2 & s3;
    const uint32_t e1 = mad(f1, k.m256, c.h1);
    const uint32_t e2 = mad(f2, k.m2_16, c.h2);
    const uint32_t e3 = mad(f3, k.m2_24, c.h3);
    const uint32_t S = (e1 | e2 | e3) ^ (w & ~s1);
    const uint32_t a = mad(w, k.m256, c.ph);
    const uint32_t a4 = a << 2;
    const uint32_t zl = (a4 & 0x7C7C7C7Cu) | (mulhi(w, k.mshr4) & 0x03030303u);
    const uint32_t R = rare(a4, zl, e1, k);
    c.h1 = mulhi(f1, k.m256);
    c.h2 = mulhi(f2, k.m2_16);
    c.h3 = mulhi(f3, k.m2_24);
    c.ph = mulhi(w, k.m256);
    return S | R;
  } else if (V == 2) {
    const uint32_t s1 = w << 1, s2 = w << 2, s3 = w << 3;
    const uint32_t f1 = w & s1 & 0x80808080u, f2 = f1 & s2, f3 = f2 & s3;
    uint64_t x = madw(f3, k.m2_24, c.cin);
    x = madw(f2, k.m2_16, x);
    x = madw(f1, k.m256, x);
    const uint32_t E = (uint32_t)x;
    c.cin = x >> 32;
    const uint32_t S = E ^ (w & ~s1);
    const uint32_t a = mad(w, k.m256, c.ph);
    const uint32_t a2 = a << 1, a4 = a << 2;
    const uint32_t zl = (a4 & 0x7C7C7C7Cu) | (mulhi(w, k.mshr4) & 0x03030303u);
    const uint32_t R = rare(a4, zl, a & a2, k);
    c.ph = mulhi(w, k.m256);
    return S | R;
  } else {
    const uint32_t s1 = w << 1, s2 = w << 2, s3 = w << 3;
    const uint32_t f1 = w & s1, f2 = f1 & s2, f3 = f2 & s3;
    const uint32_t e1 = __funnelshift_l(c.f1, f1, 8);
    const uint32_t e2 = __funnelshift_l(c.f2, f2, 16);
    const uint32_t e3 = __funnelshift_l(c.f3, f3, 24);
    const uint32_t S = (e1 | e2 | e3) ^ (w & ~s1);
    const uint32_t a = __funnelshift_l(c.p, w, 8);
    const uint32_t zl = ((a & 0x1F1F1F1Fu) << 2) | ((w >> 4) & 0x03030303u);
    const uint32_t ge08 = zl + 0x78787878u, ge02 = zl + 0x7E7E7E7Eu, ge36 = zl + 0x4A4A4A4Au;
    const uint32_t ge38 = zl + 0x48484848u, ge40 = zl + 0x40404040u, ge41 = zl + 0x3F3F3F3Fu;
    const uint32_t ge51 = zl + 0x2F2F2F2Fu;
    const uint32_t age = __funnelshift_l(c.f2, f2, 8);
    const uint32_t bad_ef = ~ge02 | (ge36 & ~ge38) | (ge40 & ~ge41) | ge51;
    const uint32_t R = (age & bad_ef) | (e1 & ~age & ~ge08);
    c.p = w; c.f1 = f1; c.f2 = f2; c.f3 = f3;
    return S | R;
  }
}

// V30: the reference's own formulation (classify with the three 16-entry
// nibble tables T1[prev1 >> 4] & T2[prev1 & 15] & T3[cur >> 4], then the
// 2/3/4-byte continuation cross-check, proj/include/utf8v/lookup_kernel.hpp:
// 21-46, tables proj/include/utf8v/tables.hpp:60-99) in 32-bit SWAR: each
// 16-entry lookup is two PRMTs over the table's four words and a select by
// the nibble's bit 3.  The north_star's suggested formulation, kept here as
// the measured comparison for DESIGN.md §2 ("nibble tables" deviation).
__device__ __forceinline__ uint32_t nib_sel(uint32_t nib) {  // byte-lane nibbles -> PRMT selector
  uint32_t x = nib & 0x07070707u;
  x = (x | (x >> 4)) & 0x00770077u;
  return (x | (x >> 8)) & 0x00007777u;
}
__device__ __forceinline__ uint32_t lookup16(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t t3, uint32_t nib) {
  const uint32_t sel = nib_sel(nib);
  const uint32_t lo = __byte_perm(t0, t1, sel), hi = __byte_perm(t2, t3, sel);
  const uint32_t m = ((nib >> 3) & 0x01010101u) * 0xFFu;
  return (hi & m) | (lo & ~m);
}
__device__ __forceinline__ uint32_t word_nib(uint32_t w, Carry& c) {
  const uint32_t prev1 = __funnelshift_l(c.p, w, 8), prev2 = __funnelshift_l(c.p, w, 16);
  const uint32_t prev3 = __funnelshift_l(c.p, w, 24);
  const uint32_t c1 = lookup16(0x02020202u, 0x02020202u, 0x80808080u, 0x49150121u, (prev1 >> 4) & 0x0F0F0F0Fu);
  const uint32_t c2 = lookup16(0x8383A3E7u, 0xCBCBCB8Bu, 0xCBCBCBCBu, 0xCBCBDBCBu, prev1 & 0x0F0F0F0Fu);
  const uint32_t c3 = lookup16(0x01010101u, 0x01010101u, 0xBABAAEE6u, 0x01010101u, (w >> 4) & 0x0F0F0F0Fu);
  const uint32_t cls = c1 & c2 & c3;
  // bit 7 of each byte: prev2 >= E0 | prev3 >= F0
  const uint32_t e2 = prev2 & (prev2 << 1) & (prev2 << 2);
  const uint32_t e3 = prev3 & (prev3 << 1) & (prev3 << 2) & (prev3 << 3);
  const uint32_t err = ((e2 | e3) & 0x80808080u) ^ cls;
  c.p = w;
  return (((err & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | err) & 0x80808080u;  // any bit of a byte -> its bit 7
}

// V4: R evaluated at the lead's own lane: key from w (s2 = w<<2 gives a5..a0)
// and the next byte's bits 5,4 via a right funnel with the next word.
__device__ __forceinline__ uint32_t word4(uint32_t w, uint32_t wn, Carry& c, const Cfg& k) {
  const uint32_t s1 = w << 1, s2 = w << 2, s3 = w << 3;
  const uint32_t f1 = w & s1, f2 = f1 & s2, f3 = f2 & s3;
  const uint32_t e1 = __funnelshift_l(c.f1, f1, 8);
  const uint32_t e2 = __funnelshift_l(c.f2, f2, 16);
  const uint32_t e3 = __funnelshift_l(c.f3, f3, 24);
  const uint32_t S = (e1 | e2 | e3) ^ (w & ~s1);
  const uint32_t t = __funnelshift_r(w, wn, 12);
  const uint32_t zl = (s2 & 0x7C7C7C7Cu) | (t & 0x03030303u);
  const uint32_t R = rare(s2, zl, f1, k);
  c.f1 = f1; c.f2 = f2; c.f3 = f3;
  return S | R;
}

// V5: V4 with the e1 funnel and the next-byte funnel on the FMA pipe.
__device__ __forceinline__ uint32_t word5(uint32_t w, uint32_t wn, Carry& c, const Cfg& k) {
  const uint32_t s1 = w << 1, s2 = w << 2, s3 = w << 3;
  const uint32_t f1 = w & s1, f2 = f1 & s2, f3 = f2 & s3;
  const uint32_t e1 = mad(f1, k.m256, c.h1);                 // f1<<8 | prev f1>>24
  const uint32_t e2 = __funnelshift_l(c.f2, f2, 16);
  const uint32_t e3 = __funnelshift_l(c.f3, f3, 24);
  const uint32_t S = (e1 | e2 | e3) ^ (w & ~s1);
  const uint32_t t = mad(wn, 1u << 20, mulhi(w, 1u << 20));  // (wn:w) >> 12
  const uint32_t zl = (s2 & 0x7C7C7C7Cu) | (t & 0x03030303u);
  const uint32_t R = rare(s2, zl, f1, k);
  c.f2 = f2; c.f3 = f3;
  c.h1 = mulhi(f1, k.m256);
  return S | R;
}

// V6: V4 with the lead flags from threshold adds on the FMA pipe:
// g1/g2/g3 = bit 7 of ((w >> 1) & 0x7F..) + 0x20/0x10/0x08 (a >= C0/E0/F0).
__device__ __forceinline__ uint32_t word6(uint32_t w, uint32_t wn, Carry& c, const Cfg& k) {
  const uint32_t s1 = mad(w, k.one, w), s2 = w << 2;
  const uint32_t hm = mulhi(w, 0x80000000u) & 0x7F7F7F7Fu;
  const uint32_t g1 = mad(hm, k.one, 0x20202020u);
  const uint32_t g2 = mad(hm, k.one, 0x10101010u);
  const uint32_t g3 = mad(hm, k.one, 0x08080808u);
  const uint32_t e1 = __funnelshift_l(c.f1, g1, 8);
  const uint32_t e2 = __funnelshift_l(c.f2, g2, 16);
  const uint32_t e3 = __funnelshift_l(c.f3, g3, 24);
  const uint32_t S = (e1 | e2 | e3) ^ (w & ~s1);
  const uint32_t t = __funnelshift_r(w, wn, 12);
  const uint32_t zl = (s2 & 0x7C7C7C7Cu) | (t & 0x03030303u);
  const uint32_t R = rare(s2, zl, g1, k);
  c.f1 = g1; c.f2 = g2; c.f3 = g3;
  return S | R;
}

// V7: V6 with s2 from IMAD and the key mask as one bitselect + clear.
__device__ __forceinline__ uint32_t word7(uint32_t w, uint32_t wn, Carry& c, const Cfg& k) {
  const uint32_t s1 = mad(w, k.one, w), s2 = mad(w, 4u * k.one, 0u);
  const uint32_t hm = mulhi(w, 0x80000000u) & 0x7F7F7F7Fu;
  const uint32_t g1 = mad(hm, k.one, 0x20202020u);
  const uint32_t g2 = mad(hm, k.one, 0x10101010u);
  const uint32_t g3 = mad(hm, k.one, 0x08080808u);
  const uint32_t e1 = __funnelshift_l(c.f1, g1, 8);
  const uint32_t e2 = __funnelshift_l(c.f2, g2, 16);
  const uint32_t e3 = __funnelshift_l(c.f3, g3, 24);
  const uint32_t S = (e1 | e2 | e3) ^ (w & ~s1);
  const uint32_t t = mad(wn, 1u << 20, mulhi(w, 1u << 20));
  const uint32_t zl = (s2 & 0x7C7C7C7Cu) | (t & 0x03030303u);
  const uint32_t R = rare(s2, zl, g1, k);
  c.f1 = g1; c.f2 = g2; c.f3 = g3;
  return S | R;
}

// V9: bit-sliced with the transpose's shifts as IMAD / IMAD.HI (FMA pipe).
__device__ __forceinline__ void t8x8_fma(uint32_t& a, uint32_t& b, const Cfg& k) {
  uint32_t t;
  t = (a ^ mulhi(a, 1u << 25)) & 0x00AA00AAu;
  a ^= t ^ mad(t, 128u * k.one, 0u);
  t = (b ^ mulhi(b, 1u << 25)) & 0x00AA00AAu;
  b ^= t ^ mad(t, 128u * k.one, 0u);
  t = (a ^ mulhi(a, 1u << 18)) & 0x0000CCCCu;
  a ^= t ^ mad(t, 16384u * k.one, 0u);
  t = (b ^ mulhi(b, 1u << 18)) & 0x0000CCCCu;
  b ^= t ^ mad(t, 16384u * k.one, 0u);
  t = (a ^ mad(b, 16u * k.one, 0u)) & 0xF0F0F0F0u;
  a ^= t;
  b ^= mulhi(t, 1u << 28);
}
__device__ __forceinline__ uint32_t planes_fma(const uint32_t (&w)[8], uint32_t prev, uint32_t next,
                                               const Cfg& k) {
  uint32_t l0 = w[0], h0 = w[1], l1 = w[2], h1 = w[3], l2 = w[4], h2 = w[5], l3 = w[6], h3 = w[7];
  t8x8_fma(l0, h0, k);
  t8x8_fma(l1, h1, k);
  t8x8_fma(l2, h2, k);
  t8x8_fma(l3, h3, k);
  uint32_t p[8];
  uint32_t A = __byte_perm(l0, l1, 0x5140), B = __byte_perm(l0, l1, 0x7362);
  uint32_t C = __byte_perm(l2, l3, 0x5140), D = __byte_perm(l2, l3, 0x7362);
  p[0] = __byte_perm(A, C, 0x5410); p[1] = __byte_perm(A, C, 0x7632);
  p[2] = __byte_perm(B, D, 0x5410); p[3] = __byte_perm(B, D, 0x7632);
  A = __byte_perm(h0, h1, 0x5140); B = __byte_perm(h0, h1, 0x7362);
  C = __byte_perm(h2, h3, 0x5140); D = __byte_perm(h2, h3, 0x7362);
  p[4] = __byte_perm(A, C, 0x5410); p[5] = __byte_perm(A, C, 0x7632);
  p[6] = __byte_perm(B, D, 0x5410); p[7] = __byte_perm(B, D, 0x7632);
  const uint32_t l1f = p[7] & p[6], l2f = l1f & p[5], l3f = l2f & p[4];
  const uint32_t q1 = prev & mad(prev, 2u * k.one, 0u);
  const uint32_t q2 = q1 & mad(prev, 4u * k.one, 0u);
  const uint32_t q3 = q2 & mad(prev, 8u * k.one, 0u);
  const uint32_t e1 = __funnelshift_l(mad(q1 & 0x80808080u, 0x00204081u * k.one, 0u), l1f, 1);
  const uint32_t e2 = __funnelshift_l(mad(q2 & 0x80808080u, 0x00204081u * k.one, 0u), l2f, 2);
  const uint32_t e3 = __funnelshift_l(mad(q3 & 0x80808080u, 0x00204081u * k.one, 0u), l3f, 3);
  const uint32_t S = (p[7] & ~p[6]) ^ (e1 | e2 | e3);
  const uint32_t n5 = __funnelshift_r(p[5], next >> 5, 1);
  const uint32_t n4 = __funnelshift_r(p[4], next >> 4, 1);
  const uint32_t z321 = ~(p[3] | p[2] | p[1]);
  const uint32_t rc = l1f & ~p[5] & ~p[4] & z321;
  const uint32_t ee = l2f & ~p[4];
  const uint32_t re0 = ee & z321 & ~p[0] & ~n5;
  const uint32_t red = ee & p[3] & p[2] & ~p[1] & p[0] & n5;
  const uint32_t rf0 = l3f & z321 & ~p[0] & ~n5 & ~n4;
  const uint32_t rf4 = l3f & ~p[3] & p[2] & ~p[1] & ~p[0] & (n5 | n4);
  const uint32_t rf5 = l3f & (p[3] | (p[2] & (p[1] | p[0])));
  return S | rc | re0 | red | rf0 | rf4 | rf5;
}

template <int V, int U, int PF = 0>
__device__ __forceinline__ void body(const uint8_t* base, int64_t steps, int64_t spw, uint32_t* flag,
                                     const Cfg& k) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t step = warp * spw;
  int64_t se = step + spw < steps ? step + spw : steps;
  if (step >= se) return;
  uint32_t carry_word = 0;
  uint32_t acc = 0;
  for (; step < se; ++step) {
    const uint8_t* sp = base + step * (int64_t)(U * 1024);
    if (PF > 0 && lane == 0 && step + PF < se)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sp + PF * (int64_t)(U * 1024)),
                   "r"(U * 1024)
                   : "memory");
    uint32_t v[U][8];
#pragma unroll
    for (int i = 0; i < U; ++i)
      asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
          : "=r"(v[i][0]), "=r"(v[i][1]), "=r"(v[i][2]), "=r"(v[i][3]), "=r"(v[i][4]),
            "=r"(v[i][5]), "=r"(v[i][6]), "=r"(v[i][7])
          : "l"(sp + (lane + 32 * i) * 32));
    bool step_ascii = false;
    if (V == 11) {
      uint32_t hb = 0;
#pragma unroll
      for (int i = 0; i < U; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) hb |= v[i][j];
      step_ascii = __all_sync(0xFFFFFFFFu, (hb & 0x80808080u) == 0);
    }
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t supply = lane == 31 ? (i == 0 ? carry_word : v[i - 1][7]) : v[i][7];
      const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
      Carry c = carry_of(prev);
      uint32_t e = 0;
      if (V == 4) {
        const uint32_t nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
#pragma unroll
        for (int j = 0; j < 8; ++j) e |= word4(v[i][j], j < 7 ? v[i][j + 1] : nextw, c, k);
      } else if (V == 5) {
        const uint32_t nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
#pragma unroll
        for (int j = 0; j < 8; ++j) e |= word5(v[i][j], j < 7 ? v[i][j + 1] : nextw, c, k);
      } else if (V == 11 || V == 12) {
        const uint32_t nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
        bool asc = step_ascii;
        if (V == 12) {
          uint32_t hb = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) hb |= v[i][j];
          asc = __all_sync(0xFFFFFFFFu, (hb & 0x80808080u) == 0);
        }
        if (asc) {
          u8v_carry cr = u8v_carry_of(prev);
          e = u8v_ascii_word_errors(v[i][0], &cr) & 0x80808080u;
        } else {
          u8v_consts kk;
          kk.one = k.one; kk.m256 = k.m256; kk.mshr4 = k.mshr4;
          { uint32_t h7; e = u8v_chunk_errors_planes_k(v[i], prev, nextw, kk, &h7); }
        }
      } else if (V == 10) {
        const uint32_t nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
        u8v_consts kk;
        kk.one = k.one; kk.m256 = k.m256; kk.mshr4 = k.mshr4;
        { uint32_t h7; e = u8v_chunk_errors_planes_k(v[i], prev, nextw, kk, &h7); }
      } else if (V == 9) {
        const uint32_t nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
        e = planes_fma(v[i], prev, nextw, k);
      } else if (V == 8) {
        const uint32_t nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
        e = u8v_chunk_errors_planes(v[i], prev, nextw);
      } else if (V == 6) {
        const uint32_t nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
#pragma unroll
        for (int j = 0; j < 8; ++j) e |= word6(v[i][j], j < 7 ? v[i][j + 1] : nextw, c, k);
      } else if (V == 30) {
#pragma unroll
        for (int j = 0; j < 8; ++j) e |= word_nib(v[i][j], c);
      } else if (V == 7) {
        const uint32_t nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
#pragma unroll
        for (int j = 0; j < 8; ++j) e |= word7(v[i][j], j < 7 ? v[i][j + 1] : nextw, c, k);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) e |= word<V>(v[i][j], c, k);
      }
      acc |= e;
    }
    if (lane == 31) carry_word = v[U - 1][7];
  }
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, V >= 8 ? acc : (acc & 0x80808080u));
  if (lane == 0 && any) atomicOr(flag, 1u);
}

// Register double buffering: step s+1's chunks are loaded before step s is
// evaluated (V6 word formula).
template <int U>
__device__ __forceinline__ void load_step(uint32_t (&v)[U][8], const uint8_t* sp, int lane) {
#pragma unroll
  for (int i = 0; i < U; ++i)
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[i][0]), "=r"(v[i][1]), "=r"(v[i][2]), "=r"(v[i][3]), "=r"(v[i][4]),
                   "=r"(v[i][5]), "=r"(v[i][6]), "=r"(v[i][7])
                 : "l"(sp + (lane + 32 * i) * 32));
}

template <int U>
__device__ __forceinline__ uint32_t eval_step(const uint32_t (&v)[U][8], uint32_t& carry_word, int lane,
                                              const Cfg& k) {
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < U; ++i) {
    const uint32_t supply = lane == 31 ? (i == 0 ? carry_word : v[i - 1][7]) : v[i][7];
    const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
    Carry c = carry_of(prev);
    const uint32_t nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
    uint32_t e = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) e |= word6(v[i][j], j < 7 ? v[i][j + 1] : nextw, c, k);
    acc |= e;
  }
  if (lane == 31) carry_word = v[U - 1][7];
  return acc;
}

template <int U>
__device__ __forceinline__ void body_db(const uint8_t* base, int64_t steps, int64_t spw, uint32_t* flag,
                                        const Cfg& k) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t step = warp * spw;
  const int64_t se = step + spw < steps ? step + spw : steps;
  if (step >= se) return;
  uint32_t carry_word = 0, acc = 0;
  uint32_t a[U][8], b[U][8];
  load_step<U>(a, base + step * (int64_t)(U * 1024), lane);
  for (; step + 1 < se; step += 2) {
    load_step<U>(b, base + (step + 1) * (int64_t)(U * 1024), lane);
    acc |= eval_step<U>(a, carry_word, lane, k);
    if (step + 2 < se) load_step<U>(a, base + (step + 2) * (int64_t)(U * 1024), lane);
    acc |= eval_step<U>(b, carry_word, lane, k);
  }
  if (step < se) acc |= eval_step<U>(a, carry_word, lane, k);
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc & 0x80808080u);
  if (lane == 0 && any) atomicOr(flag, 1u);
}

#define KB_KERNEL_DB(U, MINB)                                                                   \
  __global__ void __launch_bounds__(256, MINB)                                                 \
      k_db_u##U##_b##MINB(const uint8_t* base, int64_t steps, int64_t spw, uint32_t* flag, Cfg k) { \
    body_db<U>(base, steps, spw, flag, k);                                                     \
  }
KB_KERNEL_DB(2, 3)
KB_KERNEL_DB(1, 4)
KB_KERNEL_DB(2, 2)
KB_KERNEL_DB(4, 2)

// V13: ASCII vote only when the previous step was all-ASCII; the plane path
// reports ASCII-ness from plane 7 after the fact.
template <int U, int NSW = 0, int PF = 0>
__device__ __forceinline__ void body13(const uint8_t* base, int64_t steps, int64_t spw, uint32_t* flag,
                                       const Cfg& k) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t step = warp * spw;
  const int64_t se = step + spw < steps ? step + spw : steps;
  if (step >= se) return;
  u8v_consts kk;
  kk.one = k.one; kk.m256 = k.m256; kk.mshr4 = k.mshr4;
  uint32_t carry_word = 0, acc = 0;
  bool was_ascii = false;
  uint32_t nsw_ahead = 0;
  if (NSW == 2 && lane == 0 && step + 1 < steps) nsw_ahead = __ldg(reinterpret_cast<const uint32_t*>(base + (step + 1) * (int64_t)(U * 1024)));
  for (; step < se; ++step) {
    const uint8_t* sp = base + step * (int64_t)(U * 1024);
    if (PF > 0 && lane == 0 && step + PF < se)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sp + PF * (int64_t)(U * 1024)),
                   "r"(U * 1024)
                   : "memory");
    uint32_t nsw = 0;
    if (NSW == 1 && lane == 0 && step + 1 < steps) nsw = __ldg(reinterpret_cast<const uint32_t*>(sp + U * 1024));
    if (NSW == 2) {
      nsw = nsw_ahead;
      if (lane == 0 && step + 2 < steps) nsw_ahead = __ldg(reinterpret_cast<const uint32_t*>(sp + 2 * U * 1024));
    }
    uint32_t v[U][8];
    uint32_t ex[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
          : "=r"(v[i][0]), "=r"(v[i][1]), "=r"(v[i][2]), "=r"(v[i][3]), "=r"(v[i][4]),
            "=r"(v[i][5]), "=r"(v[i][6]), "=r"(v[i][7])
          : "l"(sp + (lane + 32 * i) * 32));
      ex[i] = 0;
      if (NSW == 3 && lane == 31 && (i + 1 < U || step + 1 < steps))
        ex[i] = __ldg(reinterpret_cast<const uint32_t*>(sp + (lane + 32 * i) * 32 + 32));
    }
    bool asc = false;
    if (was_ascii) {
      uint32_t hb = 0;
#pragma unroll
      for (int i = 0; i < U; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) hb |= v[i][j];
      asc = __all_sync(0xFFFFFFFFu, (hb & 0x80808080u) == 0);
    }
    if (asc) {
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const uint32_t supply = lane == 31 ? (i == 0 ? carry_word : v[i - 1][7]) : v[i][7];
        const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
        u8v_carry cr = u8v_carry_of(prev);
        acc |= u8v_ascii_word_errors(v[i][0], &cr) & 0x80808080u;
      }
    } else {
      uint32_t h7 = 0;
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const uint32_t supply = lane == 31 ? (i == 0 ? carry_word : v[i - 1][7]) : v[i][7];
        const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
        uint32_t nextw;
        if (NSW == 0) {
          nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
        } else if (NSW == 3) {
          nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
          if (lane == 31) nextw = ex[i];
        } else {
          const uint32_t dn = lane == 0 ? (i + 1 < U ? v[i + 1][0] : nsw) : v[i][0];
          nextw = __shfl_sync(0xFFFFFFFFu, dn, (lane + 1) & 31);
        }
        uint32_t hi;
        acc |= u8v_chunk_errors_planes_k(v[i], prev, nextw, kk, &hi);
        h7 |= hi;
      }
      asc = __all_sync(0xFFFFFFFFu, h7 == 0);
    }
    was_ascii = asc;
    if (lane == 31) carry_word = v[U - 1][7];
  }
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc);
  if (lane == 0 && any) atomicOr(flag, 1u);
}
#define KB_KERNEL13(U, MINB)                                                                     \
  __global__ void __launch_bounds__(256, MINB)                                                 \
      k_v13_u##U##_b##MINB(const uint8_t* base, int64_t steps, int64_t spw, uint32_t* flag, Cfg k) { \
    body13<U>(base, steps, spw, flag, k);                                                      \
  }
KB_KERNEL13(4, 4)
__global__ void __launch_bounds__(256, 4) k_v14_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  body13<4, 1>(base, steps, spw, flag, k);
}
__global__ void __launch_bounds__(256, 4) k_v16_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  body13<4, 3>(base, steps, spw, flag, k);
}
__global__ void __launch_bounds__(256, 4) k_p1_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                     uint32_t* flag, Cfg k) {
  body13<4, 3, 1>(base, steps, spw, flag, k);
}
__global__ void __launch_bounds__(256, 4) k_p2_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                     uint32_t* flag, Cfg k) {
  body13<4, 3, 2>(base, steps, spw, flag, k);
}
__global__ void __launch_bounds__(256, 4) k_p4_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                     uint32_t* flag, Cfg k) {
  body13<4, 3, 4>(base, steps, spw, flag, k);
}
__global__ void __launch_bounds__(256, 4) k_v15_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  body13<4, 2>(base, steps, spw, flag, k);
}

// V17: per-warp TMA ring.  Lane 0 streams steps into shared memory with
// cp.async.bulk (completion on one mbarrier per stage), S stages ahead; the
// warp computes from shared memory.  In-flight data costs no registers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void ld_shared_chunk(uint32_t (&w)[8], const uint8_t* p) {
  const uint32_t a = smem_u32(p);
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(a));
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]) : "r"(a + 16));
}

template <int U, int S>
__device__ __forceinline__ void body_tma(const uint8_t* base, int64_t steps, int64_t spw, uint32_t* flag,
                                         const Cfg& k) {
  constexpr int STEP = U * 1024;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint8_t* ring = smem + wib * S * STEP;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (blockDim.x >> 5) * S * STEP) + wib * S;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t step = warp * spw;
  const int64_t se = step + spw < steps ? step + spw : steps;
  if (step >= se) return;
  u8v_consts kk;
  kk.one = k.one; kk.m256 = k.m256; kk.mshr4 = k.mshr4;
  if (lane == 0) {
    for (int j = 0; j < S; ++j) mb_init(bars + j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int j = 0; j < S; ++j)
      if (step + j < se) {
        mb_expect_tx(bars + j, STEP);
        tma_load(ring + j * STEP, base + (step + j) * (int64_t)STEP, STEP, bars + j);
      }
  }
  __syncwarp();
  uint32_t carry_word = 0, acc = 0, phase = 0;
  bool was_ascii = false;
  for (int it = 0; step < se; ++step, ++it) {
    const int st = it % S;
    mb_wait(bars + st, (phase >> st) & 1);
    phase ^= 1u << st;
    const uint8_t* sb = ring + st * STEP;
    uint32_t v[U][8];
#pragma unroll
    for (int i = 0; i < U; ++i) ld_shared_chunk(v[i], sb + (i * 32 + lane) * 32);
    // Next step's first word (lookahead of the step's last lane).
    uint32_t nsw = 0;
    if (step + 1 < se) {
      const int sn = (it + 1) % S;
      mb_wait(bars + sn, (phase >> sn) & 1);
      if (lane == 0) nsw = *reinterpret_cast<const uint32_t*>(ring + sn * STEP);
    } else if (lane == 0 && step + 1 < steps) {
      nsw = __ldg(reinterpret_cast<const uint32_t*>(base + (step + 1) * (int64_t)STEP));
    }
    bool asc = false;
    if (was_ascii) {
      uint32_t hb = 0;
#pragma unroll
      for (int i = 0; i < U; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) hb |= v[i][j];
      asc = __all_sync(0xFFFFFFFFu, (hb & 0x80808080u) == 0);
    }
    if (asc) {
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const uint32_t supply = lane == 31 ? (i == 0 ? carry_word : v[i - 1][7]) : v[i][7];
        const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
        u8v_carry cr = u8v_carry_of(prev);
        acc |= u8v_ascii_word_errors(v[i][0], &cr) & 0x80808080u;
      }
    } else {
      uint32_t h7 = 0;
#pragma unroll
      for (int i = 0; i < U; ++i) {
        const uint32_t supply = lane == 31 ? (i == 0 ? carry_word : v[i - 1][7]) : v[i][7];
        const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
        const uint32_t dn = lane == 0 ? (i + 1 < U ? v[i + 1][0] : nsw) : v[i][0];
        const uint32_t nextw = __shfl_sync(0xFFFFFFFFu, dn, (lane + 1) & 31);
        uint32_t hi;
        acc |= u8v_chunk_errors_planes_k(v[i], prev, nextw, kk, &hi);
        h7 |= hi;
      }
      asc = __all_sync(0xFFFFFFFFu, h7 == 0);
    }
    was_ascii = asc;
    if (lane == 31) carry_word = v[U - 1][7];
    // Stage st is consumed (values in registers): refill it S steps ahead.
    __syncwarp();
    if (lane == 0 && step + S < se) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mb_expect_tx(bars + st, STEP);
      tma_load(ring + st * STEP, base + (step + S) * (int64_t)STEP, STEP, bars + st);
    }
  }
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc);
  if (lane == 0 && any) atomicOr(flag, 1u);
}
#define KB_KERNEL_TMA(U, S, MINB)                                                                \
  __global__ void __launch_bounds__(256, MINB)                                                 \
      k_tma_u##U##_s##S##_b##MINB(const uint8_t* base, int64_t steps, int64_t spw, uint32_t* flag, \
                                  Cfg k) {                                                     \
    body_tma<U, S>(base, steps, spw, flag, k);                                                 \
  }
KB_KERNEL_TMA(2, 3, 4)
KB_KERNEL_TMA(2, 4, 3)
KB_KERNEL_TMA(4, 2, 3)
KB_KERNEL_TMA(4, 3, 2)
KB_KERNEL_TMA(1, 6, 4)

// V25: V17's per-warp TMA ring with the production permuted plane form, no
// ASCII path, and bank-conflict-free shared reads: lane L reads half
// (L >> 2) & 1 of its 32-byte chunk first, so each quarter-warp's 16-byte
// reads hit 8 distinct 4-bank groups.
__device__ __forceinline__ void ld_shared_chunk_swz(uint32_t (&w)[8], const uint8_t* p, int lane) {
  const uint32_t a = smem_u32(p);
  const uint32_t h = ((lane >> 2) & 1) * 16u;
  uint32_t x[8];
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]) : "r"(a + h));
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]) : "r"(a + (16u - h)));
  const bool sw = h != 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    w[j] = sw ? x[4 + j] : x[j];
    w[4 + j] = sw ? x[j] : x[4 + j];
  }
}

template <int U, int S>
__device__ __forceinline__ void body25(const uint8_t* base, int64_t steps, int64_t spw, uint32_t* flag,
                                       const Cfg& k) {
  constexpr int STEP = U * 1024;
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint8_t* ring = smem + wib * S * STEP;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (blockDim.x >> 5) * S * STEP) + wib * S;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t step = warp * spw;
  const int64_t se = step + spw < steps ? step + spw : steps;
  if (step >= se) return;
  u8v_consts kk;
  kk.one = k.one; kk.m256 = k.m256; kk.mshr4 = k.mshr4;
  if (lane == 0) {
    for (int j = 0; j < S; ++j) mb_init(bars + j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int j = 0; j < S; ++j)
      if (step + j < se) {
        mb_expect_tx(bars + j, STEP);
        tma_load(ring + j * STEP, base + (step + j) * (int64_t)STEP, STEP, bars + j);
      }
  }
  __syncwarp();
  uint32_t carry_word = 0, acc = 0, phase = 0;
  if (lane == 31 && step > 0) carry_word = __ldg(reinterpret_cast<const uint32_t*>(base + step * (int64_t)STEP - 4));
  for (int it = 0; step < se; ++step, ++it) {
    const int st = it % S;
    mb_wait(bars + st, (phase >> st) & 1);
    phase ^= 1u << st;
    const uint8_t* sb = ring + st * STEP;
    uint32_t v[U][8];
#pragma unroll
    for (int i = 0; i < U; ++i) ld_shared_chunk_swz(v[i], sb + (i * 32 + lane) * 32, lane);
    uint32_t nsw = 0;
    if (lane == 0 && step + 1 < steps) nsw = __ldg(reinterpret_cast<const uint32_t*>(base + (step + 1) * (int64_t)STEP));
    // Stage st is in registers: refill it S steps ahead before computing.
    __syncwarp();
    if (lane == 0 && step + S < se) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mb_expect_tx(bars + st, STEP);
      tma_load(ring + st * STEP, base + (step + S) * (int64_t)STEP, STEP, bars + st);
    }
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t supply = lane == 31 ? (i == 0 ? carry_word : v[i - 1][7]) : v[i][7];
      const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
      const uint32_t dn = lane == 0 ? (i + 1 < U ? v[i + 1][0] : nsw) : v[i][0];
      const uint32_t nextw = __shfl_sync(0xFFFFFFFFu, dn, (lane + 1) & 31);
      uint32_t hi;
      acc |= u8v_chunk_errors_planes_perm_k(v[i], prev, nextw, kk, &hi);
    }
    if (lane == 31) carry_word = v[U - 1][7];
  }
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc);
  if (lane == 0 && any) atomicOr(flag, 1u);
}
#define KB_KERNEL25(U, S, MINB)                                                                  \
  __global__ void __launch_bounds__(256, MINB)                                                 \
      k_v25_u##U##_s##S##_b##MINB(const uint8_t* base, int64_t steps, int64_t spw, uint32_t* flag, \
                                  Cfg k) {                                                     \
    body25<U, S>(base, steps, spw, flag, k);                                                   \
  }
KB_KERNEL25(4, 3, 2)
KB_KERNEL25(4, 2, 3)
KB_KERNEL25(2, 3, 4)
KB_KERNEL25(2, 2, 4)
KB_KERNEL25(4, 4, 1)

// V18: rolling reload.  Each chunk slot is refilled with the next step's
// chunk right after it is consumed, so every load overlaps ~3/4 of a step of
// compute, with no extra registers.
__device__ __forceinline__ void ldg_chunk(uint32_t (&w)[8], const uint8_t* p) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
                 "=r"(w[7])
               : "l"(p));
}
template <int U>
__device__ __forceinline__ void body18(const uint8_t* base, int64_t steps, int64_t spw, uint32_t* flag,
                                       const Cfg& k) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t step = warp * spw;
  const int64_t se = step + spw < steps ? step + spw : steps;
  if (step >= se) return;
  u8v_consts kk;
  kk.one = k.one; kk.m256 = k.m256; kk.mshr4 = k.mshr4;
  uint32_t v[U][8];
  const uint8_t* p = base + step * (int64_t)(U * 1024) + lane * 32;
#pragma unroll
  for (int i = 0; i < U; ++i) ldg_chunk(v[i], p + i * 1024);
  uint32_t carry_word = 0, acc = 0;
  for (; step < se; ++step, p += U * 1024) {
    const bool more = step + 1 < se;
    uint32_t h7 = 0;
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t supply = lane == 31 ? carry_word : v[i][7];
      const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
      // Lane 0's next chunk (slot i+1 of this step, or slot 0 already holding
      // the next step's first chunk).
      const uint32_t dn = lane == 0 ? (i + 1 < U ? v[i + 1][0] : v[0][0]) : v[i][0];
      const uint32_t nextw = __shfl_sync(0xFFFFFFFFu, dn, (lane + 1) & 31);
      uint32_t hi;
      acc |= u8v_chunk_errors_planes_k(v[i], prev, nextw, kk, &hi);
      h7 |= hi;
      carry_word = v[i][7];  // lane 31's value feeds lane 0 of the next chunk
      if (more) ldg_chunk(v[i], p + U * 1024 + i * 1024);
    }
    (void)h7;
  }
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc);
  if (lane == 0 && any) atomicOr(flag, 1u);
}
__global__ void __launch_bounds__(256, 4) k_v18_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  body18<4>(base, steps, spw, flag, k);
}
__global__ void __launch_bounds__(256, 3) k_v18_u4_b3(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  body18<4>(base, steps, spw, flag, k);
}
__global__ void __launch_bounds__(256, 4) k_v18_u2_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  body18<2>(base, steps, spw, flag, k);
}

// V19: grid-stride step assignment (all warps sweep one moving window of
// memory, for DRAM page locality); the halo word and the lookahead word are
// loaded per step (their neighbours belong to other warps).
template <int U>
__device__ __forceinline__ void body19(const uint8_t* base, int64_t steps, uint32_t* flag, const Cfg& k) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  u8v_consts kk;
  kk.one = k.one; kk.m256 = k.m256; kk.mshr4 = k.mshr4;
  uint32_t acc = 0;
  for (int64_t step = warp; step < steps; step += nwarps) {
    const uint8_t* sp = base + step * (int64_t)(U * 1024);
    uint32_t v[U][8];
#pragma unroll
    for (int i = 0; i < U; ++i) ldg_chunk(v[i], sp + (lane + 32 * i) * 32);
    uint32_t carry_word = 0, nsw = 0;
    if (lane == 31 && step > 0) carry_word = __ldg(reinterpret_cast<const uint32_t*>(sp - 4));
    if (lane == 0 && step + 1 < steps) nsw = __ldg(reinterpret_cast<const uint32_t*>(sp + U * 1024));
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t supply = lane == 31 ? (i == 0 ? carry_word : v[i - 1][7]) : v[i][7];
      const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
      const uint32_t dn = lane == 0 ? (i + 1 < U ? v[i + 1][0] : nsw) : v[i][0];
      const uint32_t nextw = __shfl_sync(0xFFFFFFFFu, dn, (lane + 1) & 31);
      uint32_t hi;
      acc |= u8v_chunk_errors_planes_k(v[i], prev, nextw, kk, &hi);
    }
  }
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc);
  if (lane == 0 && any) atomicOr(flag, 1u);
}
__global__ void __launch_bounds__(256, 4) k_v19_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  (void)spw;
  body19<4>(base, steps, flag, k);
}
__global__ void __launch_bounds__(256, 4) k_v19_u2_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  (void)spw;
  body19<2>(base, steps, flag, k);
}

// V20: V19 (grid-stride) with lane 31's follower words (the first word of
// lane 0's next chunk, and of the next step) and its halo word fetched one
// step ahead, so no chunk waits on another chunk's load.
template <int U>
__device__ __forceinline__ void body20(const uint8_t* base, int64_t steps, uint32_t* flag, const Cfg& k) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  u8v_consts kk;
  kk.one = k.one; kk.m256 = k.m256; kk.mshr4 = k.mshr4;
  uint32_t acc = 0;
  uint32_t fw[U], hw = 0;  // follower words and halo word of the current step (lane 31)
  auto fetch = [&](int64_t st, uint32_t (&f)[U], uint32_t& h) {
    const uint8_t* sp = base + st * (int64_t)(U * 1024);
#pragma unroll
    for (int i = 0; i < U; ++i)
      f[i] = (i + 1 < U || st + 1 < steps) ? __ldg(reinterpret_cast<const uint32_t*>(sp + (i + 1) * 1024)) : 0u;
    h = st > 0 ? __ldg(reinterpret_cast<const uint32_t*>(sp - 4)) : 0u;
  };
  if (lane == 31 && warp < steps) fetch(warp, fw, hw);
  for (int64_t step = warp; step < steps; step += nwarps) {
    const uint8_t* sp = base + step * (int64_t)(U * 1024);
    uint32_t v[U][8];
#pragma unroll
    for (int i = 0; i < U; ++i) ldg_chunk(v[i], sp + (lane + 32 * i) * 32);
    uint32_t nf[U], nh = 0;
    if (lane == 31 && step + nwarps < steps) fetch(step + nwarps, nf, nh);
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t supply = lane == 31 ? (i == 0 ? hw : v[i - 1][7]) : v[i][7];
      const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
      uint32_t nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
      if (lane == 31) nextw = fw[i];
      uint32_t hi;
      acc |= u8v_chunk_errors_planes_k(v[i], prev, nextw, kk, &hi);
    }
    if (lane == 31) {
#pragma unroll
      for (int i = 0; i < U; ++i) fw[i] = nf[i];
      hw = nh;
    }
  }
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc);
  if (lane == 0 && any) atomicOr(flag, 1u);
}
__global__ void __launch_bounds__(256, 4) k_v20_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  (void)spw;
  body20<4>(base, steps, flag, k);
}

// V21: load-only ceiling of the access pattern (grid-stride 4 KiB steps,
// 256-bit loads, OR-reduce; no validation).
template <int U>
__device__ __forceinline__ void body21(const uint8_t* base, int64_t steps, uint32_t* flag) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (int64_t step = warp; step < steps; step += nwarps) {
    const uint8_t* sp = base + step * (int64_t)(U * 1024);
    uint32_t v[U][8];
#pragma unroll
    for (int i = 0; i < U; ++i) ldg_chunk(v[i], sp + (lane + 32 * i) * 32);
#pragma unroll
    for (int i = 0; i < U; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc ^= v[i][j];
  }
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc == 0x12345678u);
  if (lane == 0 && any) atomicOr(flag, 1u);
}
__global__ void __launch_bounds__(256, 4) k_v21_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  (void)spw; (void)k;
  body21<4>(base, steps, flag);
}
__global__ void __launch_bounds__(256, 8) k_v21_u4_b8(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  (void)spw; (void)k;
  body21<4>(base, steps, flag);
}

// V22: V19 with other load flavours: LF = 1 adds the L2::256B prefetch-size
// hint, LF = 2 is a plain ld.global.v8 (L1-allocating).
template <int LF>
__device__ __forceinline__ void ldg_chunk_lf(uint32_t (&w)[8], const uint8_t* p) {
  if (LF == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
                   "=r"(w[7])
                 : "l"(p));
  else
    asm volatile("ld.global.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]),
                   "=r"(w[7])
                 : "l"(p));
}
template <int U, int LF>
__device__ __forceinline__ void body22(const uint8_t* base, int64_t steps, uint32_t* flag, const Cfg& k) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  u8v_consts kk;
  kk.one = k.one; kk.m256 = k.m256; kk.mshr4 = k.mshr4;
  uint32_t acc = 0;
  for (int64_t step = warp; step < steps; step += nwarps) {
    const uint8_t* sp = base + step * (int64_t)(U * 1024);
    uint32_t v[U][8];
#pragma unroll
    for (int i = 0; i < U; ++i) ldg_chunk_lf<LF>(v[i], sp + (lane + 32 * i) * 32);
    uint32_t carry_word = 0, nsw = 0;
    if (lane == 31 && step > 0) carry_word = __ldg(reinterpret_cast<const uint32_t*>(sp - 4));
    if (lane == 0 && step + 1 < steps) nsw = __ldg(reinterpret_cast<const uint32_t*>(sp + U * 1024));
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t supply = lane == 31 ? (i == 0 ? carry_word : v[i - 1][7]) : v[i][7];
      const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
      const uint32_t dn = lane == 0 ? (i + 1 < U ? v[i + 1][0] : nsw) : v[i][0];
      const uint32_t nextw = __shfl_sync(0xFFFFFFFFu, dn, (lane + 1) & 31);
      uint32_t hi;
      acc |= u8v_chunk_errors_planes_k(v[i], prev, nextw, kk, &hi);
    }
  }
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc);
  if (lane == 0 && any) atomicOr(flag, 1u);
}
__global__ void __launch_bounds__(256, 4) k_v22a_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                       uint32_t* flag, Cfg k) {
  (void)spw;
  body22<4, 1>(base, steps, flag, k);
}
__global__ void __launch_bounds__(256, 4) k_v22b_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                       uint32_t* flag, Cfg k) {
  (void)spw;
  body22<4, 2>(base, steps, flag, k);
}

__global__ void __launch_bounds__(256, 2) k_v19_u8_b2(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  (void)spw;
  body19<8>(base, steps, flag, k);
}
__global__ void __launch_bounds__(256, 6) k_v19_u2_b6(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  (void)spw;
  body19<2>(base, steps, flag, k);
}
__global__ void __launch_bounds__(256, 5) k_v19_u2_b5(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  (void)spw;
  body19<2>(base, steps, flag, k);
}
__global__ void __launch_bounds__(256, 3) k_v19_u4_b3(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  (void)spw;
  body19<4>(base, steps, flag, k);
}

// V23: V19 (grid-stride, correct halo/lookahead) with the permuted-order
// planes (production K1's chunk form), for occupancy / unroll sweeps.
template <int U>
__device__ __forceinline__ void body23(const uint8_t* base, int64_t steps, uint32_t* flag, const Cfg& k) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  u8v_consts kk;
  kk.one = k.one; kk.m256 = k.m256; kk.mshr4 = k.mshr4;
  uint32_t acc = 0;
  for (int64_t step = warp; step < steps; step += nwarps) {
    const uint8_t* sp = base + step * (int64_t)(U * 1024);
    uint32_t v[U][8];
#pragma unroll
    for (int i = 0; i < U; ++i) ldg_chunk(v[i], sp + (lane + 32 * i) * 32);
    uint32_t carry_word = 0, nsw = 0;
    if (lane == 31 && step > 0) carry_word = __ldg(reinterpret_cast<const uint32_t*>(sp - 4));
    if (lane == 0 && step + 1 < steps) nsw = __ldg(reinterpret_cast<const uint32_t*>(sp + U * 1024));
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t supply = lane == 31 ? (i == 0 ? carry_word : v[i - 1][7]) : v[i][7];
      const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
      const uint32_t dn = lane == 0 ? (i + 1 < U ? v[i + 1][0] : nsw) : v[i][0];
      const uint32_t nextw = __shfl_sync(0xFFFFFFFFu, dn, (lane + 1) & 31);
      uint32_t hi;
      acc |= u8v_chunk_errors_planes_perm_k(v[i], prev, nextw, kk, &hi);
    }
  }
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc);
  if (lane == 0 && any) atomicOr(flag, 1u);
}
#define KB_KERNEL23(U, MINB)                                                                     \
  __global__ void __launch_bounds__(256, MINB)                                                 \
      k_v23_u##U##_b##MINB(const uint8_t* base, int64_t steps, int64_t spw, uint32_t* flag, Cfg k) { \
    (void)spw;                                                                                 \
    body23<U>(base, steps, flag, k);                                                           \
  }
KB_KERNEL23(4, 4)
KB_KERNEL23(4, 3)
KB_KERNEL23(8, 2)
KB_KERNEL23(2, 5)
KB_KERNEL23(2, 4)
KB_KERNEL23(4, 5)
KB_KERNEL23(2, 6)
KB_KERNEL23(2, 8)
KB_KERNEL23(1, 8)
KB_KERNEL23(3, 5)
KB_KERNEL23(3, 4)

// V24: V23 (grid-stride, permuted planes) with rolling reload: each chunk
// slot is refilled with the same chunk of this warp's next step as soon as
// it is consumed; lane 31's last word is kept for the next chunk's halo.
template <int U>
__device__ __forceinline__ void body24(const uint8_t* base, int64_t steps, uint32_t* flag, const Cfg& k) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  u8v_consts kk;
  kk.one = k.one; kk.m256 = k.m256; kk.mshr4 = k.mshr4;
  uint32_t acc = 0;
  int64_t step = warp;
  if (step >= steps) return;
  const int64_t stride = nwarps * (int64_t)(U * 1024);
  const uint8_t* sp = base + step * (int64_t)(U * 1024);
  uint32_t v[U][8];
#pragma unroll
  for (int i = 0; i < U; ++i) ldg_chunk(v[i], sp + (lane + 32 * i) * 32);
  uint32_t carry_word = 0, nsw = 0;
  if (lane == 31 && step > 0) carry_word = __ldg(reinterpret_cast<const uint32_t*>(sp - 4));
  if (lane == 0 && step + 1 < steps) nsw = __ldg(reinterpret_cast<const uint32_t*>(sp + U * 1024));
  for (; step < steps; step += nwarps, sp += stride) {
    const bool more = step + nwarps < steps;
    const uint8_t* np = sp + stride;
    // Next step's halo / lookahead words, early.
    uint32_t ncarry = 0, nnsw = 0;
    if (more) {
      if (lane == 31) ncarry = __ldg(reinterpret_cast<const uint32_t*>(np - 4));
      if (lane == 0 && step + nwarps + 1 < steps) nnsw = __ldg(reinterpret_cast<const uint32_t*>(np + U * 1024));
    }
    uint32_t last = carry_word;  // lane 31: the word before the chunk being processed
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const uint32_t supply = lane == 31 ? last : v[i][7];
      const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
      const uint32_t dn = lane == 0 ? (i + 1 < U ? v[i + 1][0] : nsw) : v[i][0];
      const uint32_t nextw = __shfl_sync(0xFFFFFFFFu, dn, (lane + 1) & 31);
      uint32_t hi;
      acc |= u8v_chunk_errors_planes_perm_k(v[i], prev, nextw, kk, &hi);
      last = v[i][7];
      if (more) ldg_chunk(v[i], np + (lane + 32 * i) * 32);
    }
    carry_word = ncarry;
    nsw = nnsw;
  }
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc);
  if (lane == 0 && any) atomicOr(flag, 1u);
}
__global__ void __launch_bounds__(256, 4) k_v24_u4_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  (void)spw;
  body24<4>(base, steps, flag, k);
}
__global__ void __launch_bounds__(256, 3) k_v24_u4_b3(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  (void)spw;
  body24<4>(base, steps, flag, k);
}
__global__ void __launch_bounds__(256, 4) k_v24_u2_b4(const uint8_t* base, int64_t steps, int64_t spw,
                                                      uint32_t* flag, Cfg k) {
  (void)spw;
  body24<2>(base, steps, flag, k);
}

#define KB_KERNEL(V, U, MINB)                                                                  \
  __global__ void __launch_bounds__(256, MINB)                                                 \
      k_v##V##_u##U##_b##MINB(const uint8_t* base, int64_t steps, int64_t spw, uint32_t* flag, \
                              Cfg k) {                                                         \
    body<V, U>(base, steps, spw, flag, k);                                                     \
  }
KB_KERNEL(0, 2, 4)
KB_KERNEL(0, 1, 4)
KB_KERNEL(0, 1, 6)
KB_KERNEL(0, 2, 5)
KB_KERNEL(1, 2, 4)
KB_KERNEL(1, 1, 6)
KB_KERNEL(2, 2, 4)
KB_KERNEL(2, 1, 6)
KB_KERNEL(3, 2, 4)
KB_KERNEL(4, 2, 4)
KB_KERNEL(0, 4, 3)
KB_KERNEL(4, 4, 3)
KB_KERNEL(4, 2, 5)
KB_KERNEL(5, 2, 4)
KB_KERNEL(5, 4, 3)
KB_KERNEL(6, 4, 3)
KB_KERNEL(6, 2, 4)
KB_KERNEL(7, 4, 3)
KB_KERNEL(8, 4, 3)
KB_KERNEL(30, 4, 3)
KB_KERNEL(30, 4, 4)
KB_KERNEL(30, 2, 4)
KB_KERNEL(8, 2, 4)
KB_KERNEL(8, 4, 2)
KB_KERNEL(8, 1, 6)
KB_KERNEL(9, 4, 3)
KB_KERNEL(9, 2, 4)
KB_KERNEL(10, 4, 3)
KB_KERNEL(10, 4, 4)
KB_KERNEL(10, 2, 4)
KB_KERNEL(11, 4, 4)
KB_KERNEL(12, 4, 4)
#define KB_KERNEL_PF(V, U, MINB, PF)                                                            \
  __global__ void __launch_bounds__(256, MINB)                                                 \
      k_v##V##_u##U##_b##MINB##_p##PF(const uint8_t* base, int64_t steps, int64_t spw,          \
                                      uint32_t* flag, Cfg k) {                                 \
    body<V, U, PF>(base, steps, spw, flag, k);                                                 \
  }
KB_KERNEL_PF(6, 4, 3, 1)
KB_KERNEL_PF(6, 4, 3, 2)
KB_KERNEL_PF(6, 4, 3, 4)
KB_KERNEL_PF(6, 2, 4, 2)
KB_KERNEL_PF(6, 2, 4, 4)
KB_KERNEL_PF(4, 4, 3, 2)

typedef void (*KFn)(const uint8_t*, int64_t, int64_t, uint32_t*, Cfg);
struct Entry {
  const char* name;
  KFn fn;
  int u;
  int smem = 0;  // dynamic shared memory bytes (TMA variants)
};
static const Entry kEntries[] = {
    {"v0_u2_b4", k_v0_u2_b4, 2}, {"v0_u1_b4", k_v0_u1_b4, 1}, {"v0_u1_b6", k_v0_u1_b6, 1},
    {"v0_u2_b5", k_v0_u2_b5, 2}, {"v1_u2_b4", k_v1_u2_b4, 2}, {"v1_u1_b6", k_v1_u1_b6, 1},
    {"v2_u2_b4", k_v2_u2_b4, 2}, {"v2_u1_b6", k_v2_u1_b6, 1}, {"v3_u2_b4", k_v3_u2_b4, 2},
    {"v4_u2_b4", k_v4_u2_b4, 2}, {"v0_u4_b3", k_v0_u4_b3, 4}, {"v4_u4_b3", k_v4_u4_b3, 4},
    {"v4_u2_b5", k_v4_u2_b5, 2}, {"v5_u2_b4", k_v5_u2_b4, 2}, {"v5_u4_b3", k_v5_u4_b3, 4},
    {"v6_u4_b3", k_v6_u4_b3, 4}, {"v6_u2_b4", k_v6_u2_b4, 2}, {"v7_u4_b3", k_v7_u4_b3, 4},
    {"v30_nibble_tables_u4_b3", k_v30_u4_b3, 4}, {"v30_nibble_tables_u4_b4", k_v30_u4_b4, 4},
    {"v30_nibble_tables_u2_b4", k_v30_u2_b4, 2}, {"v8_u4_b3", k_v8_u4_b3, 4}, {"v8_u2_b4", k_v8_u2_b4, 2}, {"v8_u4_b2", k_v8_u4_b2, 4}, {"v8_u1_b6", k_v8_u1_b6, 1},
    {"v9_u4_b3", k_v9_u4_b3, 4}, {"v9_u2_b4", k_v9_u2_b4, 2},
    {"v10_u4_b3", k_v10_u4_b3, 4}, {"v10_u4_b4", k_v10_u4_b4, 4}, {"v10_u2_b4", k_v10_u2_b4, 2},
    {"v11_u4_b4", k_v11_u4_b4, 4}, {"v13_u4_b4", k_v13_u4_b4, 4},
    {"v14_u4_b4", k_v14_u4_b4, 4}, {"v15_u4_b4", k_v15_u4_b4, 4}, {"v16_u4_b4", k_v16_u4_b4, 4},
    {"v24_u4_b4", k_v24_u4_b4, 4}, {"v24_u4_b3", k_v24_u4_b3, 4}, {"v24_u2_b4", k_v24_u2_b4, 2},
    {"v23_u4_b4", k_v23_u4_b4, 4}, {"v23_u4_b3", k_v23_u4_b3, 4}, {"v23_u8_b2", k_v23_u8_b2, 8},
    {"v23_u2_b5", k_v23_u2_b5, 2}, {"v23_u2_b4", k_v23_u2_b4, 2}, {"v23_u4_b5", k_v23_u4_b5, 4},
    {"v23_u2_b6", k_v23_u2_b6, 2}, {"v23_u2_b8", k_v23_u2_b8, 2}, {"v23_u1_b8", k_v23_u1_b8, 1},
    {"v23_u3_b5", k_v23_u3_b5, 3}, {"v23_u3_b4", k_v23_u3_b4, 3},
    {"v19_u8_b2", k_v19_u8_b2, 8}, {"v19_u2_b6", k_v19_u2_b6, 2}, {"v19_u2_b5", k_v19_u2_b5, 2},
    {"v19_u4_b3", k_v19_u4_b3, 4},
    {"v22a_u4_b4", k_v22a_u4_b4, 4}, {"v22b_u4_b4", k_v22b_u4_b4, 4},
    {"v21_u4_b4", k_v21_u4_b4, 4}, {"v21_u4_b8", k_v21_u4_b8, 4},
    {"v20_u4_b4", k_v20_u4_b4, 4}, {"v19_u4_b4", k_v19_u4_b4, 4}, {"v19_u2_b4", k_v19_u2_b4, 2},
    {"v18_u4_b4", k_v18_u4_b4, 4}, {"v18_u4_b3", k_v18_u4_b3, 4}, {"v18_u2_b4", k_v18_u2_b4, 2},
    {"v25_u4_s3_b2", k_v25_u4_s3_b2, 4, 8 * 3 * 4096 + 8 * 3 * 8},
    {"v25_u4_s2_b3", k_v25_u4_s2_b3, 4, 8 * 2 * 4096 + 8 * 2 * 8},
    {"v25_u2_s3_b4", k_v25_u2_s3_b4, 2, 8 * 3 * 2048 + 8 * 3 * 8},
    {"v25_u2_s2_b4", k_v25_u2_s2_b4, 2, 8 * 2 * 2048 + 8 * 2 * 8},
    {"v25_u4_s4_b1", k_v25_u4_s4_b1, 4, 8 * 4 * 4096 + 8 * 4 * 8},
    {"tma_u2_s3_b4", k_tma_u2_s3_b4, 2, 8 * 3 * 2048 + 8 * 3 * 8},
    {"tma_u2_s4_b3", k_tma_u2_s4_b3, 2, 8 * 4 * 2048 + 8 * 4 * 8},
    {"tma_u4_s2_b3", k_tma_u4_s2_b3, 4, 8 * 2 * 4096 + 8 * 2 * 8},
    {"tma_u4_s3_b2", k_tma_u4_s3_b2, 4, 8 * 3 * 4096 + 8 * 3 * 8},
    {"tma_u1_s6_b4", k_tma_u1_s6_b4, 1, 8 * 6 * 1024 + 8 * 6 * 8},
    {"p1_u4_b4", k_p1_u4_b4, 4}, {"p2_u4_b4", k_p2_u4_b4, 4}, {"p4_u4_b4", k_p4_u4_b4, 4}, {"v12_u4_b4", k_v12_u4_b4, 4},
    {"db_u2_b3", k_db_u2_b3, 2}, {"db_u1_b4", k_db_u1_b4, 1}, {"db_u2_b2", k_db_u2_b2, 2}, {"db_u4_b2", k_db_u4_b2, 4},
    {"v6_u4_b3_p1", k_v6_u4_b3_p1, 4}, {"v6_u4_b3_p2", k_v6_u4_b3_p2, 4}, {"v6_u4_b3_p4", k_v6_u4_b3_p4, 4},
    {"v6_u2_b4_p2", k_v6_u2_b4_p2, 2}, {"v6_u2_b4_p4", k_v6_u2_b4_p4, 2}, {"v4_u4_b3_p2", k_v4_u4_b3_p2, 4},
};

}  // namespace kb

extern "C" {

int kb_count() { return (int)(sizeof(kb::kEntries) / sizeof(kb::kEntries[0])); }
const char* kb_name(int i) { return kb::kEntries[i].name; }

// Launch variant i over d_p[0..n) (n % 2048 == 0); returns blocks launched.
int kb_launch(int i, const uint8_t* d_p, uint64_t n, uint32_t* d_flag, void* stream) {
  const kb::Entry& e = kb::kEntries[i];
  int dev = 0, sms = 0, blocks_per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e.smem > 0) cudaFuncSetAttribute(e.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, e.smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, e.fn, 256, e.smem);
  const int64_t steps = (int64_t)(n / (e.u * 1024));
  int64_t warps = (int64_t)sms * blocks_per_sm * 8;
  if (warps > steps) warps = steps;
  const int64_t spw = (steps + warps - 1) / warps;
  warps = (steps + spw - 1) / spw;
  const int64_t blocks = (warps * 32 + 255) / 256;
  kb::Cfg k{1u, 256u, 1u << 28, 1u << 16, 1u << 24, 1u << 8};
  e.fn<<<(unsigned)blocks, 256, e.smem, (cudaStream_t)stream>>>(d_p, steps, spw, d_flag, k);
  return blocks_per_sm;
}

}  // extern "C"
