// tools/kbench.cu -- DEVELOPMENT HARNESS (not product code): times variants of
// the K1 inner loop (word formulation x occupancy x chunks-per-step) on the
// same device buffer, so formulation choices are made on measurements.
// Interior-only skeleton: n must be a multiple of 2 KiB and 32-byte aligned.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../paper_2010_03090_b200/csrc/utf8v_swar.h"

namespace kb {

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
      } else if (V == 6) {
        const uint32_t nextw = __shfl_down_sync(0xFFFFFFFFu, v[i][0], 1);
#pragma unroll
        for (int j = 0; j < 8; ++j) e |= word6(v[i][j], j < 7 ? v[i][j + 1] : nextw, c, k);
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
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc & 0x80808080u);
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
};
static const Entry kEntries[] = {
    {"v0_u2_b4", k_v0_u2_b4, 2}, {"v0_u1_b4", k_v0_u1_b4, 1}, {"v0_u1_b6", k_v0_u1_b6, 1},
    {"v0_u2_b5", k_v0_u2_b5, 2}, {"v1_u2_b4", k_v1_u2_b4, 2}, {"v1_u1_b6", k_v1_u1_b6, 1},
    {"v2_u2_b4", k_v2_u2_b4, 2}, {"v2_u1_b6", k_v2_u1_b6, 1}, {"v3_u2_b4", k_v3_u2_b4, 2},
    {"v4_u2_b4", k_v4_u2_b4, 2}, {"v0_u4_b3", k_v0_u4_b3, 4}, {"v4_u4_b3", k_v4_u4_b3, 4},
    {"v4_u2_b5", k_v4_u2_b5, 2}, {"v5_u2_b4", k_v5_u2_b4, 2}, {"v5_u4_b3", k_v5_u4_b3, 4},
    {"v6_u4_b3", k_v6_u4_b3, 4}, {"v6_u2_b4", k_v6_u2_b4, 2}, {"v7_u4_b3", k_v7_u4_b3, 4},
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
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, e.fn, 256, 0);
  const int64_t steps = (int64_t)(n / (e.u * 1024));
  int64_t warps = (int64_t)sms * blocks_per_sm * 8;
  if (warps > steps) warps = steps;
  const int64_t spw = (steps + warps - 1) / warps;
  warps = (steps + spw - 1) / spw;
  const int64_t blocks = (warps * 32 + 255) / 256;
  kb::Cfg k{1u, 256u, 1u << 28, 1u << 16, 1u << 24, 1u << 8};
  e.fn<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d_p, steps, spw, d_flag, k);
  return blocks_per_sm;
}

}  // extern "C"
