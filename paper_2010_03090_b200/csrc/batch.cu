// batch.cu -- K2: segmented validation, one verdict per record.
//
// Reference behaviour: each record is validated as its own stream -- the
// reference harness loops validate_lookup per record/segment (SURVEY.md
// §8(d)); every stream starts with a zero prev vector and ends with the
// incomplete check (proj/include/utf8v/lookup_kernel.hpp:115, :111, :128-132).
//
// B200 design: the records' bytes are contiguous in HBM with a CSR offsets
// array, so the kernel ignores record sizes for load balance and sweeps the
// byte array exactly like K1 (4 KiB warp steps, 32-byte chunks, one 256-bit
// LDG each, halo and lookahead by SHFL, the same unbounded permuted plane
// form).  A lane's record-bounded flag can differ from its unbounded one
// only for the first three lanes of a record (their look-back crosses the
// start) and for the previous record's end-of-stream lanes, so:
//   * a flagged lane is attributed, out of line, to its record (a shuffle
//     search over a window of 32 record starts) unless it is one of that
//     record's first three lanes or lies past the data;
//   * every record start is checked on its own, 32 starts per warp pass once
//     the sweep has passed them: each lane reads the 8 bytes around its start
//     (mostly L2 hits) and runs u8v_boundary_errors (utf8v_swar.h) for the
//     record ending there and the record starting there.
// The decomposition is proven against per-record validation on the CPU
// (tests/test_swar.py::test_k2_*).  Verdicts start at 1 (memset by the
// caller) and invalid records get a plain 0 store (idempotent, no atomics).
// Batches of few, large records (C2) go to K2L instead (validate.cu,
// launch_batch_large): K1's own sweep needs no record cursor there.
#include <cuda_runtime.h>
#include <stdint.h>

#include "chunk.cuh"
#include "kernels.cuh"
#include "serve.h"
#include "utf8v_state.h"
#include "utf8v_swar.h"

namespace u8v {

// CTA shape of K2: one 32-warp CTA per SM.  With four 8-warp CTAs per SM
// the warp scheduler's preference for older CTAs left the youngest CTA's
// equal share running alone at the end of the launch (as for K1,
// scripts/probes/k1_timeline.py); one CTA per SM keeps the warps in step:
// C3 0.200 -> 0.179 ms (tools/k2bench.py; 512 threads: 0.189).
#ifndef U8V_K2_THREADS
#define U8V_K2_THREADS 1024
#endif
constexpr int kK2Threads = U8V_K2_THREADS;
constexpr int kK2Blocks = 1024 / kK2Threads;

struct BatchDesc {
  const uint8_t* base;   // 32-aligned; data byte i is base[off32 + i]
  const uint64_t* offsets;
  uint8_t* verdicts;
  int64_t off32;
  int64_t lo, hi;        // bytes [lo, hi) (base coords) belong to some record
  int64_t c_begin, c_end;
  int64_t steps, steps_per_warp;
  int64_t n_records;
  int64_t n_bytes;  // data size (clamp for malformed offsets)
  u8v_consts k;  // runtime multipliers (FMA-pipe routing, utf8v_swar.h)
};

// What the record lookups need, passed by value: out-of-line helpers taking
// the whole descriptor by reference would pin it in local memory and turn
// every offset lookup into an LDL.
struct RecView {
  const uint64_t* offsets;
  uint8_t* verdicts;
  int64_t off32;
  int64_t n_records;
};

// Offset of record start r in base coordinates (r > n_records: +inf).
__device__ __forceinline__ int64_t rec_start(const RecView& d, int64_t r) {
  return r <= d.n_records ? (int64_t)__ldg(d.offsets + r) + d.off32 : INT64_MAX;
}

// Warp-cooperative: the largest record r in [0, n_records-1] with
// start(r) <= pos (0 when pos precedes every record).  32-ary search.
__device__ int64_t find_record(const RecView& d, int64_t pos, int64_t lo = 0, int64_t hi = 0) {
  const int lane = threadIdx.x & 31;
  int64_t a = 0, b = d.n_records;  // answer index in [a, b], start(a) <= pos
  // First probe: 32 starts around the record the byte position suggests
  // (records of equal size), 128 records apart.  On C3 the guess is within
  // +-2048 records nearly always, which saves two of the search's dependent
  // offset loads; otherwise the 32-ary search runs from the whole range.
  if (hi > lo && d.n_records > 4096) {
    const double f = (double)(pos - lo) / (double)(hi - lo);
    const int64_t g = (int64_t)(f * (double)d.n_records);
    constexpr int64_t kW = 128;
    int64_t p = g + (int64_t)(lane - 16) * kW;
    p = p < 0 ? 0 : (p > d.n_records ? d.n_records : p);
    const unsigned m = __ballot_sync(0xFFFFFFFFu, rec_start(d, p) <= pos);
    if (m != 0u && m != 0xFFFFFFFFu && (m & 1u)) {  // a bracket inside the probe
      const int top = 31 - __clz(m);
      const int64_t pa = g + (int64_t)(top - 16) * kW;
      a = pa < 0 ? 0 : pa;
      const int64_t pb = pa + kW - 1;
      b = pb < d.n_records ? pb : d.n_records;
    } else if (rec_start(d, 0) > pos) {
      return 0;
    }
  } else if (rec_start(d, 0) > pos) {
    return 0;
  }
  while (b - a >= 32) {
    const int64_t stride = (b - a) / 32 + 1;
    const int64_t p = a + lane * stride;
    const bool ok = p <= b && rec_start(d, p) <= pos;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, ok);
    const int top = 31 - __clz(m);
    const int64_t na = a + top * stride;
    const int64_t nb = na + stride - 1;
    a = na;
    b = nb < b ? nb : b;
  }
  const int64_t p = a + lane;
  const bool ok = p <= b && rec_start(d, p) <= pos;
  const unsigned m = __ballot_sync(0xFFFFFFFFu, ok);
  int64_t r = a + (31 - __clz(m));
  return r < d.n_records ? r : d.n_records - 1;
}

// Positions as 32-bit offsets from a base (a step or the warp's range start),
// clamped far out on either side, so compares and shuffles stay 32-bit.
constexpr int kFar = 1 << 30;
__device__ __forceinline__ int rel32(int64_t pos, int64_t s0) {
  const int64_t r = pos - s0;
  return r > kFar ? kFar : (r < -kFar ? -kFar : (int)r);
}

// Out of line, for steps with a flagged lane: each flagged lane q goes to
// its record -- the last window start at or before q, found by a 5-step
// shuffle search over the window (lane L holds start(r0 + L) - s0, with
// start(r0) <= s0 or r0 = 0) -- unless q is one of that record's first three
// lanes or lies past the data (those lanes are settled by fix_boundary).
// e0..e3: lane bits of chunk (lane + 32 i) of the step in the permuted plane
// order of utf8v_bits.h (bit pos(i) = byte i).
// kState (segment states, utf8v_state.h): a flagged lane counts only when it
// is one of its record's interior lanes [start+3, end-1) -- it also must not
// read the next record's first byte.
template <bool kState>
__device__ __forceinline__ void attribute_step(RecView d, int64_t s0, int64_t hi, uint32_t e0, uint32_t e1,
                                            uint32_t e2, uint32_t e3, int o, int64_t r0) {
  const int lane = threadIdx.x & 31;
  const bool full = __all_sync(0xFFFFFFFFu, o < kStepChunks * kChunkBytes);
  const int hi_rel = rel32(hi, s0);
  static_assert(kU == 4, "attribute_step takes one mask per chunk of a step");
  // One flagged lane per lane and round, lowest chunk first.
  while (__any_sync(0xFFFFFFFFu, (e0 | e1 | e2 | e3) != 0u)) {
    // chunks of lane L in the paired layout: 2L, 2L+1, 64+2L, 64+2L+1
    int q = -1, c = 2 * lane;
    uint32_t e = 0;
    if (e0) {
      e = e0;
      e0 &= e0 - 1;
    } else if (e1) {
      e = e1;
      e1 &= e1 - 1;
      c += 1;
    } else if (e2) {
      e = e2;
      e2 &= e2 - 1;
      c += 64;
    } else if (e3) {
      e = e3;
      e3 &= e3 - 1;
      c += 65;
    }
    if (e) q = c * kChunkBytes + (int)u8v_perm_byte((unsigned)(__ffs(e) - 1));
    int L = 0;
#pragma unroll
    for (int st = 16; st > 0; st >>= 1) {
      const int cand = L + st;
      const int t = __shfl_sync(0xFFFFFFFFu, o, cand & 31);
      if (cand <= 31 && t <= q) L = cand;
    }
    const int start = __shfl_sync(0xFFFFFFFFu, o, L);
    const int nxt = kState ? __shfl_sync(0xFFFFFFFFu, o, (L + 1) & 31) : 0;
    if (q >= 0 && q < hi_rel && q >= start) {
      int64_t r = r0 + L;
      int64_t st_abs = s0 + start;
      int64_t end_abs = s0 + nxt;  // kState: start(r + 1) when L < 31
      if (full && L == 31) {
        // More starts than one window holds (dense records): gallop, then
        // binary search the offsets -- O(log) loads in the records skipped.
        const int64_t qa = s0 + q;
        int64_t a = r, span = 4;  // start(a) <= qa
        while (a + span <= d.n_records && rec_start(d, a + span) <= qa) {  // gallop
          a += span;
          span <<= 1;
        }
        int64_t b = a + span - 1 < d.n_records ? a + span - 1 : d.n_records;
        while (a < b) {  // largest r in [a, b] with start(r) <= qa
          const int64_t mid = (a + b + 1) >> 1;
          if (rec_start(d, mid) <= qa) a = mid;
          else b = mid - 1;
        }
        r = a;
        st_abs = rec_start(d, r);
      }
      if (kState && (L == 31 || r != r0 + L)) end_abs = rec_start(d, r + 1);
      if (r < d.n_records && s0 + q - st_abs >= 3 && (!kState || s0 + q < end_abs - 1)) d.verdicts[r] = 0;
    }
  }
}


// The usual flagged step of a mostly-valid batch, settled without building
// the attribution window: one lane (src) has flagged chunks, they lie inside
// one record at least three bytes past its start and before the data end --
// one verdict store.  The record is found directly in the two consecutive
// batches of starts the warp holds (T, the taken batch in shared memory, and
// nx, the next one, both relative to range_lo): no start in (ql, qh], the
// last start <= ql.  Chunk granularity ([ql, qh] spans src's flagged chunks);
// anything else (a flagged chunk near a record start, dense records, several
// flagged lanes) returns false for the exact attribution.
__device__ __forceinline__ bool settle_fast(const RecView& d, const int* T, int nx, int64_t rb, int s0, int hi_rel,
                                            uint32_t e0, uint32_t e1, uint32_t e2, uint32_t e3, int src) {
  const int lane = threadIdx.x & 31;
  const int cl = 2 * lane + (e0 ? 0 : (e1 ? 1 : (e2 ? 64 : 65)));
  const int ch = 2 * lane + (e3 ? 65 : (e2 ? 64 : (e1 ? 1 : 0)));
  const int ql = s0 + __shfl_sync(0xFFFFFFFFu, cl, src) * kChunkBytes;
  const int qh = s0 + __shfl_sync(0xFFFFFFFFu, ch, src) * kChunkBytes + kChunkBytes - 1;
  const unsigned nl = __ballot_sync(0xFFFFFFFFu, nx <= ql);
  if (nl != __ballot_sync(0xFFFFFFFFu, nx <= qh) || nl == 0xFFFFFFFFu) return false;
  int start;
  int64_t r;
  if (nl) {
    const int L = 31 - __clz(nl);
    start = __shfl_sync(0xFFFFFFFFu, nx, L);
    r = rb + L;
  } else {
    const int tv = T[lane];
    const unsigned tl = __ballot_sync(0xFFFFFFFFu, tv <= ql);
    if (tl == 0u || tl != __ballot_sync(0xFFFFFFFFu, tv <= qh)) return false;
    const int L = 31 - __clz(tl);
    start = __shfl_sync(0xFFFFFFFFu, tv, L);
    r = rb - 32 + L;
  }
  if (ql < start + 3 || qh >= hi_rel) return false;
  if (lane == 0 && r < d.n_records) d.verdicts[r] = 0;
  return true;
}

// attribute_step when exactly one lane (src) of the warp has flagged bits
// and settle_fast did not apply.  Its masks are broadcast and the warp walks
// their bits together, one flagged lane q per iteration: its window slot is
// the last lane whose start is <= q (one ballot: the window is ascending),
// instead of the 5-round shuffle search per round of attribute_step.
template <bool kState>
__device__ __forceinline__ void attribute_lane(RecView d, int64_t s0, int64_t hi, uint32_t e0, uint32_t e1,
                                               uint32_t e2, uint32_t e3, int o, int64_t r0, int src) {
  const int lane = threadIdx.x & 31;
  const int hi_rel = rel32(hi, s0);
  uint32_t f0 = __shfl_sync(0xFFFFFFFFu, e0, src), f1 = __shfl_sync(0xFFFFFFFFu, e1, src);
  uint32_t f2 = __shfl_sync(0xFFFFFFFFu, e2, src), f3 = __shfl_sync(0xFFFFFFFFu, e3, src);
  const bool full = __all_sync(0xFFFFFFFFu, o < kStepChunks * kChunkBytes);
  while ((f0 | f1 | f2 | f3) != 0u) {  // warp-uniform
    // chunks of lane src in the paired layout: 2 src, 2 src + 1, 64 + 2 src, 64 + 2 src + 1
    int c = 2 * src;
    uint32_t e;
    if (f0) {
      e = f0;
      f0 &= f0 - 1;
    } else if (f1) {
      e = f1;
      f1 &= f1 - 1;
      c += 1;
    } else if (f2) {
      e = f2;
      f2 &= f2 - 1;
      c += 64;
    } else {
      e = f3;
      f3 &= f3 - 1;
      c += 65;
    }
    const int q = c * kChunkBytes + (int)u8v_perm_byte((unsigned)(__ffs(e) - 1));
    const unsigned le = __ballot_sync(0xFFFFFFFFu, o <= q);
    const int L = le ? 31 - __clz(le) : 0;
    const int start = __shfl_sync(0xFFFFFFFFu, o, L);
    const int nxt = kState ? __shfl_sync(0xFFFFFFFFu, o, (L + 1) & 31) : 0;
    if (lane == 0 && q < hi_rel && q >= start) {
      int64_t r = r0 + L;
      int64_t st_abs = s0 + start;
      int64_t end_abs = s0 + nxt;
      if (full && L == 31) {  // dense records: as attribute_step
        const int64_t qa = s0 + q;
        int64_t a = r, span = 4;
        while (a + span <= d.n_records && rec_start(d, a + span) <= qa) {
          a += span;
          span <<= 1;
        }
        int64_t b = a + span - 1 < d.n_records ? a + span - 1 : d.n_records;
        while (a < b) {
          const int64_t mid = (a + b + 1) >> 1;
          if (rec_start(d, mid) <= qa) a = mid;
          else b = mid - 1;
        }
        r = a;
        st_abs = rec_start(d, r);
      }
      if (kState && (L == 31 || r != r0 + L)) end_abs = rec_start(d, r + 1);
      if (r < d.n_records && s0 + q - st_abs >= 3 && (!kState || s0 + q < end_abs - 1)) d.verdicts[r] = 0;
    }
  }
}


// Record boundaries, a batch of 32 starts at a time (lane L: start rb + L
// at o, relative to the warp's range_lo, a multiple of 32).  The taken
// batch waits in shared memory, not registers (the sweep needs them all):
// take_batch stores each lane's start and issues asynchronous copies of the
// bytes s-4 .. s+3 around it -- two aligned 8-byte words when they lie in
// chunks the sweep reads anyway, else the word is assembled byte by byte
// inside [lo, hi) and stored pre-shifted, so check_batch combines both cases
// the same way.  Bytes outside the two records are masked by check_batch.
struct WarpCtx {
  int64_t lo, hi, c_end, range_lo, rb;
  int prev_last, range_rel;
  int hi_rel;  // hi - range_lo (clamped, rel32)
  int taken;  // a batch sits in the slot (starts rb-32 .. rb-1)
};

struct BatchSlot {
  unsigned long long w[32][2];
  int o[32];
  int a0;  // start(rb - 1)
};

__device__ __forceinline__ void take_batch(BatchSlot* sl, const uint8_t* base, int64_t lo, int64_t hi,
                                           int64_t range_lo, int o, int a0, int range_rel) {
  const int lane = threadIdx.x & 31;
  sl->o[lane] = o;
  if (lane == 0) sl->a0 = a0;
  if (o < 0 || o >= range_rel) return;
  const int64_t s = range_lo + o;
  const int64_t w0 = (s - 4) & ~(int64_t)7;
  if (w0 >= (lo & ~(int64_t)31) && w0 + 16 <= ((hi + 31) & ~(int64_t)31)) {
    const unsigned dst = (unsigned)__cvta_generic_to_shared(&sl->w[lane][0]);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(base + w0) : "memory");
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8), "l"(base + w0 + 8) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    return;
  }
  uint64_t w = 0;
  for (int k = 0; k < 8; ++k) {
    const int64_t q = s - 4 + k;
    if (q >= lo && q < hi) w |= (uint64_t)base[q] << (8 * k);
  }
  const unsigned sh = (unsigned)((o - 4) & 7) * 8u;
  sl->w[lane][0] = w << sh;
  sl->w[lane][1] = sh ? w >> (64u - sh) : 0ull;
}

// The boundary at start o of record rr = rf + lane: record rr-1 = [a, o)
// ends there, record rr = [o, b) starts there (either may be empty or
// absent).  nx: the following batch (lane 0 = start(rf + 32)).
template <bool kState>
__device__ __forceinline__ void check_batch(const RecView& rv, BatchSlot* sl, int nx, int64_t rf, int range_rel,
                                            u8v_consts k) {
  const int lane = threadIdx.x & 31;
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncwarp();
  const int o = sl->o[lane];
  int a = __shfl_up_sync(0xFFFFFFFFu, o, 1);
  if (lane == 0) a = sl->a0;
  int b = __shfl_down_sync(0xFFFFFFFFu, o, 1);
  const int nb = __shfl_sync(0xFFFFFFFFu, nx, 0);
  if (lane == 31) b = nb;
  const int64_t rr = rf + lane;
  // kState: the boundary lanes are seam lanes, evaluated by combine().
  if (!kState && o >= 0 && o < range_rel) {
    const uint64_t w0 = sl->w[lane][0], w1 = sl->w[lane][1];
    const unsigned sh = (unsigned)((o - 4) & 7) * 8u;
    const uint64_t w8 = sh ? (w0 >> sh) | (w1 << (64u - sh)) : w0;
    int ka = rr > 0 ? a - (o - 4) : 4, kb = rr < rv.n_records ? b - (o - 4) : 4;
    ka = ka < 0 ? 0 : (ka > 4 ? 4 : ka);
    kb = kb < 4 ? 4 : (kb > 8 ? 8 : kb);
    const uint32_t f = u8v_boundary_errors(w8, (unsigned)ka, (unsigned)kb, k);
    if ((f & 1u) && rr > 0) rv.verdicts[rr - 1] = 0;
    if ((f & 2u) && rr < rv.n_records) rv.verdicts[rr] = 0;
  }
  __syncwarp();  // the slot is refilled next
}

#ifdef U8V_TIMELINE
// DEVELOPMENT (tools/kvar.sh builds only): per-warp start/end %globaltimer
// and SM id of K2 (scripts/probes/k2_timeline.py).
__device__ unsigned long long* g_timeline_k2;
__device__ __forceinline__ unsigned long long k2_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
template <bool kState>
__device__ void batch_body(BatchDesc d);
template <bool kState>
__global__ void __launch_bounds__(kK2Threads, kK2Blocks) k_batch(BatchDesc d) {
  const unsigned long long t0 = k2_gtimer();
  batch_body<kState>(d);
  if ((threadIdx.x & 31) == 0 && g_timeline_k2 != nullptr) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int64_t w = ((int64_t)blockIdx.x * kK2Threads + threadIdx.x) >> 5;
    g_timeline_k2[3 * w] = t0;
    g_timeline_k2[3 * w + 1] = k2_gtimer();
    g_timeline_k2[3 * w + 2] = smid;
  }
}
extern "C" int u8v_timeline_k2_set(unsigned long long* p) {
  return (int)cudaMemcpyToSymbol(g_timeline_k2, &p, sizeof(p));
}
template <bool kState>
__device__ __forceinline__ void batch_body(BatchDesc d) {
#else
template <bool kState>
__global__ void __launch_bounds__(kK2Threads, kK2Blocks) k_batch(BatchDesc d) {
#endif
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kK2Threads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kK2Threads) >> 5;
  // The byte range comes from the offsets themselves (read here, so the
  // launch needs no host round trip).  Malformed offsets are clamped to the
  // data: the kernel never reads outside [0, n).
  const RecView rv{d.offsets, d.verdicts, d.off32, d.n_records};
  d.lo = d.off32 + (int64_t)__ldg(d.offsets);
  d.hi = d.off32 + (int64_t)__ldg(d.offsets + d.n_records);
  if (d.hi > d.off32 + d.n_bytes) d.hi = d.off32 + d.n_bytes;
  if (d.lo > d.hi) d.lo = d.hi;
  if (d.hi <= d.lo) return;  // every record empty: all valid
  // Lanes [lo, hi]: the chunk holding byte hi is swept too; the last
  // record's end is settled by the boundary at hi.
  d.c_begin = d.lo / kChunkBytes;
  d.c_end = d.hi / kChunkBytes + 1;
  d.steps = (d.c_end - d.c_begin + kStepChunks - 1) / kStepChunks;
  d.steps_per_warp = (d.steps + nwarps - 1) / nwarps;
  const int64_t step0 = warp * d.steps_per_warp;
  int64_t step_end = step0 + d.steps_per_warp;
  if (step_end > d.steps) step_end = d.steps;
  if (step0 >= step_end) return;
  const int nsteps = (int)(step_end - step0);

  constexpr int kStepBytes = kStepChunks * kChunkBytes;
  // A batch of 32 starts is taken once the sweep passes its 16th start: its
  // bytes are copied asynchronously (no stall), the older half from L2, the
  // newer half from DRAM just ahead of the sweep, which then finds them in
  // L2.  Taking it at its last start left the oldest sectors ~6 steps back,
  // partly evicted: 0.210 -> 0.206 ms on C3 (tools/k2bench.py).
  constexpr int kTrigger = 15;
  // Loop state is kept 32-bit and relative (positions to range_lo, records
  // to r_in) so it stays in registers across the chunk math.
  const int64_t range_lo = (d.c_begin + step0 * kStepChunks) * kChunkBytes;
  uint32_t carry_word = 0;
  if (lane == 31 && range_lo > 0) carry_word = ld_word_masked(d.base, range_lo - 4, d.lo, d.hi);
  // Record starts are consumed in batches of 32 (lane L: start(rb + L),
  // 32-bit relative to range_lo), each batch prefetched one batch ahead:
  //   nx      the next batch's starts (loaded when the previous one was taken)
  //   p_*     the taken batch: its bytes around each start are loaded when
  //           the sweep passes its last start (L2-hot) and checked one step
  //           later, so neither load sits on the sweep's critical path.
  // A batch is correct whenever it is checked (verdicts only go 1 -> 0).
  // The same registers give the attribution window: start(rb - 1) (the
  // taken batch's last start, before the current step) followed by nx.
  const int64_t r_in = find_record(rv, range_lo - 1, d.lo, d.hi);  // last start before the range (or 0)
  const int64_t s_in = rec_start(rv, r_in);
  int64_t rb = r_in + (s_in < range_lo ? 1 : 0);
  int nx = rel32(rec_start(rv, rb + lane), range_lo);
  int prev_last = rb > r_in ? rel32(s_in, range_lo) : -kFar;  // start(rb - 1); rb == r_in only at rb = 0
  const int range_rel = nsteps * kStepBytes;
  __shared__ BatchSlot slots[kK2Threads / 32];
  BatchSlot* const sl = &slots[threadIdx.x >> 5];
  // Warp-uniform state the sweep does not touch each step lives in shared
  // memory (every lane writes the same value), so the hot loop's registers
  // hold only the chunk math and its cursor (no spills).
  __shared__ WarpCtx ctxs[kK2Threads / 32];
  volatile WarpCtx* const cx = &ctxs[threadIdx.x >> 5];
  cx->lo = d.lo;
  cx->hi = d.hi;
  cx->c_end = d.c_end;
  cx->range_lo = range_lo;
  cx->rb = rb;
  cx->prev_last = prev_last;
  cx->taken = 0;
  cx->range_rel = range_rel;
  cx->hi_rel = rel32(d.hi, range_lo);
  bool pend = false;
  int fire = 0;
  bool was_ascii = true;

  // Steps [jb, jd) are interior (all bytes real, lookahead word in range):
  // plain loads from a pointer advanced 4 KiB per step.
  int jb = (int)((d.lo - range_lo + kStepBytes - 1) / kStepBytes);
  int jd = d.hi - 4 - range_lo >= 0 ? (int)((d.hi - 4 - range_lo) / kStepBytes) : 0;
  jb = jb < 0 ? 0 : jb;
  jd = jd > nsteps ? nsteps : jd;
  const uint8_t* p = d.base + range_lo + lane * kChunkBytes;
  // K2 follows its verdict-initialisation kernel with programmatic
  // serialisation (launch_batch): the prologue above -- offsets, the record
  // search, the first batch -- overlaps it; verdict stores start only after
  // it has completed.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int j = 0; j < nsteps; ++j, p += kStepBytes) {
    Chunk v[kU];
    uint32_t nsw = 0;
    if (j >= jb && j < jd) {
#pragma unroll
      for (int i = 0; i < kU; ++i) v[i] = ld_chunk(p + ((i >> 1) * 64 + (i & 1) + lane) * kChunkBytes);
      ld_word_if(lane == 0, p + kStepBytes, nsw);
    } else {
      const int64_t lo = cx->lo, hi = cx->hi, c_end = cx->c_end;
      const int64_t cstep = (cx->range_lo + (int64_t)j * kStepBytes) / kChunkBytes;
#pragma unroll
      for (int i = 0; i < kU; ++i) {
        const int64_t c = cstep + (i >> 1) * 64 + 2 * lane + (i & 1);
        v[i] = c <= c_end ? ld_chunk_masked(d.base, c, lo, hi) : zero_chunk();
      }
      if (lane == 0) nsw = ld_word_guarded(d.base, (cstep + kStepChunks) * kChunkBytes, lo, hi);
    }

    // Paired layout (K1's interior steps): lane L holds chunks 2L, 2L+1,
    // 64+2L, 64+2L+1; the odd chunks' halo words and the even chunks'
    // lookahead words come from the lane itself.
    const uint32_t up0 = lane == 31 ? carry_word : v[1].w[kChunkWords - 1];
    const uint32_t up2 = lane == 31 ? v[1].w[kChunkWords - 1] : v[3].w[kChunkWords - 1];
    const uint32_t prev[kU] = {__shfl_sync(0xFFFFFFFFu, up0, (lane + 31) & 31), v[0].w[kChunkWords - 1],
                               __shfl_sync(0xFFFFFFFFu, up2, (lane + 31) & 31), v[2].w[kChunkWords - 1]};
    // Unbounded lane flags (K1's chunk form).  ASCII fast path (voted only
    // after an all-ASCII step): a step of bytes < 0x80 only needs the
    // pending incomplete check of the bytes before each chunk; if that
    // fires, the step is recomputed exactly (attribution needs the lanes).
    bool all_ascii = false;
    if (was_ascii) {
      uint32_t hibits = 0;
#pragma unroll
      for (int i = 0; i < kU; ++i) hibits |= chunk_hibits(v[i]);
      all_ascii = __all_sync(0xFFFFFFFFu, (hibits & U8V_B7) == 0);
      if (all_ascii) {
        uint32_t ae = 0;
#pragma unroll
        for (int i = 0; i < kU; ++i) {
          u8v_carry cr = u8v_carry_of(prev[i]);
          ae |= u8v_ascii_word_errors(v[i].w[0], &cr) & U8V_B7;
        }
        all_ascii = !__any_sync(0xFFFFFFFFu, ae != 0u);
      }
    }
    if (!all_ascii) {
      uint32_t h7 = 0, err[kU], any = 0;
      const uint32_t dn1 = lane == 0 ? v[2].w[0] : v[0].w[0];
      const uint32_t dn3 = lane == 0 ? nsw : v[2].w[0];
      const uint32_t n1 = __shfl_sync(0xFFFFFFFFu, dn1, (lane + 1) & 31);
      const uint32_t n3 = __shfl_sync(0xFFFFFFFFu, dn3, (lane + 1) & 31);
      const uint32_t next[kU] = {v[1].w[0], n1, v[3].w[0], n3};
#pragma unroll
      for (int i = 0; i < kU; ++i) {
        uint32_t hi7 = 0;
        err[i] = u8v_chunk_errors_planes_perm_k(v[i].w, prev[i], next[i], d.k, &hi7);
        if (i == kU - 1) h7 = hi7;  // the step's last KiB predicts the next step (K1)
        any |= err[i];
      }
      was_ascii = __all_sync(0xFFFFFFFFu, h7 == 0);
#ifdef U8V_K2_NO_ATTR  // DEVELOPMENT (tools/kvar.sh): the sweep without attribution
      const unsigned flagged = __ballot_sync(0xFFFFFFFFu, any == 0xFFFFFFFFu);
#else
      const unsigned flagged = __ballot_sync(0xFFFFFFFFu, any != 0u);
#endif
      if (flagged) {
        // Window: lane L = start(r0 + L) - s0 with start(r0) <= s0 (or r0 = 0):
        // the taken batch's last start (< s0, else that batch would not have
        // been taken) followed by the next batch's first 31.
        const int s0 = j * kStepBytes;
        const int64_t rbc = cx->rb;
#ifndef U8V_K2_NO_LANE_PATH
        if (!kState && (flagged & (flagged - 1)) == 0 && cx->taken &&
            settle_fast(rv, sl->o, nx, rbc, s0, cx->hi_rel, err[0], err[1], err[2], err[3], __ffs(flagged) - 1))
          goto settled;
#endif
        {
        int o;
        int64_t r0;
        if (cx->taken) {
          // The taken batch T (starts rbc-32 ..) and the next one (nx) are
          // consecutive: the window is T[k ..] then nx, k = T's last start
          // <= s0 (T[kTrigger] < s0: T was taken at an earlier step's end).
          const int tv = sl->o[lane];
          const unsigned le = __ballot_sync(0xFFFFFFFFu, tv <= s0);
          const int k = 31 - __clz(le);
          const int src = lane + k;
          const int a = __shfl_sync(0xFFFFFFFFu, tv, src & 31);
          const int b = __shfl_sync(0xFFFFFFFFu, nx, (src - 32) & 31);
          o = (src < 32 ? a : b) - s0;
          r0 = rbc - 32 + k;
        } else {
          const int up = __shfl_up_sync(0xFFFFFFFFu, nx, 1);
          o = (rbc == 0 ? nx : (lane == 0 ? cx->prev_last : up)) - s0;
          r0 = rbc == 0 ? 0 : rbc - 1;
        }
#ifndef U8V_K2_NO_LANE_PATH
        if ((flagged & (flagged - 1)) == 0)
          attribute_lane<kState>(rv, cx->range_lo + s0, cx->hi, err[0], err[1], err[2], err[3], o, r0,
                                 __ffs(flagged) - 1);
        else
#endif
          attribute_step<kState>(rv, cx->range_lo + s0, cx->hi, err[0], err[1], err[2], err[3], o, r0);
        }
      }
    }
  settled:
    if (lane == 31) carry_word = v[kU - 1].w[kChunkWords - 1];

    // Boundary batches: the pending one is checked a step after it was
    // taken; the trigger reads nx a step after it was loaded (no stall).
#ifdef U8V_K2_OLD_TRIGGER
    if (pend || __shfl_sync(0xFFFFFFFFu, nx, kTrigger) < (j + 1) * kStepBytes) {
#else
    // `fire`: the next step with boundary work -- the step after a take (the
    // pending batch is checked then), else the step whose end passes the
    // next batch's trigger start (computed when the block last ran, a step
    // after nx was loaded): one compare per step.
    if (j >= fire) {
#endif
      if (pend) {
        check_batch<kState>(rv, sl, nx, cx->rb - 32, cx->range_rel, d.k);
        pend = false;
      }
      while (__shfl_sync(0xFFFFFFFFu, nx, kTrigger) < (j + 1) * kStepBytes) {
        const int64_t rbc = cx->rb;
        if (pend) check_batch<kState>(rv, sl, nx, rbc - 32, cx->range_rel, d.k);
        take_batch(sl, d.base, cx->lo, cx->hi, cx->range_lo, nx, cx->prev_last, cx->range_rel);
        pend = true;
        cx->taken = 1;
        cx->prev_last = __shfl_sync(0xFFFFFFFFu, nx, 31);
        cx->rb = rbc + 32;
        nx = rel32(rec_start(rv, rbc + 32 + lane), cx->range_lo);
      }
      // (the loop left nx's trigger start >= (j + 1) * kStepBytes > 0)
      fire = pend ? j + 1 : (int)((unsigned)__shfl_sync(0xFFFFFFFFu, nx, kTrigger) / (unsigned)kStepBytes);
    }
  }
  // The range's remaining boundaries.
  {
    int64_t rbc = cx->rb;
    int pl = cx->prev_last;
    const int64_t lo = cx->lo, hi = cx->hi, rlo = cx->range_lo;
    const int rrel = cx->range_rel;
    if (pend) check_batch<kState>(rv, sl, nx, rbc - 32, rrel, d.k);
    while (__shfl_sync(0xFFFFFFFFu, nx, 0) < rrel) {
      take_batch(sl, d.base, lo, hi, rlo, nx, pl, rrel);
      pl = __shfl_sync(0xFFFFFFFFu, nx, 31);
      rbc += 32;
      nx = rel32(rec_start(rv, rbc + lane), rlo);
      check_batch<kState>(rv, sl, nx, rbc - 32, rrel, d.k);
    }
  }
}
}  // namespace u8v

// Launcher used by capi.cu.  Fully asynchronous: the kernel reads the first
// and last offsets itself; the grid is sized from the data size n.  K2L
// takes the batch when it has <= kLargeMaxRecords records of >= 64 KiB on
// average (known here from n and n_records).
namespace u8v {
int batch_threads() { return kK2Threads; }

int batch_blocks_per_sm() {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_batch<false>, kK2Threads, 0) != cudaSuccess)
    cudaGetLastError();
  return b < 1 ? 1 : b;
}

// verdicts[0 .. n) = 1, 16 bytes per store.  Both launches of a batch call
// allow programmatic serialisation:
//   * this grid triggers its dependent (K2 / K2L) on entry, so that grid's
//     CTAs start their prologue (offsets, record search, first boundary
//     batch) at once and wait for this grid's completion only before their
//     first verdict store;
//   * this grid itself may start while the previous kernel on the stream
//     (say the previous batch's K2, which triggers on entry too) drains, and
//     waits for it to complete before its first store -- so the next call's
//     prologue overlaps the previous call's drain.  A predecessor that does
//     not trigger early (a producer of the input) is waited for in full
//     before this grid starts, and everything K2 reads was complete by then.
// A small grid (<= 16 CTAs) leaves the other SMs free for K2's CTAs.
// C3 back to back 170.1 -> 167.6 us, C2 49.2 -> 46.6 us (tools/k2cmp.py).
__global__ void k_init_verdicts(uint8_t* __restrict__ v, uint64_t n) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t head = (16 - ((uintptr_t)v & 15)) & 15;  // bytes before the first 16-byte boundary
  if (i < head && i < n) v[i] = 1;
  const uint64_t body = n > head ? (n - head) / 16 : 0;
  const uint4 ones = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
  for (uint64_t k = i; k < body; k += (uint64_t)gridDim.x * blockDim.x)
    reinterpret_cast<uint4*>(v + head)[k] = ones;
  const uint64_t tail0 = head + body * 16;
  if (tail0 + i < n && i < 16) v[tail0 + i] = 1;
}

template <class... Args>
static void launch_pdl(void (*kernel)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args);

static void init_verdicts(uint8_t* v, uint64_t n, cudaStream_t st) {
  const uint64_t vecs = n / 16 + 1;
  uint64_t blocks = (vecs + 255) / 256;
  if (blocks > 16) blocks = 16;
  launch_pdl(k_init_verdicts, dim3((unsigned)(blocks ? blocks : 1)), dim3(256), 0, st, v, n);
}

template <class... Args>
static void launch_pdl(void (*kernel)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

void launch_batch(const uint8_t* data, uint64_t n, const uint64_t* d_offsets, uint64_t n_records,
                  uint8_t* d_verdicts, cudaStream_t st, bool states) {
  if (n_records == 0) return;
  serve_quiesce();  // K2's grid holds the resident CTAs of every SM (static partition)
  init_verdicts(d_verdicts, n_records, st);
  if (n == 0) return;
  if (!states && launch_batch_large(data, n, d_offsets, n_records, d_verdicts, st)) return;
  BatchDesc d;
  const uintptr_t up = (uintptr_t)data;
  d.off32 = (int64_t)(up & (kChunkBytes - 1));
  d.base = (const uint8_t*)(up - (uintptr_t)d.off32);
  d.offsets = d_offsets;
  d.verdicts = d_verdicts;
  d.n_records = (int64_t)n_records;
  d.n_bytes = (int64_t)n;
  d.k = u8v_make_consts();
  d.lo = d.hi = d.c_begin = d.c_end = d.steps = d.steps_per_warp = 0;  // set by the kernel
  const int64_t max_steps = ((int64_t)n + d.off32 + 2 * kChunkBytes) / (kStepChunks * kChunkBytes) + 1;
  int64_t warps = k2_resident_warps();
  if (warps > max_steps) warps = max_steps;
  const int64_t blocks = (warps * 32 + kK2Threads - 1) / kK2Threads;
  if (states)
    launch_pdl(k_batch<true>, dim3((unsigned)blocks), dim3(kK2Threads), 0, st, d);
  else
    launch_pdl(k_batch<false>, dim3((unsigned)blocks), dim3(kK2Threads), 0, st, d);
}

// Per-record segment states (utf8v_state.h) from K2's state-mode output
// (clean[r] = 1 iff none of record r's interior lanes is flagged): length,
// first and last four bytes.  One thread per record; offsets clamped to the
// data as in K2.
__global__ void k_record_states(const uint8_t* __restrict__ data, uint64_t n, const uint64_t* __restrict__ offsets,
                                uint64_t n_records, const uint8_t* __restrict__ clean, u8v_state* __restrict__ out) {
  const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_records) return;
  uint64_t a = __ldg(offsets + r), b = __ldg(offsets + r + 1);
  a = a < n ? a : n;
  b = b < n ? b : n;
  b = b > a ? b : a;
  u8v_state s = u8v_state_empty();
  s.len = b - a;
  s.flag = s.len > 4 && clean[r] == 0 ? 1u : 0u;
  const uint64_t k = s.len < 4 ? s.len : 4;
  for (uint64_t i = 0; i < k; ++i) {
    s.head[i] = data[a + i];
    s.tail[4 - k + i] = data[b - k + i];
  }
  out[r] = s;
}

void launch_record_states(const uint8_t* data, uint64_t n, const uint64_t* d_offsets, uint64_t n_records,
                          const uint8_t* d_clean, u8v_state* d_out, cudaStream_t st) {
  if (n_records == 0) return;
  k_record_states<<<(unsigned)((n_records + 255) / 256), 256, 0, st>>>(data, n, d_offsets, n_records, d_clean,
                                                                       d_out);
}

// In-order fold of count states into *out (one CTA): each thread folds a
// contiguous run, then the runs are combined pairwise in order, a tree over
// shared memory (combine() is associative, not commutative).
__global__ void __launch_bounds__(256) k_states_reduce(const u8v_state* __restrict__ in, uint64_t count,
                                                       u8v_state* __restrict__ out) {
  __shared__ u8v_state part[256];
  const uint64_t t = threadIdx.x, T = blockDim.x;
  const uint64_t a = count * t / T, b = count * (t + 1) / T;
  u8v_state s = u8v_state_empty();
  for (uint64_t i = a; i < b; ++i) s = u8v_state_combine(s, in[i]);
  part[t] = s;
  __syncthreads();
  for (uint64_t w = 1; w < T; w <<= 1) {
    if ((t & (2 * w - 1)) == 0 && t + w < T) part[t] = u8v_state_combine(part[t], part[t + w]);
    __syncthreads();
  }
  if (t == 0) *out = part[0];
}

void launch_states_reduce(const u8v_state* d_in, uint64_t count, u8v_state* d_out, cudaStream_t st) {
  k_states_reduce<<<1, 256, 0, st>>>(d_in, count, d_out);
}
}  // namespace u8v
