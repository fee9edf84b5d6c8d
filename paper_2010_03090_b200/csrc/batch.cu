// batch.cu -- K2: segmented validation, one verdict per record.
//
// Reference behaviour: each record is validated as its own stream -- the
// reference harness loops validate_lookup per record/segment (SURVEY.md
// §8(d)); every stream starts with a zero prev vector and ends with the
// incomplete check (proj/include/utf8v/lookup_kernel.hpp:115, :111, :128-132).
//
// B200 design: the records' bytes are contiguous in HBM with a CSR offsets
// array, so the kernel ignores record sizes for load balance and sweeps the
// byte array in the same 2 KiB warp steps as K1 (coalesced LDG.128, halo via
// SHFL).  Record starts are turned into per-chunk boundary masks: each step
// loads a window of 32 offsets (one coalesced load), every lane builds the
// 20-bit mask of record starts over its chunk's [start-4, end) bytes, and
// chunks with a start inside use u8v_word_errors_bounded, which drops
// look-back sources from earlier records and emits the previous record's
// end check.  Error attribution to records (a few offset reads) only runs
// when a chunk actually holds an error.  Verdicts start at 1 (memset) and
// invalid records get a plain 0 store (idempotent, no atomics).
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"
#include "utf8v_swar.h"

namespace u8v {

struct BatchDesc {
  const uint8_t* base;   // 16-aligned; data byte i is base[off16 + i]
  const uint64_t* offsets;
  uint8_t* verdicts;
  int64_t off16;
  int64_t lo, hi;        // bytes [lo, hi) (base coords) belong to some record
  int64_t c_begin, c_end;
  int64_t steps, steps_per_warp;
  int64_t n_records;
  u8v_consts k;  // runtime multipliers (FMA-pipe routing, utf8v_swar.h)
};

__device__ __forceinline__ uint4 ld_stream_b(const uint8_t* p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
      : "l"(p));
  return r;
}

__device__ __forceinline__ uint4 ld_chunk_masked_b(const uint8_t* base, int64_t c, int64_t lo,
                                                   int64_t hi) {
  const int64_t b0 = c * 16;
  if (b0 >= lo && b0 + 16 <= hi) return ld_stream_b(base + b0);
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int64_t q = b0 + k;
    if (q >= lo && q < hi) w[k >> 2] |= (uint32_t)base[q] << (8 * (k & 3));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// Offset of record start r in base coordinates (r > n_records: +inf).
__device__ __forceinline__ int64_t rec_start(const BatchDesc& d, int64_t r) {
  return r <= d.n_records ? (int64_t)__ldg(d.offsets + r) + d.off16 : INT64_MAX;
}

// Warp-cooperative: the largest record r in [0, n_records-1] with
// start(r) <= pos (0 when pos precedes every record).  32-ary search.
__device__ int64_t find_record(const BatchDesc& d, int64_t pos) {
  const int lane = threadIdx.x & 31;
  int64_t a = 0, b = d.n_records;  // answer index in [a, b], start(a) <= pos
  if (rec_start(d, 0) > pos) return 0;
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

// Record holding byte q (base coords), scanning forward from record r
// (start(r) <= q).  n_records when q is past the last record.
__device__ int64_t record_of(const BatchDesc& d, int64_t r, int64_t q) {
  while (r < d.n_records && rec_start(d, r + 1) <= q) ++r;
  return r < d.n_records ? r : d.n_records;
}

// Rare path: store 0 for the record of every flagged lane, and for the
// record ending at every flagged record start (end check).
__device__ void attribute(const BatchDesc& d, int64_t r_from, int64_t pos0, uint32_t err,
                          uint32_t end_err) {
  for (int j = 0; j < 4; ++j) {
    const int64_t q = pos0 + j;
    if ((err >> (8 * j + 7)) & 1) {
      if (q >= rec_start(d, 0)) {
        const int64_t r = record_of(d, r_from, q);
        if (r < d.n_records) d.verdicts[r] = 0;
      }
    }
    if ((end_err >> (8 * j + 7)) & 1) {
      if (q - 1 >= rec_start(d, 0)) {
        const int64_t r = record_of(d, r_from, q - 1);
        if (r < d.n_records) d.verdicts[r] = 0;
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 4) k_batch(BatchDesc d) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  int64_t step = warp * d.steps_per_warp;
  int64_t step_end = step + d.steps_per_warp;
  if (step_end > d.steps) step_end = d.steps;
  if (step >= step_end) return;

  uint32_t carry_word = 0;
  int64_t cstep = d.c_begin + step * kBStepChunks;
  if (lane == 31 && cstep > 0) {
    const int64_t pos = cstep * 16 - 4;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (pos + k >= d.lo && pos + k < d.hi) carry_word |= (uint32_t)d.base[pos + k] << (8 * k);
  }
  int64_t r0 = find_record(d, cstep * 16 - 4);

  for (; step < step_end; ++step) {
    cstep = d.c_begin + step * kBStepChunks;
    const int64_t hs = cstep * 16 - 4;                  // first halo byte of the step
    const int64_t se = (cstep + kBStepChunks) * 16;       // step end (exclusive)
    // Window of record starts: O_k = start(r0 + k).
    const int64_t ok = rec_start(d, r0 + lane);
    const unsigned inside = __ballot_sync(0xFFFFFFFFu, ok < se);
    const int nb = __popc(inside);  // starts before the step end (O_0 <= hs included)
    const bool dense = nb == 32;    // window may not hold every start of the step

    const bool interior = cstep * 16 >= d.lo && se <= d.hi;
    uint4 v[kBU];
    if (interior) {
#pragma unroll
      for (int i = 0; i < kBU; ++i) v[i] = ld_stream_b(d.base + (cstep + lane + 32 * i) * 16);
    } else {
#pragma unroll
      for (int i = 0; i < kBU; ++i) {
        const int64_t c = cstep + lane + 32 * i;
        v[i] = c < d.c_end ? ld_chunk_masked_b(d.base, c, d.lo, d.hi) : make_uint4(0, 0, 0, 0);
      }
    }
    const bool single = !dense && nb == 1;  // the whole step lies in record r0
    uint32_t hibits = 0;
#pragma unroll
    for (int i = 0; i < kBU; ++i) hibits |= v[i].x | v[i].y | v[i].z | v[i].w;
    const bool all_ascii = single && __all_sync(0xFFFFFFFFu, (hibits & U8V_B7) == 0);

#pragma unroll
    for (int i = 0; i < kBU; ++i) {
      const uint32_t supply = lane == 31 ? (i == 0 ? carry_word : v[i - 1].w) : v[i].w;
      const uint32_t prev = __shfl_sync(0xFFFFFFFFu, supply, (lane + 31) & 31);
      const int64_t c = cstep + lane + 32 * i;
      const int64_t cb = c * 16 - 4;  // mask bit j <-> byte cb + j
      // 20-bit mask of record starts over bytes [16c-4, 16c+16).
      uint32_t mask = 0;
      int64_t rc = r0;  // a record starting at or before cb (for attribution)
      if (!single) {
        if (!dense) {
          for (int k = 0; k < nb; ++k) {
            const int64_t b = __shfl_sync(0xFFFFFFFFu, ok, k);
            if (b <= cb) rc = r0 + k;
            if (b >= cb && b < cb + 20) mask |= 1u << (b - cb);
          }
        } else {
          // Pathological density (> 31 records per 2 KiB): per-lane scan.
          rc = record_of(d, r0, cb < 0 ? 0 : cb);
          if (rc >= d.n_records) rc = d.n_records - 1;
          for (int64_t r = rc; r <= d.n_records; ++r) {
            const int64_t b = rec_start(d, r);
            if (b >= cb + 20) break;
            if (b >= cb) mask |= 1u << (b - cb);
          }
        }
      }
      if (c >= d.c_end) continue;  // after the warp-wide shuffles above
      if (all_ascii) {
        u8v_carry cr = u8v_carry_of(prev);
        const uint32_t e = u8v_ascii_word_errors(v[i].x, &cr) & U8V_B7;
        if (e) attribute(d, rc, c * 16, e, 0);
      } else if ((mask >> 2) == 0) {
        u8v_carry cr = u8v_carry_of(prev);
        const uint32_t w4[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t e = u8v_word_errors_k(w4[k], &cr, d.k) & U8V_B7;
          if (e) attribute(d, rc, c * 16 + 4 * k, e, 0);
        }
      } else {
        u8v_carry cr = u8v_carry_of(prev);
        const uint32_t w4[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t bm = u8v_spread4(mask >> (4 + 4 * k));
          const uint32_t pbm = u8v_spread4(mask >> (4 * k));
          uint32_t end_err;
          const uint32_t e = u8v_word_errors_bounded_k(w4[k], &cr, bm, pbm, &end_err, d.k);
          if (e | end_err) attribute(d, rc, c * 16 + 4 * k, e, end_err);
        }
      }
    }
    if (lane == 31) carry_word = v[kBU - 1].w;
    // Advance the record pointer to the record holding the next step's halo.
    const int64_t nhs = hs + kBStepChunks * 16;
    if (!dense) {
      const unsigned le = __ballot_sync(0xFFFFFFFFu, ok <= nhs);
      r0 += (31 - __clz(le));
    } else {
      r0 = find_record(d, nhs);
    }
  }
}

}  // namespace u8v

// Launcher used by capi.cu: needs the first and last offsets (host values).
namespace u8v {
void launch_batch_known(const uint8_t* data, const uint64_t* d_offsets, uint64_t n_records,
                        uint64_t first_off, uint64_t last_off, uint8_t* d_verdicts,
                        cudaStream_t st) {
  if (n_records == 0) return;
  BatchDesc d;
  const uintptr_t up = (uintptr_t)data;
  d.off16 = (int64_t)(up & 15u);
  d.base = (const uint8_t*)(up - (uintptr_t)d.off16);
  d.offsets = d_offsets;
  d.verdicts = d_verdicts;
  d.lo = d.off16 + (int64_t)first_off;
  d.hi = d.off16 + (int64_t)last_off;
  d.n_records = (int64_t)n_records;
  d.k = u8v_make_consts();
  if (d.hi <= d.lo) return;  // every record empty: all valid
  d.c_begin = d.lo / 16;
  d.c_end = (d.hi + 3 + 15) / 16;
  const int64_t chunks = d.c_end - d.c_begin;
  d.steps = (chunks + kBStepChunks - 1) / kBStepChunks;
  int64_t warps = max_resident_warps();
  if (warps > d.steps) warps = d.steps;
  if (warps < 1) warps = 1;
  d.steps_per_warp = (d.steps + warps - 1) / warps;
  warps = (d.steps + d.steps_per_warp - 1) / d.steps_per_warp;
  const int64_t blocks = (warps * 32 + kThreads - 1) / kThreads;
  k_batch<<<(unsigned)blocks, kThreads, 0, st>>>(d);
}
}  // namespace u8v
