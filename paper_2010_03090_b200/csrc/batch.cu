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
// LDG each, halo and lookahead by SHFL).  Record starts only matter where
// they fall inside a chunk's look-back window:
//   * each step reads a window of 32 record starts (one coalesced load; more
//     windows only if the step holds more than 31 starts);
//   * a step with no start in it ("single") runs K1's chunk code unchanged;
//   * otherwise the lanes holding a start OR a bit into a per-warp shared
//     mask of the chunk it falls in (and the next chunk's look-back bits), and
//     only chunks with a nonzero mask take the record-bounded word function
//     (u8v_word_errors_bounded_lead), out of line so the hot loop stays small
//     in the instruction cache.
// Record attribution (a short scan of the offsets) runs only for chunks that
// hold an error.  Verdicts start at 1 (memset by the caller) and invalid
// records get a plain 0 store (idempotent, no atomics).
//
// The rare-pair check needs no record masking in the lead form: a flagged
// pair (j, j+1) that crosses into the next record means byte j is a lead
// ending its record, which is invalid anyway (utf8v_swar.h).
#include <cuda_runtime.h>
#include <stdint.h>

#include "chunk.cuh"
#include "kernels.cuh"
#include "utf8v_swar.h"

namespace u8v {

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

constexpr int kWarpsPerCta = kThreads / 32;

// What the record lookups need, passed by value: the out-of-line
// attribution taking the whole descriptor by reference would pin it in local
// memory and turn every offset lookup of the hot window loop into an LDL.
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
__device__ int64_t find_record(const RecView& d, int64_t pos) {
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
__device__ int64_t record_of(const RecView& d, int64_t r, int64_t q) {
  while (r < d.n_records && rec_start(d, r + 1) <= q) ++r;
  return r < d.n_records ? r : d.n_records;
}

__device__ __forceinline__ void mark_invalid(const RecView& d, int64_t r_from, int64_t q) {
  if (q < rec_start(d, 0)) return;
  const int64_t r = record_of(d, r_from, q);
  if (r < d.n_records) d.verdicts[r] = 0;
}

// Out-of-line, only for chunks with a flagged lane: the record of every
// flagged lane, and the record ending at every flagged record start (its end
// check), is marked invalid.  err / end: lane bits of chunk c in the permuted
// plane order of utf8v_bits.h (bit pos(i) = byte i).
__device__ __noinline__ void attribute_chunk(RecView d, int64_t c, uint32_t err, uint32_t end,
                                             int64_t r_from) {
  const int64_t q0 = c * kChunkBytes;
  while (err) {
    const int i = __ffs(err) - 1;
    err &= err - 1;
    mark_invalid(d, r_from, q0 + u8v_perm_byte((unsigned)i));
  }
  while (end) {
    const int i = __ffs(end) - 1;
    end &= end - 1;
    mark_invalid(d, r_from, q0 + u8v_perm_byte((unsigned)i) - 1);
  }
}

__global__ void __launch_bounds__(kThreads, 4) k_batch(BatchDesc d) {
  __shared__ unsigned long long s_mask[kWarpsPerCta][kStepChunks];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t warp = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kThreads) >> 5;
  // The byte range comes from the offsets themselves (read here, so the
  // launch needs no host round trip).  Malformed offsets are clamped to the
  // data: the kernel never reads outside [0, n).
  const RecView rv{d.offsets, d.verdicts, d.off32, d.n_records};
  d.lo = d.off32 + (int64_t)__ldg(d.offsets);
  d.hi = d.off32 + (int64_t)__ldg(d.offsets + d.n_records);
  if (d.hi > d.off32 + d.n_bytes) d.hi = d.off32 + d.n_bytes;
  if (d.lo > d.hi) d.lo = d.hi;
  if (d.hi <= d.lo) return;  // every record empty: all valid
  // Lanes [lo, hi]: lane hi carries the last record's end check; lanes past
  // it read zeros behind a record start and cannot flag.
  d.c_begin = d.lo / kChunkBytes;
  d.c_end = d.hi / kChunkBytes + 1;
  d.steps = (d.c_end - d.c_begin + kStepChunks - 1) / kStepChunks;
  d.steps_per_warp = (d.steps + nwarps - 1) / nwarps;
  int64_t step = warp * d.steps_per_warp;
  int64_t step_end = step + d.steps_per_warp;
  if (step_end > d.steps) step_end = d.steps;
  if (step >= step_end) return;
  unsigned long long* m = s_mask[wib];
#pragma unroll
  for (int i = 0; i < kU; ++i) m[lane + 32 * i] = 0;

  constexpr int64_t kStepBytes = (int64_t)kStepChunks * kChunkBytes;
  int64_t cstep = d.c_begin + step * kStepChunks;
  uint32_t carry_word = 0;
  if (lane == 31 && cstep > 0)
    carry_word = ld_word_masked(d.base, cstep * kChunkBytes - 4, d.lo, d.hi);
  // r0: the record holding byte hs = step start - 2, the first byte whose
  // record matters to the step (look-back of its first lanes).
  int64_t r0 = find_record(rv, cstep * kChunkBytes - 2);
  bool was_ascii = true;

  for (; step < step_end; ++step) {
    cstep = d.c_begin + step * kStepChunks;
    const int64_t s0 = cstep * kChunkBytes;
    const int64_t hs = s0 - 2;
    const int64_t se = s0 + kStepBytes;
    const int64_t nhs = se - 2;  // next step's hs

    const bool direct = s0 >= d.lo && se + 4 <= d.hi;
    Chunk v[kU];
    uint32_t nsw = 0;
    if (direct) {
#pragma unroll
      for (int i = 0; i < kU; ++i) v[i] = ld_chunk(d.base + (cstep + lane + 32 * i) * kChunkBytes);
      if (lane == 0) nsw = __ldg(reinterpret_cast<const uint32_t*>(d.base + se));
    } else {
#pragma unroll
      for (int i = 0; i < kU; ++i) {
        const int64_t c = cstep + lane + 32 * i;
        v[i] = c <= d.c_end ? ld_chunk_masked(d.base, c, d.lo, d.hi) : zero_chunk();
      }
      if (lane == 0) nsw = ld_word_guarded(d.base, se, d.lo, d.hi);
    }

    // Record starts in [hs, se): the window of the 32 records from r0.
    int64_t ob = rec_start(rv, r0 + lane);
    unsigned below = __ballot_sync(0xFFFFFFFFu, ob < se);
    const bool single = below == 1u && __shfl_sync(0xFFFFFFFFu, ob, 0) < hs;  // ob(0) = start(r0)
    int64_t r_next = r0;
    if (!single) {
      __syncwarp();  // the previous step's readers have cleared their masks
      int64_t r = r0;
      for (;;) {
        if (ob >= hs && ob < se) {
          const int64_t c = ob >> 5;  // chunk of the start (base coords)
          const int li = (int)(c - cstep);
          const int bit = (int)(ob & 31);
          // Low word: the chunk's record-start plane in permuted order; high
          // word of the next chunk: starts at its bytes -1 / -2 (bits 31 / 23).
          if (li >= 0) atomicOr(&m[li], 1ull << u8v_perm_pos((unsigned)bit));
          if (bit >= 30 && li + 1 < kStepChunks)
            atomicOr(&m[li + 1], 1ull << (bit == 31 ? 63 : 55));
        }
        // The next step's r0: the last record starting at or before nhs.
        const unsigned le = __ballot_sync(0xFFFFFFFFu, ob <= nhs);
        if (le != 0u) r_next = r + (31 - __clz(le));
        if (below != 0xFFFFFFFFu) break;
        r += 32;  // more than 31 starts in this step: next window
        ob = rec_start(rv, r + lane);
        below = __ballot_sync(0xFFFFFFFFu, ob < se);
        if (below == 0u) break;
      }
      __syncwarp();
    }

    // ASCII fast path, voted only after an all-ASCII step (as in K1).
    bool all_ascii = false;
    if (single && was_ascii) {
      uint32_t hibits = 0;
#pragma unroll
      for (int i = 0; i < kU; ++i) hibits |= chunk_hibits(v[i]);
      all_ascii = __all_sync(0xFFFFFFFFu, (hibits & U8V_B7) == 0);
    }
    uint32_t h7 = 0;
#pragma unroll
    for (int i = 0; i < kU; ++i) {
      const uint32_t up =
          lane == 31 ? (i == 0 ? carry_word : v[i - 1].w[kChunkWords - 1]) : v[i].w[kChunkWords - 1];
      const uint32_t prev = __shfl_sync(0xFFFFFFFFu, up, (lane + 31) & 31);
      const uint32_t dn = lane == 0 ? (i + 1 < kU ? v[i + 1].w[0] : nsw) : v[i].w[0];
      const uint32_t next = __shfl_sync(0xFFFFFFFFu, dn, (lane + 1) & 31);
      const int64_t c = cstep + lane + 32 * i;
      uint32_t err, end = 0, hi7 = 0;
      if (all_ascii) {
        u8v_carry cr = u8v_carry_of(prev);
        err = u8v_ascii_word_errors(v[i].w[0], &cr) & U8V_B7;
        if (err) err = u8v_chunk_errors_planes_perm_k(v[i].w, prev, next, d.k, &hi7);  // exact lanes
      } else if (single) {
        err = u8v_chunk_errors_planes_perm_k(v[i].w, prev, next, d.k, &hi7);
      } else {
        // Every chunk of a step holding record starts takes the bounded form
        // (uniform control flow; a zero mask gives the plain flags).
        const unsigned long long mask = m[lane + 32 * i];
        m[lane + 32 * i] = 0;
        err = u8v_chunk_errors_planes_perm_bounded_k(v[i].w, prev, next, d.k, (uint32_t)mask,
                                                     (uint32_t)(mask >> 32), &end, &hi7);
      }
      h7 |= hi7;
      if (err | end) attribute_chunk(rv, c, err, end, r0);
    }
    was_ascii = all_ascii || __all_sync(0xFFFFFFFFu, h7 == 0);
    if (lane == 31) carry_word = v[kU - 1].w[kChunkWords - 1];
    r0 = r_next;
  }
}

}  // namespace u8v

// Launcher used by capi.cu.  Fully asynchronous: the kernel reads the first
// and last offsets itself; the grid is sized from the data size n.
namespace u8v {
void launch_batch(const uint8_t* data, uint64_t n, const uint64_t* d_offsets, uint64_t n_records,
                  uint8_t* d_verdicts, cudaStream_t st) {
  if (n_records == 0 || n == 0) return;
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
  int64_t warps = max_resident_warps();
  if (warps > max_steps) warps = max_steps;
  const int64_t blocks = (warps * 32 + kThreads - 1) / kThreads;
  k_batch<<<(unsigned)blocks, kThreads, 0, st>>>(d);
}
}  // namespace u8v
