// validate.cu -- sm_100a kernels for single-stream Lookup validation.
//
//   k_validate          K1: OR of the per-lane error flags of one stream (or
//                       of one lane range of it: a pipeline piece, a shard),
//                       reduced with REDUX + one atomicOr per warp.
//   k_validate_track    K1 for the verdict path: also records the first
//                       flagged step (each lane's first, atomicMin).
//   k_locate_step       K3: one warp recomputes that step, takes its first
//                       flagged 32-byte chunk, and one thread decodes the
//                       <= 42-byte window around it into the reference's
//                       (offset, kind).
//
// Reference path replaced: validate_with<V> / lookup_checker<V>
// (proj/include/utf8v/lookup_kernel.hpp:82-134) reached through
// validate_lookup (proj/src/lookup.cpp:39-41); error positions as produced by
// oracle_validate (proj/src/oracle.cpp:10-44) in the CLI's failure path
// (proj/tools/main.cpp:129-147).
//
// Data layout: the caller's bytes stay where they are in HBM.  A stream is
// viewed through a 32-byte aligned base; chunk c is bytes [32c, 32c+32) of
// that base, bytes outside the valid range [lo, hi) read as zero (the
// reference's zero prev vector and zero-padded tail).  A warp owns a
// contiguous run of 4 KiB steps; in a step lane L holds chunks L, L+32, L+64, L+96,
// each fetched by one 256-bit LDG (LDG.E.ENL2.256: a warp instruction is one
// fully coalesced 1 KiB sweep) and gets the word before each chunk from lane
// L-1 with one SHFL (lane 0 from lane 31's previous chunk), so the 3-byte
// look-back halo never touches memory twice.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "chunk.cuh"
#include "kernels.cuh"
#include "locate.cuh"
#include "serve.h"
#include "stream_edge.cuh"
#include "utf8v_swar.h"

namespace u8v {

// Errors of one step's chunks v[i] (chunk cstep + lane + 32 i).  The word
// before each chunk comes from lane L-1 (lane 0: lane 31's previous chunk,
// or carry_word), the word after from lane L+1 (lane 31: lane 0's next
// chunk, or nsw = the next step's first word, loaded by lane 0).
//
// ASCII fast path (lookup_kernel.hpp:94-96): a step whose bytes are all
// < 0x80 only needs the pending incomplete check of the bytes before it.
// The warp vote that detects such a step waits for all of the step's loads
// and costs ~7% on multibyte text, so it is only taken when the previous
// step looked ASCII (`was_ascii`); otherwise the plane path runs and
// reports ASCII-ness after the fact from plane 7 of the step's last chunk
// per lane (its last KiB: one vote, no OR over the chunks; +1.2 % on C1,
// tools/k1bench.py).  The prediction only gates the attempt: the fast path
// checks every byte of the step with its own vote.
template <bool kPos, bool kRanged>
__device__ __forceinline__ uint32_t step_errors(const StreamDesc& d, const Chunk (&v)[kU],
                                                int64_t cstep, int lane, uint32_t& carry_word,
                                                uint32_t nsw, int& first_i, bool& was_ascii) {
  bool all_ascii = false;
  if (!kRanged && was_ascii) {
    uint32_t hibits = 0;
#pragma unroll
    for (int i = 0; i < kU; ++i) hibits |= chunk_hibits(v[i]);
    all_ascii = __all_sync(0xFFFFFFFFu, (hibits & U8V_B7) == 0);
  }
  uint32_t step_err = 0;
  if (all_ascii) {
#pragma unroll
    for (int i = 0; i < kU; ++i) {
      const uint32_t up =
          lane == 31 ? (i == 0 ? carry_word : v[i - 1].w[kChunkWords - 1]) : v[i].w[kChunkWords - 1];
      const uint32_t prev = __shfl_sync(0xFFFFFFFFu, up, (lane + 31) & 31);
      u8v_carry cr = u8v_carry_of(prev);
      const uint32_t e = u8v_ascii_word_errors(v[i].w[0], &cr) & U8V_B7;
      step_err |= e;
      if (kPos && e != 0 && first_i == kU) first_i = i;
    }
  } else {
    uint32_t h7 = 0;
#pragma unroll
    for (int i = 0; i < kU; ++i) {
      const uint32_t up =
          lane == 31 ? (i == 0 ? carry_word : v[i - 1].w[kChunkWords - 1]) : v[i].w[kChunkWords - 1];
      const uint32_t prev = __shfl_sync(0xFFFFFFFFu, up, (lane + 31) & 31);
      const uint32_t dn = lane == 0 ? (i + 1 < kU ? v[i + 1].w[0] : nsw) : v[i].w[0];
      const uint32_t next = __shfl_sync(0xFFFFFFFFu, dn, (lane + 1) & 31);
      const int64_t c = cstep + lane + 32 * i;
      uint32_t e = 0;
      if (!(kRanged && c >= d.c_end)) {
        uint32_t hi7;
        e = chunk_errors<kRanged>(v[i], prev, next, d.k, c * kChunkBytes, d.L0, d.L1, &hi7);
        if (i == kU - 1) h7 = hi7;  // the step's last KiB predicts the next step
      }
      step_err |= e;
      if (kPos && e != 0 && first_i == kU) first_i = i;
    }
    all_ascii = !kRanged && __all_sync(0xFFFFFFFFu, h7 == 0);
  }
  was_ascii = all_ascii;
  if (lane == 31) carry_word = v[kU - 1].w[kChunkWords - 1];
  return step_err;
}

// Interior steps of K1's sweep use a paired chunk layout: lane L holds
// chunks 2L, 2L+1, 64+2L, 64+2L+1 of the step (v[0..3]).  The odd chunks take
// their halo word, and the even ones their lookahead word, from the same
// lane; the rest come by one rotate-shuffle each: 4 SHFL + 4 SEL per step
// instead of 8 + 8 (+1.7 % on C1, tools/k1bench.py).  Each load instruction
// then covers 16 half-used 128-byte lines instead of 8 full ones; the step's
// four instructions still read every sector once.  Lane flags do not depend
// on the layout, so edge steps, K3's recompute and the batch kernels keep
// the one-chunk-per-lane layout of step_errors.
__device__ __forceinline__ uint32_t step_errors_pairs(const StreamDesc& d, const Chunk (&v)[kU], int lane,
                                                      uint32_t carry_word, uint32_t nsw, bool& was_ascii) {
  const uint32_t up0 = lane == 31 ? carry_word : v[1].w[kChunkWords - 1];
  const uint32_t up2 = lane == 31 ? v[1].w[kChunkWords - 1] : v[3].w[kChunkWords - 1];
  const uint32_t p0 = __shfl_sync(0xFFFFFFFFu, up0, (lane + 31) & 31);
  const uint32_t p2 = __shfl_sync(0xFFFFFFFFu, up2, (lane + 31) & 31);
  const uint32_t prev[kU] = {p0, v[0].w[kChunkWords - 1], p2, v[2].w[kChunkWords - 1]};
  bool all_ascii = false;
  if (was_ascii) {
    uint32_t hibits = 0;
#pragma unroll
    for (int i = 0; i < kU; ++i) hibits |= chunk_hibits(v[i]);
    all_ascii = __all_sync(0xFFFFFFFFu, (hibits & U8V_B7) == 0);
  }
  uint32_t step_err = 0;
  if (all_ascii) {
#pragma unroll
    for (int i = 0; i < kU; ++i) {
      u8v_carry cr = u8v_carry_of(prev[i]);
      step_err |= u8v_ascii_word_errors(v[i].w[0], &cr) & U8V_B7;
    }
  } else {
    const uint32_t dn1 = lane == 0 ? v[2].w[0] : v[0].w[0];
    const uint32_t dn3 = lane == 0 ? nsw : v[2].w[0];
    const uint32_t n1 = __shfl_sync(0xFFFFFFFFu, dn1, (lane + 1) & 31);
    const uint32_t n3 = __shfl_sync(0xFFFFFFFFu, dn3, (lane + 1) & 31);
    const uint32_t next[kU] = {v[1].w[0], n1, v[3].w[0], n3};
    uint32_t h7 = 0;
#pragma unroll
    for (int i = 0; i < kU; ++i) {
      uint32_t hi7;
      step_err |= u8v_chunk_errors_planes_perm_k(v[i].w, prev[i], next[i], d.k, &hi7);
      if (i == kU - 1) h7 = hi7;
    }
    all_ascii = __all_sync(0xFFFFFFFFu, h7 == 0);
  }
  was_ascii = all_ascii;
  return step_err;
}

// Interior steps (all bytes real, all lanes wanted, lookahead word in range)
// form one contiguous run [*int_b, *int_d) of step indices; only the
// head/tail steps take masked loads.
__device__ __forceinline__ void interior_steps(const StreamDesc& d, int64_t* int_b, int64_t* int_d) {
  const int64_t in_lo = d.lo > d.L0 ? d.lo : d.L0;
  const int64_t in_hi = d.hi < d.L1 ? d.hi : d.L1;
  const int64_t sb = kStepChunks * (int64_t)kChunkBytes;
  // + 4: the word before an interior step is real too (plain halo load).
  int64_t b = (in_lo + 4 - d.c_begin * kChunkBytes + sb - 1) / sb;
  if (b < 0) b = 0;
  int64_t e = (in_hi - d.c_begin * kChunkBytes) / sb;
  const int64_t h = (d.hi - 4 - d.c_begin * kChunkBytes) / sb;
  if (e > h) e = h;
  if (e < b) e = b;
  *int_b = b;
  *int_d = e;
}

// Errors of step `step` (any step: interior steps take the plain loads, edge
// steps the masked ones and lane ranges).  The chunk after the last evaluated
// one is loaded too: its first byte is the lookahead of the last evaluated
// lane (lead form).
template <bool kPos>
__device__ __forceinline__ uint32_t any_step_errors(const StreamDesc& d, int64_t step, bool interior, int lane,
                                                    int& first_i, bool& was_ascii) {
  const int64_t sb = kStepChunks * (int64_t)kChunkBytes;
  const int64_t cstep = d.c_begin + step * kStepChunks;
  const int64_t s0 = cstep * kChunkBytes;
  Chunk v[kU];
  uint32_t carry_word = 0, nsw = 0;
  if (interior) {
    const uint8_t* p = d.base + s0 + lane * kChunkBytes;
#pragma unroll
    for (int i = 0; i < kU; ++i) v[i] = ld_chunk(p + 32 * i * kChunkBytes);
    ld_word_if(lane == 31, d.base + s0 - 4, carry_word);
    ld_word_if(lane == 0, d.base + s0 + sb, nsw);
    return step_errors<kPos, false>(d, v, cstep, lane, carry_word, nsw, first_i, was_ascii);
  }
#pragma unroll
  for (int i = 0; i < kU; ++i) {
    const int64_t c = cstep + lane + 32 * i;
    v[i] = c <= d.c_end ? ld_chunk_masked(d.base, c, d.lo, d.hi) : zero_chunk();
  }
  if (lane == 31) carry_word = ld_word_guarded(d.base, s0 - 4, d.lo, d.hi);
  if (lane == 0) nsw = ld_word_guarded(d.base, s0 + sb, d.lo, d.hi);
  return step_errors<kPos, true>(d, v, cstep, lane, carry_word, nsw, first_i, was_ascii);
}

// K1.  One CTA of kK1Threads (32 warps) per SM; CTA c owns the steps
// c, c + G, c + 2G, ... (G = grid size), so at any moment the grid sweeps one
// window of ~G x 32 x 4 KiB, which keeps DRAM pages open.  Inside the CTA the
// warps take those steps from a shared-memory ticket counter: warp w starts
// with the CTA's step w, then each ticket t is the CTA's step 32 + t.  The
// SM's warp scheduler favours older warps strongly (with four static 8-warp
// CTAs per SM the oldest finished its equal share at 100 us of a 172 us C1
// launch, the youngest at 169 us; scripts/probes/k1_timeline.py), so static
// shares leave the SM running on a few warps for the last ~15 % of a launch;
// with the shared pool every warp of the SM stays busy until the pool is dry.
// A warp asks for its next ticket when it starts a step, so the shared
// atomic's latency hides behind the step.
// Each warp's steps increase, so a lane's first flagged step is recorded
// once (kTrack): the chunk index of the step's first chunk goes to
// *first_step (atomicMin, one elected lane of those that saw it), and the
// minimum over lanes and warps is the step holding the stream's first
// flagged chunk.
__device__ __forceinline__ void note_first_step(unsigned long long* first_step, int64_t cstep) {
  const unsigned m = __activemask();
  if ((int)(threadIdx.x & 31) == __ffs(m) - 1) atomicMin(first_step, (unsigned long long)cstep);
}

// Lane 0 takes the next ticket of the CTA's step pool (a predicated
// atom.shared: the compiler's warp-aggregated atomicAdd -- ballot, popc,
// leader election and convergence barriers -- cost ~40 instructions per step,
// 9 % of K1's; profiles/r02_ncu_k_validate_source.txt).
__device__ __forceinline__ unsigned take_ticket(unsigned pool_addr, int lane, unsigned keep) {
  unsigned t = keep;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.eq.s32 p, %1, 0;\n\t@p atom.shared.add.u32 %0, [%2], 1;\n\t}"
      : "+r"(t)
      : "r"(lane), "r"(pool_addr)
      : "memory");
  return t;
}

#ifdef U8V_K2P_SKELETON
// DEVELOPMENT (tools/kvar.sh builds only): the memory traffic of a pooled K2
// -- per step, the step's first-record index from a step table (with the
// data), then the record starts of the step (after the chunk math), and with
// U8V_K2P_SKELETON >= 2 the 8 bytes around each start -- folded into the
// flag so nothing is dropped.  scripts/probes/k2p_skeleton.py.
__device__ const unsigned* g_k2p_table;
__device__ const uint64_t* g_k2p_offsets;
__device__ unsigned g_k2p_n;
extern "C" int u8v_k2p_set(const unsigned* table, const uint64_t* offsets, unsigned n) {
  cudaMemcpyToSymbol(g_k2p_table, &table, sizeof(table));
  cudaMemcpyToSymbol(g_k2p_offsets, &offsets, sizeof(offsets));
  return (int)cudaMemcpyToSymbol(g_k2p_n, &n, sizeof(n));
}
#endif

template <bool kTrack>
__device__ __forceinline__ void sweep(const StreamDesc& d, uint32_t* __restrict__ flag) {
  __shared__ unsigned s_ticket;
  __shared__ unsigned s_zero[32];
  if (threadIdx.x == 0) s_ticket = 0;
  if (threadIdx.x < 32) s_zero[threadIdx.x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // The pool's shared address plus a per-lane zero read from shared memory:
  // ptxas cannot prove the address warp-uniform, so it does not wrap the
  // single-lane atom in its warp-aggregation sequence.
  const unsigned pool_addr = (unsigned)__cvta_generic_to_shared(&s_ticket) + s_zero[lane];
  const int64_t sb = kStepChunks * (int64_t)kChunkBytes;
  int64_t int_b, int_d;
  interior_steps(d, &int_b, &int_d);
  // Step indices fit 32 bits (make_desc: fewer than 2^31 steps, 8 TiB).
  const unsigned G = gridDim.x, nsteps = (unsigned)d.steps;
  const unsigned ib = (unsigned)int_b, id = (unsigned)int_d;
  const uint8_t* const base = d.base + d.c_begin * kChunkBytes;

  uint32_t acc = 0;
  bool was_ascii = true;  // try the vote on the first step
  bool noted = false;     // kTrack: this lane has recorded its first flagged step
  int unused = kU;
  unsigned step = blockIdx.x + G * (threadIdx.x >> 5);
  unsigned next = 0;
  if (step < nsteps) next = take_ticket(pool_addr, lane, next);
  while (step < nsteps) {
    uint32_t e;
    if (step >= ib && step < id) {
      const uint8_t* p = base + (int64_t)step * sb;
      Chunk v[kU];
#pragma unroll
      for (int i = 0; i < kU; ++i) v[i] = ld_chunk(p + ((i >> 1) * 64 + 2 * lane + (i & 1)) * kChunkBytes);
      uint32_t carry_word = 0, nsw = 0;
      ld_word_if(lane == 31, p - 4, carry_word);
      ld_word_if(lane == 0, p + sb, nsw);
#ifdef U8V_K2P_SKELETON
      const unsigned t0 = __ldg(g_k2p_table + step), t1 = __ldg(g_k2p_table + step + 1);
#endif
      e = step_errors_pairs(d, v, lane, carry_word, nsw, was_ascii);
#ifdef U8V_K2P_SKELETON
      const unsigned r = t0 + lane;
      if (r <= t1 && r <= g_k2p_n) {
        const uint64_t o = __ldg(g_k2p_offsets + r);
#if U8V_K2P_SKELETON >= 2
        const uint8_t* q = d.base + d.off32 + o;
        uint32_t a = 0, b = 0;
        if (o >= 4) a = *(const uint32_t*)((uintptr_t)(q - 4) & ~(uintptr_t)3);
        b = *(const uint32_t*)((uintptr_t)q & ~(uintptr_t)3);
        e |= (a & b) == 0xFFFFFFFFu ? 0x80000000u : 0u;
#endif
        e |= (uint32_t)(o >> 62);
      }
#endif
    } else {
      e = any_step_errors<false>(d, step, false, lane, unused, was_ascii);
    }
    acc |= e;
    if (kTrack && e != 0u && !noted) {
      noted = true;
      note_first_step(d.first_step, d.c_begin + (int64_t)step * kStepChunks);
    }
    const unsigned t = __shfl_sync(0xFFFFFFFFu, next, 0);
    step = blockIdx.x + G * (kK1Warps + t);
    if (step < nsteps) next = take_ticket(pool_addr, lane, next);
  }
  const unsigned any = __reduce_or_sync(0xFFFFFFFFu, acc);
  if (lane == 0 && any) {
    if (d.flag_store)
      *(volatile uint32_t*)flag = 1u;  // host-mapped word: a store, no PCIe atomic
    else
      atomicOr(flag, 1u);
    // P2P combine (comm.cu): the error also goes straight to every other
    // rank's flag word over NVLink, so the 4-byte allreduce(MAX) costs
    // nothing on valid input.
    for (int r = 0; r < d.n_peers; ++r) atomicOr(d.peer_flags[r], 1u);
  }
}

#ifdef U8V_TIMELINE
// DEVELOPMENT (tools/kvar.sh builds only): per-warp start/end %globaltimer
// and SM id of K1, to measure the launch ramp and the drain.
__device__ unsigned long long* g_timeline;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

__global__ void __launch_bounds__(kK1Threads, 1) k_validate(StreamDesc d, uint32_t* __restrict__ flag) {
#ifdef U8V_TIMELINE
  const unsigned long long t_start = gtimer();
#endif
  // Dependents (a following K1 launched with PDL, see launch_k1) may start
  // as soon as every CTA of this grid has started.
  asm volatile("griddepcontrol.launch_dependents;");
  sweep<false>(d, flag);
#ifdef U8V_TIMELINE
  if ((threadIdx.x & 31) == 0 && g_timeline != nullptr) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const int64_t w = ((int64_t)blockIdx.x * kK1Threads + threadIdx.x) >> 5;
    g_timeline[3 * w] = t_start;
    g_timeline[3 * w + 1] = gtimer();
    g_timeline[3 * w + 2] = smid;
  }
#endif
}

// K1 for a stream-session feed (launch_validate_piece): the piece's own
// lanes, then the edge thread -- which reads the carry the previous feed
// wrote -- waits for that feed, after its own share of the sweep, so no
// CTA's sweep waits behind the previous piece.  (A separate entry keeps the
// session code out of k_validate.)
__global__ void __launch_bounds__(kK1Threads, 1) k_validate_piece(StreamDesc d, uint32_t* __restrict__ flag) {
  asm volatile("griddepcontrol.launch_dependents;");
  sweep<false>(d, flag);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    stream_edge_piece(d.session, d.base + d.off32, (uint64_t)(d.hi - d.lo), 0);
  }
}

// K1 for the verdict path: also records the first flagged step
// (d.first_step), so an invalid stream needs no second pass -- k_locate_step
// recomputes that one step and decodes the window around its first flagged
// chunk.
__global__ void __launch_bounds__(kK1Threads, 1) k_validate_track(StreamDesc d, uint32_t* __restrict__ flag) {
  asm volatile("griddepcontrol.launch_dependents;");
  sweep<true>(d, flag);
}

// K3: one warp recomputes the step K1 recorded as the first flagged one
// (every lane range of the stream, masked loads), takes its first flagged
// chunk (chunks ordered (i, lane)), and lane 0 decodes the window around it.
// Lane flags are a function of the bytes alone, so the step recomputed over
// the stream's whole lane range flags the same chunks K1 (or a pipeline
// piece of it) did, and no chunk before it is flagged.
__global__ void k_locate_step(StreamDesc d, uint64_t n, const unsigned long long* __restrict__ first_step,
                              unsigned long long* __restrict__ out_offset, int* __restrict__ out_kind) {
  const int lane = threadIdx.x & 31;
  const unsigned long long cs = *first_step;
  StreamDesc w = d;
  w.c_begin = (int64_t)cs;
  int first_i = kU;
  bool was_ascii = false;
  any_step_errors<true>(w, 0, false, lane, first_i, was_ascii);
  unsigned long long m = first_i < kU ? cs + (unsigned long long)(lane + 32 * first_i) : ~0ull;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xFFFFFFFFu, m, o);
    m = t < m ? t : m;
  }
  if (lane != 0) return;
  if (m == ~0ull) {  // no flagged chunk (cannot happen after a flagged K1)
    *out_kind = -1;
    *out_offset = ~0ull;
    return;
  }
  locate_chunk(d.base + d.off32, n, d.off32, d.L0 - d.off32, m, out_offset, out_kind);
}

// ---- K2L: batches of few, large records (C2) ------------------------------
// Same decomposition as K2 (batch.cu): the unbounded lane flags of the data
// buffer, each flagged lane attributed to its record unless it is one of
// the record's first three lanes or lies past the data, plus one boundary
// check per record start.  With few records (launch_batch dispatches here
// for <= kLargeMaxRecords records of >= 64 KiB on average) the sweep is K1's
// own: one 1024-thread CTA per SM drawing steps from a shared pool, no
// record cursor (C2 back to back over two copies: 51.4 -> 49.2 us against
// four static 8-warp CTAs per SM, tools/k2cmp.py).  A flagged step (rare: a
// few per invalid record) is attributed out of line.  A flagged lane whose
// four chunks lie inside one record settles that record directly; the
// others recompute the step in natural lane order and find each flagged
// lane's record by binary search over the offsets held in shared memory.

// Largest r in [-1, N] with s_off[r] <= q (s_off[-1] = -inf).
__device__ __forceinline__ int rec_of(const int64_t* s_off, int N, int64_t q) {
  int a = -1, b = N;  // s_off[a] <= q (a = -1: none), answer in [a, b]
  while (a < b) {
    const int m = (a + b + 1) >> 1;
    if (s_off[m] <= q) a = m;
    else b = m - 1;
  }
  return a;
}

__device__ __forceinline__ void attribute_large(const StreamDesc& d, int64_t cstep, uint32_t e_or,
                                                const int64_t* s_off, int N, uint8_t* verdicts) {
  const int lane = threadIdx.x & 31;
  const int64_t sb = kStepChunks * (int64_t)kChunkBytes;
  const int64_t s0 = cstep * kChunkBytes;
  const int64_t data_hi = s_off[N];
  // A flagged lane whose four chunks all lie inside one record r, past its
  // first three lanes and before the data end, settles r without knowing
  // which lane fired (the common case for large records).
  bool open = false;
  if (e_or) {
    const int64_t a = (cstep + lane) * kChunkBytes, z = (cstep + lane + 32 * (kU - 1) + 1) * kChunkBytes;
    const int r = rec_of(s_off, N, a);
    if (r >= 0 && r < N && a - s_off[r] >= 3 && z <= s_off[r + 1] && z <= data_hi)
      verdicts[r] = 0;
    else
      open = true;
  }
  if (!__any_sync(0xFFFFFFFFu, open)) return;
  // Otherwise the step's lane flags again, natural order (bit i = lane 32 c
  // + i), for the lanes still open.
  Chunk v[kU];
#pragma unroll
  for (int i = 0; i < kU; ++i) {
    const int64_t c = cstep + lane + 32 * i;
    v[i] = c <= d.c_end ? ld_chunk_masked(d.base, c, d.lo, d.hi) : zero_chunk();
  }
  uint32_t carry_word = 0, nsw = 0;
  if (lane == 31) carry_word = ld_word_guarded(d.base, s0 - 4, d.lo, d.hi);
  if (lane == 0) nsw = ld_word_guarded(d.base, s0 + sb, d.lo, d.hi);
  uint32_t e[kU];
#pragma unroll
  for (int i = 0; i < kU; ++i) {
    const uint32_t up =
        lane == 31 ? (i == 0 ? carry_word : v[i - 1].w[kChunkWords - 1]) : v[i].w[kChunkWords - 1];
    const uint32_t prev = __shfl_sync(0xFFFFFFFFu, up, (lane + 31) & 31);
    const uint32_t dn = lane == 0 ? (i + 1 < kU ? v[i + 1].w[0] : nsw) : v[i].w[0];
    const uint32_t next = __shfl_sync(0xFFFFFFFFu, dn, (lane + 1) & 31);
    const int64_t c = cstep + lane + 32 * i;
    uint32_t hi7;
    e[i] = c < d.c_end ? chunk_errors<true>(v[i], prev, next, d.k, c * kChunkBytes, d.L0, d.L1, &hi7) : 0u;
  }
  // Each flagged lane q goes to its record r; once r is marked invalid every
  // other flagged lane of r in the chunk is dropped with it.
#pragma unroll
  for (int i = 0; i < kU; ++i) {
    const int64_t c0 = (cstep + lane + 32 * i) * kChunkBytes;
    uint32_t m = open ? e[i] : 0u;
    while (m) {
      const int b = __ffs(m) - 1;
      const int64_t q = c0 + b;
      m &= m - 1;
      if (q >= data_hi) break;  // past the data: the boundary at data_hi settles it
      const int r = rec_of(s_off, N, q);
      if (r < 0 || q - s_off[r] < 3) continue;  // before the data / a record's first lanes
      verdicts[r] = 0;
      const int64_t end = s_off[r + 1] - c0;  // drop the rest of record r
      m = end >= 32 ? 0u : (end <= 0 ? m : (m & ~((1u << end) - 1u)));
    }
  }
}

constexpr int kK2LThreads = kK1Threads;
__global__ void __launch_bounds__(kK1Threads, 1)
    k_batch_large(StreamDesc d, const uint64_t* __restrict__ offsets, int N, uint8_t* __restrict__ verdicts) {
  extern __shared__ int64_t s_off[];  // start(r) in base coordinates, clamped to the data
  __shared__ unsigned s_ticket;
  __shared__ unsigned s_zero[32];
  const int64_t nb = d.hi - d.lo;
  for (int i = threadIdx.x; i <= N; i += blockDim.x) {
    const uint64_t o = __ldg(offsets + i);
    s_off[i] = d.off32 + (int64_t)(o < (uint64_t)nb ? o : (uint64_t)nb);
  }
  if (threadIdx.x == 0) s_ticket = 0;
  if (threadIdx.x < 32) s_zero[threadIdx.x] = 0;
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t)blockIdx.x * kK1Threads + threadIdx.x;
  if (g <= N) {
    const int64_t s = s_off[g], lo = s_off[0], hi = s_off[N];
    const int64_t a = g > 0 ? s_off[g - 1] : s, b = g < N ? s_off[g + 1] : s;
    uint64_t w8 = 0;
    for (int k = 0; k < 8; ++k) {
      const int64_t q = s - 4 + k;
      if (q >= lo && q < hi) w8 |= (uint64_t)d.base[q] << (8 * k);
    }
    int64_t ka = a - (s - 4), kb = b - (s - 4);
    ka = ka < 0 ? 0 : (ka > 4 ? 4 : ka);
    kb = kb < 4 ? 4 : (kb > 8 ? 8 : kb);
    const uint32_t f = u8v_boundary_errors(w8, (unsigned)ka, (unsigned)kb, d.k);
    if ((f & 1u) && g > 0) verdicts[g - 1] = 0;
    if ((f & 2u) && g < N) verdicts[g] = 0;
  }
  const unsigned pool_addr = (unsigned)__cvta_generic_to_shared(&s_ticket) + s_zero[lane];
  const int64_t sb = kStepChunks * (int64_t)kChunkBytes;
  int64_t int_b, int_d;
  interior_steps(d, &int_b, &int_d);
  const unsigned G = gridDim.x, nsteps = (unsigned)d.steps;
  const unsigned ib = (unsigned)int_b, id = (unsigned)int_d;
  const uint8_t* const base = d.base + d.c_begin * kChunkBytes;
  bool was_ascii = true;
  int unused = kU;
  unsigned step = blockIdx.x + G * (threadIdx.x >> 5);
  unsigned next = 0;
  if (step < nsteps) next = take_ticket(pool_addr, lane, next);
  while (step < nsteps) {
    uint32_t e;
    if (step >= ib && step < id) {
      const uint8_t* p = base + (int64_t)step * sb;
      Chunk v[kU];
#pragma unroll
      for (int i = 0; i < kU; ++i) v[i] = ld_chunk(p + (lane + 32 * i) * kChunkBytes);
      uint32_t carry_word = 0, nsw = 0;
      ld_word_if(lane == 31, p - 4, carry_word);
      ld_word_if(lane == 0, p + sb, nsw);
      e = step_errors<false, false>(d, v, 0, lane, carry_word, nsw, unused, was_ascii);
    } else {
      e = any_step_errors<false>(d, step, false, lane, unused, was_ascii);
    }
    if (__any_sync(0xFFFFFFFFu, e != 0u))
      attribute_large(d, d.c_begin + (int64_t)step * kStepChunks, e, s_off, N, verdicts);
    const unsigned t = __shfl_sync(0xFFFFFFFFu, next, 0);
    step = blockIdx.x + G * (kK1Warps + t);
    if (step < nsteps) next = take_ticket(pool_addr, lane, next);
  }
}
}  // namespace u8v

// ---- host-side launchers (called by capi.cu) ------------------------------
namespace u8v {

// Grid sizes from each kernel's occupancy, per device (queried once per
// device, thread-safe: ShardPool workers on different devices launch at the
// same time).
namespace {
struct DevInfo {
  int k1_ctas = 1;    // resident K1 CTAs (kK1Threads each) on the device
  int k2_warps = 1;   // resident K2 warps (batch.cu)
};
constexpr int kMaxDev = 64;
DevInfo g_info[kMaxDev];
std::once_flag g_info_once[kMaxDev];
}  // namespace

static int blocks_per_sm(const void* fn, int threads, size_t smem) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, threads, smem) != cudaSuccess) cudaGetLastError();
  return b < 1 ? 1 : b;
}

static const DevInfo& dev_info() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) dev = 0;
  std::call_once(g_info_once[dev], [dev] {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 1;
    DevInfo& i = g_info[dev];
    i.k1_ctas = sms * blocks_per_sm((const void*)k_validate, kK1Threads, 0);
    i.k2_warps = sms * batch_blocks_per_sm() * (batch_threads() / 32);
  });
  return g_info[dev];
}

int k2_resident_warps() { return dev_info().k2_warps; }

StreamDesc make_desc(const uint8_t* p, uint64_t n, uint64_t lane_lo, uint64_t lane_hi) {
  // Stream coordinates: byte i of the stream is p[i]; lanes [lane_lo,
  // lane_hi) are evaluated (lane_hi <= n + 3).  Chunk coordinates are
  // relative to the 32-byte aligned base below p.
  StreamDesc d;
  const uintptr_t up = (uintptr_t)p;
  const int64_t off = (int64_t)(up & (kChunkBytes - 1));
  d.base = (const uint8_t*)(up - (uintptr_t)off);
  d.lo = off;
  d.hi = off + (int64_t)n;
  d.off32 = off;
  d.k = u8v_make_consts();
  d.L0 = off + (int64_t)lane_lo;
  d.L1 = off + (int64_t)lane_hi;
  d.c_begin = d.L0 / kChunkBytes;
  d.c_end = (d.L1 + kChunkBytes - 1) / kChunkBytes;
  const int64_t chunks = d.c_end - d.c_begin;
  d.steps = (chunks + kStepChunks - 1) / kStepChunks;
  d.session = nullptr;
  d.first_step = nullptr;
  d.peer_flags = nullptr;
  d.n_peers = 0;
  d.flag_store = 0;
  return d;
}

// K1 grid: one CTA per SM, fewer for inputs of fewer steps (every CTA gets
// at least one step).
static unsigned k1_grid(const StreamDesc& d) {
  int64_t g = dev_info().k1_ctas;
  if (g > d.steps) g = d.steps;
  return (unsigned)(g < 1 ? 1 : g);
}

// Every K1 launch allows programmatic stream serialization (PDL), and every
// K1 grid triggers its dependents on entry: when K1 follows K1 on a stream,
// the next grid's CTAs take each SM as soon as the previous grid's CTA there
// retires, so one launch's ramp overlaps the other's drain.  This is safe
// because K1 consumes nothing a preceding K1 produces (both only OR into
// flags / atomicMin positions), and any other predecessor (a kernel that does
// not trigger early, a copy, a memset, an event wait) is waited for in full;
// by induction every K1 starts after the last non-K1 work before it on the
// stream has completed.  Successors that read K1's results are not launched
// with PDL and wait for it in full.
static void launch_k1(void (*kernel)(StreamDesc, uint32_t*), const StreamDesc& d, uint32_t* flag,
                      cudaStream_t st) {
  serve_quiesce();  // the grid holds one CTA per SM
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(k1_grid(d));
  cfg.blockDim = dim3(kK1Threads);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, d, flag);
}

void launch_validate(const StreamDesc& d, uint32_t* flag, cudaStream_t st) {
  if (d.steps <= 0) return;
  launch_k1(d.first_step ? k_validate_track : k_validate, d, flag, st);
}

void launch_validate_piece(const StreamDesc& d, uint32_t* flag, cudaStream_t st) {
  launch_k1(k_validate_piece, d, flag, st);
}

bool launch_batch_large(const uint8_t* data, uint64_t n, const uint64_t* d_offsets, uint64_t n_records,
                        uint8_t* d_verdicts, cudaStream_t st) {
  if (n_records == 0 || n_records > (uint64_t)kLargeMaxRecords || n / n_records < kLargeMinAvgBytes) return false;
  // Lanes [0, n) of the data buffer: lanes past offsets[N] are ignored and
  // the last record's end is settled by the boundary check at offsets[N].
  const StreamDesc d = make_desc(data, n, 0, n);
  int64_t blocks = k1_grid(d);
  const int64_t need = ((int64_t)n_records + kK2LThreads) / kK2LThreads;  // boundary threads: N + 1
  if (blocks < need) blocks = need;
  const size_t smem = (n_records + 1) * sizeof(int64_t);
  serve_quiesce();  // the grid holds one CTA per SM
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)blocks);
  cfg.blockDim = dim3(kK2LThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_batch_large, d, d_offsets, (int)n_records, d_verdicts);  // after k_init_verdicts
  return true;
}

#ifdef U8V_TIMELINE
extern "C" int u8v_timeline_set(unsigned long long* p) {
  return (int)cudaMemcpyToSymbol(g_timeline, &p, sizeof(p));
}
#endif

void launch_locate(const StreamDesc& d, uint64_t n, const unsigned long long* first_step,
                   unsigned long long* out_offset, int* out_kind, cudaStream_t st) {
  k_locate_step<<<1, 32, 0, st>>>(d, n, first_step, out_offset, out_kind);
}

}  // namespace u8v
