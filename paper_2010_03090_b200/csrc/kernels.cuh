// kernels.cuh -- shared declarations between the sm_100a kernels and capi.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "utf8v_state.h"
#include "utf8v_swar.h"

namespace u8v {

constexpr int kThreads = 256;              // K2/K2L: 8 warps per CTA
constexpr int kK1Threads = 1024;           // K1: one 32-warp CTA per SM
constexpr int kK1Warps = kK1Threads / 32;
// K1/K3 (validate.cu) and K2 (batch.cu): 32-byte lane chunks, one 256-bit
// LDG each; a warp step is 4 chunks per lane.
constexpr int kChunkBytes = 32;
constexpr int kChunkWords = kChunkBytes / 4;
constexpr int kU = 4;                      // chunks per lane per step
constexpr int kStepChunks = 32 * kU;       // 128 chunks = 4 KiB per warp step

// error_kind numbering of proj/include/utf8v/verdict.hpp:20-27.
enum { kHeaderBits = 0, kTooShort = 1, kTooLong = 2, kOverlong = 3, kTooLarge = 4, kSurrogate = 5 };

struct StreamDesc {
  const uint8_t* base;     // 32-byte aligned view of the stream
  int64_t lo, hi;          // valid bytes [lo, hi) relative to base; others read 0
  int64_t off32;           // stream byte 0 is base[off32]
  int64_t L0, L1;          // lanes evaluated: [L0, L1) relative to base
  int64_t c_begin, c_end;  // chunks evaluated: [c_begin, c_end)
  int64_t steps;           // ceil((c_end - c_begin) / kStepChunks)
  u8v_consts k;  // runtime multipliers (FMA-pipe routing, utf8v_swar.h)
  uint32_t* session;  // a stream-session piece (launch_validate_piece): K1's first
                      // thread also runs the edge of this piece (stream_edge.cuh)
                      // on session[0..1]
  unsigned long long* first_step;  // non-null: K1 records its first flagged step
                                   // there (atomicMin of the step's first chunk)
  uint32_t* const* peer_flags;     // n_peers device pointers (other GPUs' flag words,
  int n_peers;                     // NVLink peer memory): a warp that finds an
                                   // error also ORs 1 into each (comm.cu, P2P combine)
  int flag_store;                  // nonzero: the flag is mapped host memory (the
                                   // small-input path) and takes a plain store of 1
};

// Resident K2 warps on the current device (cached per device).
int k2_resident_warps();
// batch.cu: k_batch's resident CTAs per SM (occupancy query).
int batch_blocks_per_sm();
int batch_threads();
StreamDesc make_desc(const uint8_t* p, uint64_t n, uint64_t lane_lo, uint64_t lane_hi);
void launch_validate(const StreamDesc& d, uint32_t* flag, cudaStream_t st);
// A stream-session piece (d.session set, d.steps > 0) on the session's own
// stream: K1 launched with programmatic stream serialization, so consecutive
// feeds overlap; the edge thread waits for the previous feed (validate.cu).
void launch_validate_piece(const StreamDesc& d, uint32_t* flag, cudaStream_t st);
// After K1 with d.first_step set flagged the stream: the first error's
// (offset, kind) from the recorded step (one warp).
void launch_locate(const StreamDesc& d, uint64_t n, const unsigned long long* first_step,
                   unsigned long long* out_offset, int* out_kind, cudaStream_t st);

// batch.cu
// Writes d_verdicts[] fully: an initialisation kernel sets them to 1, then K2
// (or K2L) stores 0 for failing records.  Asynchronous: the kernel reads
// offsets[0] and offsets[n_records] itself (clamped to the n data bytes).
// states = true: K2 in segment-state mode -- d_verdicts[r] = 1 iff none of
// record r's interior lanes [start+3, end-1) is flagged (no boundary checks;
// always K2, never K2L).
void launch_batch(const uint8_t* data, uint64_t n, const uint64_t* d_offsets, uint64_t n_records,
                  uint8_t* d_verdicts, cudaStream_t st, bool states = false);
// Segment states (utf8v_state.h) of the records from launch_batch(states) output.
void launch_record_states(const uint8_t* data, uint64_t n, const uint64_t* d_offsets, uint64_t n_records,
                          const uint8_t* d_clean, u8v_state* d_out, cudaStream_t st);
// *d_out = the in-order combine of d_in[0 .. count) (one CTA).
void launch_states_reduce(const u8v_state* d_in, uint64_t count, u8v_state* d_out, cudaStream_t st);

// validate.cu: K2L, the batch kernel for few, large records (<= 2048
// records of >= 64 KiB on average): K1's sweep + out-of-line attribution.
// Returns false (nothing launched) outside that range; same contract as
// launch_batch otherwise.
constexpr int kLargeMaxRecords = 2048;
constexpr uint64_t kLargeMinAvgBytes = 64 << 10;
bool launch_batch_large(const uint8_t* data, uint64_t n, const uint64_t* d_offsets, uint64_t n_records,
                        uint8_t* d_verdicts, cudaStream_t st);

// stream.cu: d_state[0] = carry, d_state[1] = error flag (utf8v_stream.h).
void launch_stream_edge(uint32_t* d_state, const uint8_t* d_piece, uint64_t n, int finish,
                        cudaStream_t st);

// lanes.cu (lane entry points of the lookup_backend table, width kLaneWidth)
constexpr int kLaneWidth = 64;
void set_tables(const uint8_t t1[16], const uint8_t t2[16], const uint8_t t3[16]);
void launch_classify_lanes(const uint8_t* in, const uint8_t* prev, uint8_t* out, int mode,
                           cudaStream_t st);
void launch_ops_self_test(uint64_t seed, int* result, cudaStream_t st);


}  // namespace u8v
