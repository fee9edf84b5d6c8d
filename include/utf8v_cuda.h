/*
 * utf8v_cuda.h -- the drop-in C-ABI boundary of the B200 Lookup validator
 * (libutf8v_cuda.so).
 *
 * It replaces, for the Lookup path of the reference `utf8v` library, the
 * backend function-pointer table and its dispatch:
 *   struct lookup_backend          proj/include/utf8v/lookup.hpp:18-28
 *   lookup_backends / find_...     proj/include/utf8v/lookup.hpp:30-35, proj/src/lookup.cpp:16-37
 *   validate_lookup[_fallback]     proj/include/utf8v/lookup.hpp:37-41, proj/src/lookup.cpp:39-45
 * and adds the position and record-batch variants the reference obtains by
 * re-running oracle_validate (proj/src/oracle.cpp:10-44; the CLI failure path
 * proj/tools/main.cpp:129-147) or by looping validate_lookup per record.
 * The C++ API of include/utf8v/lookup.hpp (same names as the reference) is a
 * thin layer over these entry points; INTEGRATION.md shows the binding.
 *
 * Host input to the synchronous entry points crosses PCIe in pieces through
 * a bounded ring of device slots (at most 4 x (32 MiB + 32 B) of HBM per
 * host thread and device, whatever n is); each piece is validated as soon as
 * it lands.  Record batches from host memory are staged whole.
 *
 * Conventions:
 *   - plain pointers and sizes only; every pointer is borrowed for the call;
 *   - return an int status: UTF8V_OK, or a mapped CUDA/argument error -- never
 *     throw, never abort; invalid UTF-8 is a normal result, not an error;
 *   - n == 0 (with any pointer, NULL included) is valid text;
 *   - `is_device` != 0: the pointer is device memory of the current device;
 *     0: host memory (pinned or pageable; copied over PCIe inside the call);
 *   - re-entrant: one lazily initialised context per device, per-thread
 *     streams and scratch; callable concurrently from many host threads;
 *   - there is no CPU fallback: without a usable CUDA device every compute
 *     entry point returns UTF8V_ERR_NO_DEVICE.
 */
#ifndef UTF8V_CUDA_H
#define UTF8V_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UTF8V_OK 0
#define UTF8V_ERR_CUDA 1
#define UTF8V_ERR_ARG 2
#define UTF8V_ERR_NO_DEVICE 3
#define UTF8V_ERR_NCCL 4

/* Width in bytes of the lane entry points below (lookup_backend::width;
 * >= 32 so the roster stays widest-first, proj/tests/test_lookup.cpp:41-42). */
#define UTF8V_CUDA_WIDTH 64

/* ABI version (bumped on any signature or contract change).
 *   1  first round-1 interface
 *   2  streaming session, utf8v_cuda_validate_sharded; the async batch entry
 *      point reads its first/last offsets on the device (no host sync)
 *   3  device input to the synchronous entry points (is_device = 1) and to
 *      utf8v_cuda_stream_feed is ordered after all work issued before the
 *      call to the legacy default stream, like a synchronous cudaMemcpy;
 *      writes made on a non-blocking stream must be synchronised by the
 *      caller
 *   4  utf8v_cuda_validate_verdict_lanes (first error of a shard)
 *   5  multi-GPU combine in the native layer (NCCL comms, P2P flags);
 *      utf8v_cuda_validate_batch_async lost its unused d_scratch argument
 *      (utf8v_cuda_batch_scratch_bytes removed); host input crosses PCIe
 *      through a bounded device ring; utf8v_cuda_release_thread_resources;
 *      device stream pieces are ordered before later legacy-stream work;
 *      composable segment states (utf8v_state)
 *   6  the small-call server answers host inputs <= UTF8V_CUDA_SERVE_MAX
 *      bytes and small host batches (utf8v_cuda_serve_stats) */
int utf8v_cuda_abi_version(void);

/* Human-readable text of the last error on this thread ("" if none). */
const char* utf8v_cuda_last_error(void);

/* lookup_backend::validate (proj/include/utf8v/lookup.hpp:21) and
 * validate_lookup (proj/src/lookup.cpp:39-41): *out_valid = 1 iff p[0..n)
 * is valid UTF-8.  Host input is streamed to the GPU in pieces, each piece
 * validated as soon as it lands (copy and compute overlap). */
int utf8v_cuda_validate(const uint8_t* p, size_t n, int is_device, uint8_t* out_valid);

/* Verdict with the first error, bit-exact with oracle_validate
 * (proj/src/oracle.cpp:10-44): *out_valid, and when 0, *out_offset (lead byte
 * of the offending sequence) and *out_kind (error_kind numbering of
 * proj/include/utf8v/verdict.hpp:20-27). */
int utf8v_cuda_validate_verdict(const uint8_t* p, size_t n, int is_device, uint8_t* out_valid,
                                uint64_t* out_offset, int* out_kind);

/* The verdict of lanes [lane_lo, lane_hi) of p[0..n) (lane_hi <= n + 3; lane
 * i reads bytes i-3 .. i+1, zero outside [0, n)): the shard form of
 * utf8v_cuda_validate_verdict for a stream split over GPUs.
 * *out_valid = 1 iff none of the lanes is flagged; otherwise *out_offset /
 * *out_kind are decoded from the bytes around the first flagged 32-byte
 * chunk, in p's coordinates.  The result is the stream's first error when
 * everything before that error is valid text, when p holds at least 6 bytes
 * before lane_lo (or lane_lo < 6 and p starts the stream), and when it holds
 * 3 bytes past the error's lead (sharding.py: a 16-byte head and a 3-byte
 * tail).  Ranks combine their (offset, kind) with one allreduce(MIN). */
int utf8v_cuda_validate_verdict_lanes(const uint8_t* p, uint64_t n, uint64_t lane_lo, uint64_t lane_hi,
                                      int is_device, uint8_t* out_valid, uint64_t* out_offset,
                                      int* out_kind);

/* Records p[offsets[r] .. offsets[r+1]) for r < n_records, each validated as
 * its own stream (the reference loops validate_lookup per record); writes
 * verdicts[r] = 1 (valid) / 0 (invalid).  offsets: n_records+1 non-decreasing
 * uint64 (CSR), offsets[n_records] <= n.  is_device applies to data, offsets
 * and verdicts alike. */
int utf8v_cuda_validate_batch(const uint8_t* data, size_t n, const uint64_t* offsets,
                              size_t n_records, int is_device, uint8_t* verdicts);

/* Lane entry points over UTF8V_CUDA_WIDTH host bytes (lookup_backend
 * ::classify_lanes / length_error_lanes / incomplete_lanes, lookup.hpp:22-26;
 * proj/src/lookup_backend_detail.hpp:16-43), computed on the GPU. */
int utf8v_cuda_classify_lanes(const uint8_t* input, const uint8_t* previous, uint8_t* out);
int utf8v_cuda_length_error_lanes(const uint8_t* input, const uint8_t* previous, uint8_t* out);
int utf8v_cuda_incomplete_lanes(const uint8_t* input, uint8_t* out);

/* lookup_backend::ops_self_test (lookup.hpp:27; lookup_kernel.hpp:139-216):
 * *out_ok = 1 iff every SWAR vector operation matches plain arithmetic. */
int utf8v_cuda_ops_self_test(uint64_t seed, int* out_ok);

/* ---- device-resident, asynchronous entry points (no host sync) ---------
 * For callers that own device memory and streams (the bench, the multi-GPU
 * shard layer).  `stream` is a cudaStream_t (NULL = legacy default stream).
 * d_flag is a device uint32 the kernels OR a nonzero value into when an
 * error is found; the caller zeroes it and reads it back. */

/* Lanes [lane_lo, lane_hi) of the stream d_p[0..n) (zero outside), lane_hi
 * <= n + 3.  Lane j reads bytes j-3 .. j+1.  Whole stream: lane_lo = 0,
 * lane_hi = n + 3.  A shard [s, e) of a larger stream passes its 3 (or up to
 * 16) preceding bytes as the head of d_p and the 1 byte after it as the tail:
 * lane_lo = head length, lane_hi = head length + (e - s), n = head + (e - s)
 * + 1 (the last shard: no tail byte, lane_hi = n + 3). */
int utf8v_cuda_validate_lanes_async(const uint8_t* d_p, uint64_t n, uint64_t lane_lo,
                                    uint64_t lane_hi, uint32_t* d_flag, void* stream);

/* Synchronous lane range over host or device bytes (the shard entry point of
 * the multi-GPU layer, paper_2010_03090_b200/sharding.py): *out_flag = 0
 * when lanes [lane_lo, lane_hi) hold no error, nonzero otherwise.  Same lane
 * contract as utf8v_cuda_validate_lanes_async. */
int utf8v_cuda_validate_lanes(const uint8_t* p, uint64_t n, uint64_t lane_lo, uint64_t lane_hi,
                              int is_device, uint32_t* out_flag);

/* One process, several GPUs (C4): host input p[0..n) is cut
 * into n_gpus byte-range shards (as paper_2010_03090_b200/sharding.py: a
 * look-back head of up to 16 bytes and a 1-byte lookahead tail per shard),
 * each copied over its GPU's own PCIe link and validated there by one host
 * thread per GPU; the 4-byte flags are combined on the host (no collective
 * is needed inside one process).  Shard g runs on visible device g % count
 * (n_gpus may exceed the device count: shards then share devices).  Device
 * input (is_device != 0) and shards under 1 MiB are validated on the
 * current GPU. */
int utf8v_cuda_validate_sharded(const uint8_t* p, size_t n, int n_gpus, int is_device,
                                uint8_t* out_valid);

/* Batch on device memory; d_verdicts is written fully (1/0 per record).
 * Fully asynchronous (no host round trip): the kernel reads d_offsets[0] and
 * d_offsets[n_records] itself.  Offsets must be non-decreasing with
 * d_offsets[n_records] <= n; malformed device offsets give unspecified
 * verdicts but never an access outside d_data[0..n) (the synchronous host
 * entry point, utf8v_cuda_validate_batch with is_device = 0, checks them).
 * No scratch memory is needed. */
int utf8v_cuda_validate_batch_async(const uint8_t* d_data, uint64_t n, const uint64_t* d_offsets,
                                    uint64_t n_records, uint8_t* d_verdicts, void* stream);

/* ---- streaming: one stream validated in pieces -------------------------
 * The device-side restatement of threading fsm_state through
 * validate_fsm(piece, state) (proj/include/utf8v/fsm.hpp:15-20; the
 * streaming non-goal of SPEC.md:312): feed pieces in order, finish() gives
 * the verdict of their concatenation.  The session carries 4 bytes and an
 * error flag on the device; every piece is validated in place (device
 * pieces are not copied) by one K1 launch whose first thread also evaluates
 * the <= 4 lanes straddling the previous piece (csrc/stream_edge.cuh).  Pieces may have any length,
 * including 0.  A device piece is read asynchronously on the session's own
 * stream (consecutive feeds overlap): it must stay valid and unmodified until
 * finish() returns (the Python LookupStream keeps a reference to every
 * device piece until then).  Host pieces are consumed before feed returns.
 * finish() resets the session.  feed and finish leave the caller's current
 * device unchanged. */
typedef struct utf8v_cuda_stream utf8v_cuda_stream;
int utf8v_cuda_stream_create(utf8v_cuda_stream** out);
int utf8v_cuda_stream_feed(utf8v_cuda_stream* s, const uint8_t* p, size_t n, int is_device);
int utf8v_cuda_stream_finish(utf8v_cuda_stream* s, uint8_t* out_valid);
uint64_t utf8v_cuda_stream_bytes(const utf8v_cuda_stream* s);
void utf8v_cuda_stream_destroy(utf8v_cuda_stream* s);

/* ---- composable segment states -----------------------
 * The Lookup counterpart of the reference's fsm_state threading
 * (proj/include/utf8v/fsm.hpp:15-20: "a stream can be validated in segments
 * by threading the returned state"), made order-free: a segment validated on
 * its own -- any device, any time -- yields a 24-byte state, and states
 * merge with an associative combine (csrc/utf8v_state.h states the rule).
 * The stream [0, n) is valid iff utf8v_state_valid() of the in-order combine
 * of its segments' states.  Empty segments are the identity. */
typedef struct utf8v_state {
  uint64_t len;      /* segment length */
  uint32_t flag;     /* nonzero: an interior lane [3, len-1) of the segment is flagged */
  uint8_t head[4];   /* first min(len, 4) bytes, zero after */
  uint8_t tail[4];   /* last min(len, 4) bytes, right-aligned, zero before */
  uint32_t reserved;
} utf8v_state;

/* Host, pure: *out = a followed by b (out may alias a or b). */
int utf8v_state_combine(const utf8v_state* a, const utf8v_state* b, utf8v_state* out);
/* Host, pure: 1 iff the stream whose whole state is *s is valid UTF-8. */
int utf8v_state_valid(const utf8v_state* s);
/* The state of one segment p[0..n) (host or device bytes; K1 over its
 * interior lanes). */
int utf8v_cuda_segment_state(const uint8_t* p, size_t n, int is_device, utf8v_state* out);
/* Per-record states of a CSR batch (records as in utf8v_cuda_validate_batch,
 * each a segment): K2 in state mode + one pass over the record edges.
 * Device form asynchronous on `stream` (d_states: n_records entries). */
int utf8v_cuda_batch_states_async(const uint8_t* d_data, uint64_t n, const uint64_t* d_offsets,
                                  uint64_t n_records, utf8v_state* d_states, void* stream);
int utf8v_cuda_batch_states(const uint8_t* data, size_t n, const uint64_t* offsets, size_t n_records,
                            int is_device, utf8v_state* states);
/* *d_out = the in-order combine of d_states[0 .. count) on the device (one
 * CTA; asynchronous on `stream`). */
int utf8v_cuda_states_reduce_async(const utf8v_state* d_states, uint64_t count, utf8v_state* d_out,
                                   void* stream);

/* ---- multi-GPU combine in the native layer (comm.cu) -------
 * A stream sharded over ranks (one GPU each) is valid iff no rank's lanes
 * hold an error: the rank flags combine with one 4-byte allreduce(MAX), the
 * first error with one 8-byte allreduce(MIN) of offset*8+kind.  The shard
 * plan (heads, tails, lanes) is sharding.py's; each rank passes its own
 * bytes and lane range with the contract of utf8v_cuda_validate_lanes.
 *
 * NCCL form.  libnccl.so.2 is loaded on first use (dlopen); without it
 * these entry points return UTF8V_ERR_NCCL, as do NCCL failures.  A comm is
 * bound to the device current at creation and used by one host thread at a
 * time. */
#define UTF8V_COMM_ID_BYTES 128
typedef struct utf8v_cuda_comm utf8v_cuda_comm;

/* ncclGetUniqueId: rank 0 creates it, the caller's bootstrap (MPI,
 * torch.distributed, a file) hands the 128 bytes to every rank. */
int utf8v_cuda_comm_unique_id(uint8_t* out_id);
/* ncclCommInitRank on the current device (collective over the nranks). */
int utf8v_cuda_comm_init_rank(const uint8_t* id, int nranks, int rank, utf8v_cuda_comm** out);
/* One process driving several GPUs (ncclCommInitAll): out_comms[i] is rank
 * i on devices[i] (devices NULL: 0 .. ndev-1). */
int utf8v_cuda_comm_init_all(int ndev, const int* devices, utf8v_cuda_comm** out_comms);
void utf8v_cuda_comm_destroy(utf8v_cuda_comm* c);

/* K1 over this rank's lanes of d_p[0..n) on `stream`, OR-ing into
 * *d_local_flag (zeroed by the caller), then ncclAllReduce(MAX) of that word
 * into *d_global_flag on the same stream: once the stream's work completes
 * every rank's *d_global_flag is 0 iff the whole stream is valid.  No host
 * synchronisation. */
int utf8v_cuda_validate_shard_allreduce_async(utf8v_cuda_comm* c, const uint8_t* d_p, uint64_t n,
                                              uint64_t lane_lo, uint64_t lane_hi, uint32_t* d_local_flag,
                                              uint32_t* d_global_flag, void* stream);
/* Synchronous, host (pipelined H2D) or device shard: *out_valid = verdict of
 * the whole stream, on every rank. */
int utf8v_cuda_validate_shard_allreduce(utf8v_cuda_comm* c, const uint8_t* p, uint64_t n, uint64_t lane_lo,
                                        uint64_t lane_hi, int is_device, uint8_t* out_valid);
/* The whole stream's first error (oracle_validate, proj/src/oracle.cpp:10-44)
 * on every rank: this rank's utf8v_cuda_validate_verdict_lanes, shifted by
 * p_stream_offset (the stream offset of p[0]), combined by one 8-byte
 * allreduce(MIN).  Exact under the conditions stated for
 * utf8v_cuda_validate_verdict_lanes (sharding.py's 16-byte head, 3-byte tail). */
int utf8v_cuda_verdict_shard_allreduce(utf8v_cuda_comm* c, const uint8_t* p, uint64_t n, uint64_t lane_lo,
                                       uint64_t lane_hi, uint64_t p_stream_offset, int is_device,
                                       uint8_t* out_valid, uint64_t* out_offset, int* out_kind);
/* One process, device-resident shards on several GPUs: comms from one
 * utf8v_cuda_comm_init_all; shard g (d_shards[g], shard_bytes[g] bytes, lanes
 * [lane_lo[g], lane_hi[g])) lives on comms[g]'s device.  K1 on every device,
 * then one grouped 4-byte ncclAllReduce(MAX); *out_valid = the stream's
 * verdict. */
int utf8v_cuda_validate_sharded_device(utf8v_cuda_comm* const* comms, int n_gpus, const uint8_t* const* d_shards,
                                       const uint64_t* shard_bytes, const uint64_t* lane_lo,
                                       const uint64_t* lane_hi, uint8_t* out_valid);

/* P2P form: the combine folded into K1.  Every rank owns one flag word; the
 * words are mapped into every other rank with CUDA IPC (NVLink peer
 * memory), and a K1 warp that finds an error ORs 1 into all of them -- on
 * valid input nothing crosses NVLink and no collective is launched.  Each
 * rank: create (-> its 64-byte IPC handle), gather all ranks' handles with
 * the bootstrap, connect; then per stream: reset, validate_async, the
 * caller's barrier after its stream completes, read.  Ranks may share a
 * GPU (separate processes). */
#define UTF8V_P2P_HANDLE_BYTES 64
typedef struct utf8v_cuda_p2p utf8v_cuda_p2p;
int utf8v_cuda_p2p_create(utf8v_cuda_p2p** out, uint8_t* out_handle);
/* handles: nranks x UTF8V_P2P_HANDLE_BYTES, rank order. */
int utf8v_cuda_p2p_connect(utf8v_cuda_p2p* g, const uint8_t* handles, int nranks, int rank);
/* K1 over this rank's lanes on `stream`; errors reach every rank's word. */
int utf8v_cuda_p2p_validate_async(utf8v_cuda_p2p* g, const uint8_t* d_p, uint64_t n, uint64_t lane_lo,
                                  uint64_t lane_hi, void* stream);
/* This rank's flag word (device pointer). */
uint32_t* utf8v_cuda_p2p_flag(utf8v_cuda_p2p* g);
/* Synchronous read / zeroing of this rank's word (0 = no rank saw an error,
 * once every rank's work has completed). */
int utf8v_cuda_p2p_read(utf8v_cuda_p2p* g, uint32_t* out_flag);
int utf8v_cuda_p2p_reset(utf8v_cuda_p2p* g);
void utf8v_cuda_p2p_destroy(utf8v_cuda_p2p* g);

/* Frees this thread's per-device resources (streams, the bounded host-input
 * ring of 4 x (32 MiB + 32 B) device bytes, pinned staging, the batch stage,
 * the small-call server and its mailbox), the unused batch scratch the
 * library's per-device memory pools keep mapped, and the resources of the
 * library's persistent shard workers
 * (utf8v_cuda_validate_sharded); the next call recreates what it needs.
 * A thread's resources are also freed when it exits. */
void utf8v_cuda_release_thread_resources(void);

/* Number of kernel launches the last call on this thread enqueued. */
int utf8v_cuda_last_launch_count(void);

/* The small-call server (host inputs of at most UTF8V_CUDA_SERVE_MAX bytes to
 * utf8v_cuda_validate / _validate_verdict / _validate_lanes /
 * _validate_verdict_lanes): one resident CTA answers requests posted in mapped
 * pinned memory, without a launch or a stream synchronisation per call.  It
 * exits after UTF8V_CUDA_SERVE_IDLE_US (default 100) microseconds without a
 * request, and before any other grid-wide launch of this library;
 * UTF8V_CUDA_SERVE=0 turns it off.  Replaces nothing in the reference: it is
 * the latency path of validate_lookup (proj/src/lookup.cpp:39-41) on short
 * buffers.  Diagnostics: server launches and requests served on this thread
 * and the current device since the thread's resources were created. */
#define UTF8V_CUDA_SERVE_MAX 65536
int utf8v_cuda_serve_stats(uint64_t* out_launches, uint64_t* out_requests);

#ifdef __cplusplus
}
#endif

#endif
