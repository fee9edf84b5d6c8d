// utf8v/lookup.hpp -- the reference's Lookup backend API
// (proj/include/utf8v/lookup.hpp:18-41), served by the B200 "cuda" backend.
//
// Same struct, same functions, same meaning:
//   * lookup_backend: name, width, validate, three lane entry points, self
//     test.  The roster holds one backend, "cuda" (width 64); there is no CPU
//     backend in this library -- a CPU fallback would void the drop-in's
//     guarantees, so validate_lookup_fallback() exists for source
//     compatibility and runs the same device kernels.
//   * validate functions return false for invalid UTF-8; a CUDA failure (no
//     device, out of memory) throws utf8v::cuda_error, because `bool` has no
//     room for it and a silent wrong verdict is worse.
// Additions (the reference derives these from oracle_validate or a loop):
//   validate_lookup_verdict  -- first error offset and kind, bit-exact with
//                               oracle_validate (proj/src/oracle.cpp:10-44)
//   validate_lookup_batch    -- one verdict per record of a CSR batch
//   lookup_stream            -- one stream validated in pieces, in order
//   segment_state            -- segments validated anywhere, merged later
//   shard_comm               -- a stream sharded over GPUs, combined by NCCL
// Latency: host inputs of at most 64 KiB (and host batches of at most 4096
// records spanning at most 64 KiB) are answered by the small-call server, one
// resident CTA per calling thread and device that polls a mapped-memory
// mailbox (3.5-7.4 us per call instead of a launch and a synchronisation);
// it exits after 100 us without a request (UTF8V_CUDA_SERVE_IDLE_US) and is
// turned off by UTF8V_CUDA_SERVE=0 (include/utf8v_cuda.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "utf8v/verdict.hpp"

namespace utf8v {

struct lookup_backend {
  const char* name;   // "cuda"
  std::size_t width;  // 64
  bool (*validate)(const std::uint8_t* data, std::size_t size);
  void (*classify_lanes)(const std::uint8_t* input, const std::uint8_t* previous,
                         std::uint8_t* out);
  void (*length_error_lanes)(const std::uint8_t* input, const std::uint8_t* previous,
                             std::uint8_t* out);
  void (*incomplete_lanes)(const std::uint8_t* input, std::uint8_t* out);
  bool (*ops_self_test)(std::uint64_t seed);
};

class cuda_error : public std::runtime_error {
 public:
  cuda_error(int status, const std::string& what) : std::runtime_error(what), status_(status) {}
  int status() const noexcept { return status_; }

 private:
  int status_;
};

std::span<const lookup_backend> lookup_backends();
const lookup_backend* find_lookup_backend(std::string_view name);
bool validate_lookup(bytes_view input);
bool validate_lookup_fallback(bytes_view input);

// Extensions.
verdict validate_lookup_verdict(bytes_view input);
std::vector<std::uint8_t> validate_lookup_batch(bytes_view data,
                                                std::span<const std::uint64_t> offsets);

// One stream validated in pieces (the Lookup counterpart of threading
// fsm_state through validate_fsm, proj/include/utf8v/fsm.hpp:15-20):
// feed() host pieces in order, finish() gives the verdict of their
// concatenation and resets the stream.
class lookup_stream {
 public:
  lookup_stream();
  ~lookup_stream();
  lookup_stream(const lookup_stream&) = delete;
  lookup_stream& operator=(const lookup_stream&) = delete;
  void feed(bytes_view piece);
  bool finish();
  std::uint64_t bytes_fed() const;

 private:
  void* handle_ = nullptr;
};

// A segment validated on its own (any device, any order): its composable
// state (utf8v_state, include/utf8v_cuda.h).  combine() is associative, so
// states of consecutive segments merge in any grouping; valid() of the
// whole stream's state is its verdict -- the order-free counterpart of
// threading fsm_state (proj/include/utf8v/fsm.hpp:15-20).
struct segment_state {
  std::uint64_t len = 0;
  std::uint32_t flag = 0;
  std::uint8_t head[4] = {0, 0, 0, 0};
  std::uint8_t tail[4] = {0, 0, 0, 0};
  std::uint32_t reserved = 0;

  static segment_state of(bytes_view segment);   // host bytes, validated on the GPU
  segment_state then(const segment_state& next) const;  // this segment followed by `next`
  bool valid() const;                            // verdict of a whole-stream state
};
std::vector<segment_state> batch_states(bytes_view data, std::span<const std::uint64_t> offsets);

// One rank of a stream sharded over GPUs (one process per GPU), the verdict
// combined with NCCL from the native layer.  The unique id
// comes from rank 0 (unique_id()) through the caller's bootstrap.  The shard
// is this rank's bytes with the look-back head and lookahead tail of
// sharding.plan, lanes [lane_lo, lane_hi) in its own coordinates.
class shard_comm {
 public:
  static std::vector<std::uint8_t> unique_id();
  shard_comm(std::span<const std::uint8_t> id, int nranks, int rank);
  ~shard_comm();
  shard_comm(const shard_comm&) = delete;
  shard_comm& operator=(const shard_comm&) = delete;
  // Collective: the whole stream's verdict / first error (shard_offset = the
  // stream offset of shard[0]).
  bool validate(bytes_view shard, std::uint64_t lane_lo, std::uint64_t lane_hi);
  verdict validate_verdict(bytes_view shard, std::uint64_t lane_lo, std::uint64_t lane_hi,
                           std::uint64_t shard_offset);

 private:
  void* handle_ = nullptr;
};

}  // namespace utf8v
