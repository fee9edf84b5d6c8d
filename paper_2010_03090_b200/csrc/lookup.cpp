// lookup.cpp -- the reference C++ API (include/utf8v/lookup.hpp) over the
// C-ABI.  Mirrors proj/src/lookup.cpp:16-45: a roster built once behind a
// function-local static, lookup by name, validate_lookup through front().
#include "utf8v/lookup.hpp"

#include <string>

#include "../../include/utf8v_cuda.h"

namespace utf8v {
namespace {

[[noreturn]] void raise(int status) {
  throw cuda_error(status, std::string("utf8v cuda backend: ") + utf8v_cuda_last_error());
}

bool cuda_validate(const std::uint8_t* data, std::size_t size) {
  std::uint8_t ok = 0;
  const int st = utf8v_cuda_validate(data, size, 0, &ok);
  if (st != UTF8V_OK) raise(st);
  return ok != 0;
}

void cuda_classify(const std::uint8_t* in, const std::uint8_t* prev, std::uint8_t* out) {
  const int st = utf8v_cuda_classify_lanes(in, prev, out);
  if (st != UTF8V_OK) raise(st);
}

void cuda_length_error(const std::uint8_t* in, const std::uint8_t* prev, std::uint8_t* out) {
  const int st = utf8v_cuda_length_error_lanes(in, prev, out);
  if (st != UTF8V_OK) raise(st);
}

void cuda_incomplete(const std::uint8_t* in, std::uint8_t* out) {
  const int st = utf8v_cuda_incomplete_lanes(in, out);
  if (st != UTF8V_OK) raise(st);
}

bool cuda_self_test(std::uint64_t seed) {
  int ok = 0;
  const int st = utf8v_cuda_ops_self_test(seed, &ok);
  if (st != UTF8V_OK) raise(st);
  return ok != 0;
}

constexpr lookup_backend k_cuda = {"cuda",          UTF8V_CUDA_WIDTH, &cuda_validate,
                                   &cuda_classify,  &cuda_length_error, &cuda_incomplete,
                                   &cuda_self_test};

}  // namespace

std::span<const lookup_backend> lookup_backends() {
  static const lookup_backend roster[1] = {k_cuda};
  return roster;
}

const lookup_backend* find_lookup_backend(std::string_view name) {
  for (const lookup_backend& b : lookup_backends())
    if (name == b.name) return &b;
  return nullptr;
}

bool validate_lookup(bytes_view input) {
  return lookup_backends().front().validate(input.data(), input.size());
}

bool validate_lookup_fallback(bytes_view input) {
  return lookup_backends().back().validate(input.data(), input.size());
}

verdict validate_lookup_verdict(bytes_view input) {
  std::uint8_t ok = 0;
  std::uint64_t off = 0;
  int kind = -1;
  const int st = utf8v_cuda_validate_verdict(input.data(), input.size(), 0, &ok, &off, &kind);
  if (st != UTF8V_OK) raise(st);
  if (ok) return verdict::ok();
  return verdict::fail(static_cast<std::size_t>(off), static_cast<error_kind>(kind));
}

std::vector<std::uint8_t> validate_lookup_batch(bytes_view data,
                                                std::span<const std::uint64_t> offsets) {
  if (offsets.empty()) return {};
  std::vector<std::uint8_t> out(offsets.size() - 1);
  const int st = utf8v_cuda_validate_batch(data.data(), data.size(), offsets.data(),
                                           offsets.size() - 1, 0, out.data());
  if (st != UTF8V_OK) raise(st);
  return out;
}

lookup_stream::lookup_stream() {
  utf8v_cuda_stream* s = nullptr;
  const int st = utf8v_cuda_stream_create(&s);
  if (st != UTF8V_OK) raise(st);
  handle_ = s;
}

lookup_stream::~lookup_stream() { utf8v_cuda_stream_destroy(static_cast<utf8v_cuda_stream*>(handle_)); }

void lookup_stream::feed(bytes_view piece) {
  const int st =
      utf8v_cuda_stream_feed(static_cast<utf8v_cuda_stream*>(handle_), piece.data(), piece.size(), 0);
  if (st != UTF8V_OK) raise(st);
}

bool lookup_stream::finish() {
  std::uint8_t ok = 0;
  const int st = utf8v_cuda_stream_finish(static_cast<utf8v_cuda_stream*>(handle_), &ok);
  if (st != UTF8V_OK) raise(st);
  return ok != 0;
}

std::uint64_t lookup_stream::bytes_fed() const {
  return utf8v_cuda_stream_bytes(static_cast<const utf8v_cuda_stream*>(handle_));
}

static_assert(sizeof(segment_state) == sizeof(utf8v_state), "segment_state mirrors utf8v_state");

segment_state segment_state::of(bytes_view segment) {
  segment_state s;
  const int st = utf8v_cuda_segment_state(segment.data(), segment.size(), 0, reinterpret_cast<utf8v_state*>(&s));
  if (st != UTF8V_OK) raise(st);
  return s;
}

segment_state segment_state::then(const segment_state& next) const {
  segment_state r;
  utf8v_state_combine(reinterpret_cast<const utf8v_state*>(this), reinterpret_cast<const utf8v_state*>(&next),
                      reinterpret_cast<utf8v_state*>(&r));
  return r;
}

bool segment_state::valid() const { return utf8v_state_valid(reinterpret_cast<const utf8v_state*>(this)) != 0; }

std::vector<segment_state> batch_states(bytes_view data, std::span<const std::uint64_t> offsets) {
  if (offsets.empty()) return {};
  std::vector<segment_state> out(offsets.size() - 1);
  const int st = utf8v_cuda_batch_states(data.data(), data.size(), offsets.data(), offsets.size() - 1, 0,
                                         reinterpret_cast<utf8v_state*>(out.data()));
  if (st != UTF8V_OK) raise(st);
  return out;
}

std::vector<std::uint8_t> shard_comm::unique_id() {
  std::vector<std::uint8_t> id(UTF8V_COMM_ID_BYTES);
  const int st = utf8v_cuda_comm_unique_id(id.data());
  if (st != UTF8V_OK) raise(st);
  return id;
}

shard_comm::shard_comm(std::span<const std::uint8_t> id, int nranks, int rank) {
  if (id.size() != UTF8V_COMM_ID_BYTES) throw cuda_error(UTF8V_ERR_ARG, "utf8v: unique id must be 128 bytes");
  utf8v_cuda_comm* c = nullptr;
  const int st = utf8v_cuda_comm_init_rank(id.data(), nranks, rank, &c);
  if (st != UTF8V_OK) raise(st);
  handle_ = c;
}

shard_comm::~shard_comm() { utf8v_cuda_comm_destroy(static_cast<utf8v_cuda_comm*>(handle_)); }

bool shard_comm::validate(bytes_view shard, std::uint64_t lane_lo, std::uint64_t lane_hi) {
  std::uint8_t ok = 0;
  const int st = utf8v_cuda_validate_shard_allreduce(static_cast<utf8v_cuda_comm*>(handle_), shard.data(),
                                                     shard.size(), lane_lo, lane_hi, 0, &ok);
  if (st != UTF8V_OK) raise(st);
  return ok != 0;
}

verdict shard_comm::validate_verdict(bytes_view shard, std::uint64_t lane_lo, std::uint64_t lane_hi,
                                     std::uint64_t shard_offset) {
  std::uint8_t ok = 0;
  std::uint64_t off = 0;
  int kind = -1;
  const int st = utf8v_cuda_verdict_shard_allreduce(static_cast<utf8v_cuda_comm*>(handle_), shard.data(),
                                                    shard.size(), lane_lo, lane_hi, shard_offset, 0, &ok, &off,
                                                    &kind);
  if (st != UTF8V_OK) raise(st);
  if (ok) return verdict::ok();
  return verdict::fail(static_cast<std::size_t>(off), static_cast<error_kind>(kind));
}

}  // namespace utf8v
