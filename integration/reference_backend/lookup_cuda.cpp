// lookup_cuda.cpp -- the B200 path as a fourth entry of the reference's
// backend roster (the "reference side" translation unit of INTEGRATION.md
// §3).  A maintainer adds this file to proj/src/ and one registration line to
// detect_backends() (proj/src/lookup.cpp:16-24); it includes only this
// repository's C-ABI header and links -lutf8v_cuda, so the reference build
// needs neither torch nor CUDA headers.
//
// The entry fills struct lookup_backend (proj/include/utf8v/lookup.hpp:18-28)
// with the C-ABI calls of include/utf8v_cuda.h:
//   validate            utf8v_cuda_validate (host bytes, PCIe inside the call)
//   classify_lanes /    utf8v_cuda_classify_lanes / _length_error_lanes /
//   length_error_lanes  _incomplete_lanes (UTF8V_CUDA_WIDTH = 64 host bytes)
//   / incomplete_lanes
//   ops_self_test       utf8v_cuda_ops_self_test
// A CUDA failure inside validate aborts with the library's message: the
// reference's bool cannot carry "no device", and a silent `false` would
// read as invalid text.
#include <cstdio>
#include <cstdlib>

#include "lookup_backend_detail.hpp"
#include "utf8v_cuda.h"

namespace utf8v::detail {
namespace {

[[noreturn]] void die(const char* what) {
  std::fprintf(stderr, "lookup-cuda: %s: %s\n", what, utf8v_cuda_last_error());
  std::abort();
}

bool cuda_validate(const std::uint8_t* data, std::size_t size) {
  std::uint8_t ok = 0;
  if (utf8v_cuda_validate(data, size, /*is_device=*/0, &ok) != UTF8V_OK) die("validate");
  return ok != 0;
}

void cuda_classify(const std::uint8_t* input, const std::uint8_t* previous, std::uint8_t* out) {
  if (utf8v_cuda_classify_lanes(input, previous, out) != UTF8V_OK) die("classify_lanes");
}

void cuda_length_error(const std::uint8_t* input, const std::uint8_t* previous, std::uint8_t* out) {
  if (utf8v_cuda_length_error_lanes(input, previous, out) != UTF8V_OK) die("length_error_lanes");
}

void cuda_incomplete(const std::uint8_t* input, std::uint8_t* out) {
  if (utf8v_cuda_incomplete_lanes(input, out) != UTF8V_OK) die("incomplete_lanes");
}

bool cuda_self_test(std::uint64_t seed) {
  int ok = 0;
  return utf8v_cuda_ops_self_test(seed, &ok) == UTF8V_OK && ok != 0;
}

}  // namespace

const lookup_backend& cuda_backend() {
  static constexpr lookup_backend backend = {"cuda",          UTF8V_CUDA_WIDTH,   &cuda_validate,
                                             &cuda_classify,  &cuda_length_error, &cuda_incomplete,
                                             &cuda_self_test};
  return backend;
}

// The device probe of the registration line: a usable B200 answers the
// self test.
bool cuda_available() {
  int ok = 0;
  return utf8v_cuda_ops_self_test(1, &ok) == UTF8V_OK && ok != 0;
}

}  // namespace utf8v::detail
