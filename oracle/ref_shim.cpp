// ref_shim.cpp -- extern "C" face of the UNMODIFIED reference utf8v library,
// compiled straight from the reference checkout by oracle/Makefile into
// oracle/_ref/libutf8v_ref.so.  TEST / BASELINE INFRASTRUCTURE ONLY: used by
// tests/ to pin the oracle restatement and by bench.py's reference arm and
// cpu_baseline leg.  No reference source is copied into this repository.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "utf8v/corpus.hpp"
#include "utf8v/lookup.hpp"
#include "utf8v/oracle.hpp"
#include "utf8v/tables.hpp"

using namespace utf8v;

extern "C" {

// oracle_validate (proj/src/oracle.cpp:10-44): 1 = valid.
int ref_oracle_validate(const uint8_t* p, size_t n, uint64_t* offset, int* kind) {
  const verdict v = oracle_validate(bytes_view{p, n});
  if (v.valid()) return 1;
  *offset = v.error->offset;
  *kind = static_cast<int>(v.error->kind);
  return 0;
}

// validate_lookup (proj/src/lookup.cpp:39-41): widest backend (AVX2 here).
int ref_validate_lookup(const uint8_t* p, size_t n) { return validate_lookup(bytes_view{p, n}); }

// validate_lookup_fallback (proj/src/lookup.cpp:43-45): scalar backend.
int ref_validate_lookup_fallback(const uint8_t* p, size_t n) {
  return validate_lookup_fallback(bytes_view{p, n});
}

int ref_backend_count() { return static_cast<int>(lookup_backends().size()); }

const char* ref_backend_name(int i) { return lookup_backends()[i].name; }

size_t ref_backend_width(int i) { return lookup_backends()[i].width; }

int ref_backend_validate(int i, const uint8_t* p, size_t n) {
  return lookup_backends()[i].validate(p, n);
}

void ref_backend_classify(int i, const uint8_t* in, const uint8_t* prev, uint8_t* out) {
  lookup_backends()[i].classify_lanes(in, prev, out);
}

void ref_backend_length_error(int i, const uint8_t* in, const uint8_t* prev, uint8_t* out) {
  lookup_backends()[i].length_error_lanes(in, prev, out);
}

void ref_backend_incomplete(int i, const uint8_t* in, uint8_t* out) {
  lookup_backends()[i].incomplete_lanes(in, out);
}

int ref_backend_self_test(int i, uint64_t seed) { return lookup_backends()[i].ops_self_test(seed); }

void ref_nibble_tables(uint8_t* t1, uint8_t* t2, uint8_t* t3) {
  std::memcpy(t1, k_nibble_tables.table1.data(), 16);
  std::memcpy(t2, k_nibble_tables.table2.data(), 16);
  std::memcpy(t3, k_nibble_tables.table3.data(), 16);
}

int ref_encode(uint32_t cp, uint8_t* out) {
  if (cp > 0x1FFFFF) return 0;
  const encoded_char e = encode_code_point(cp);
  std::memcpy(out, e.bytes.data(), e.size);
  return e.size;
}

static std::vector<int> kinds_of(unsigned mask) {
  std::vector<int> k;
  for (int i = 1; i <= 4; ++i)
    if (mask & (1u << (i - 1))) k.push_back(i);
  return k;
}

// generate_valid (proj/src/corpus.cpp:84-95); returns size or -1 if cap short.
long long ref_generate_valid(unsigned mask, size_t target, uint64_t seed, uint8_t* out,
                             size_t cap) {
  const std::vector<uint8_t> b = generate_valid(generator_spec{kinds_of(mask), target, seed});
  if (b.size() > cap) return -1;
  std::memcpy(out, b.data(), b.size());
  return static_cast<long long>(b.size());
}

// generate_invalid (proj/src/corpus.cpp:107-188).
long long ref_generate_invalid(unsigned mask, size_t target, uint64_t seed, int strategy,
                               uint8_t* out, size_t cap) {
  const std::vector<uint8_t> b = generate_invalid(generator_spec{kinds_of(mask), target, seed},
                                                  static_cast<mutation_strategy>(strategy));
  if (b.size() > cap) return -1;
  std::memcpy(out, b.data(), b.size());
  return static_cast<long long>(b.size());
}

// The reference Lookup path on T host threads: cut at floor(k*n/T), advance
// each cut at most 3 bytes to a non-continuation byte (the region_start rule
// of proj/src/fsm.cpp:25-34), validate_lookup each region, AND the results.
// Exact: two valid pieces that meet on a character boundary concatenate to
// valid text, and a cut that cannot find a boundary means 4 continuations in
// a row, which is invalid.  This is the multi-core CPU baseline.
int ref_validate_lookup_mt(const uint8_t* p, size_t n, int threads) {
  if (threads <= 1 || n < static_cast<size_t>(threads) * 4096) return validate_lookup(bytes_view{p, n});
  std::vector<size_t> cut(threads + 1);
  cut[0] = 0;
  cut[threads] = n;
  for (int t = 1; t < threads; ++t) {
    size_t c = static_cast<size_t>((static_cast<unsigned __int128>(n) * t) / threads);
    size_t k = 0;
    while (k < 4 && c + k < n && (p[c + k] & 0xC0) == 0x80) ++k;
    if (k == 4) return 0;
    cut[t] = std::max(c + k, cut[t - 1]);
  }
  std::vector<int> ok(threads, 1);
  std::vector<std::thread> pool;
  pool.reserve(threads);
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] { ok[t] = validate_lookup(bytes_view{p + cut[t], cut[t + 1] - cut[t]}); });
  for (auto& th : pool) th.join();
  for (int v : ok)
    if (!v) return 0;
  return 1;
}

}  // extern "C"
