// api_test.cpp -- the reference's Lookup test plan (proj/tests/test_lookup.cpp,
// proj/tests/test_oracle.cpp) run against the B200 library through its C++
// API (include/utf8v/lookup.hpp), i.e. the way a reference caller links it.
// The checker is the C restatement in oracle/ (test infrastructure).
//
// Build: paper_2010_03090_b200/_build.py (build_test_helpers).  Run on a GPU
// box: tests/cpp/api_test  (exit 0 = every case passed).
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#include "utf8_oracle.h"
#include "utf8v/lookup.hpp"

namespace {

int g_failures = 0;
int g_checks = 0;

#define CHECK(cond)                                                                 \
  do {                                                                              \
    ++g_checks;                                                                     \
    if (!(cond)) {                                                                  \
      ++g_failures;                                                                 \
      if (g_failures < 20) std::fprintf(stderr, "  FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                               \
  } while (0)

using bytes = std::vector<std::uint8_t>;

bytes B(std::initializer_list<int> v) {
  bytes b;
  for (int x : v) b.push_back(static_cast<std::uint8_t>(x));
  return b;
}

bool oracle_ok(const bytes& b) {
  std::uint64_t off;
  int kind;
  return orc_validate(b.data(), b.size(), &off, &kind) != 0;
}

utf8v::verdict oracle_verdict(const bytes& b) {
  std::uint64_t off = 0;
  int kind = -1;
  if (orc_validate(b.data(), b.size(), &off, &kind)) return utf8v::verdict::ok();
  return utf8v::verdict::fail(off, static_cast<utf8v::error_kind>(kind));
}

std::uint64_t xorshift(std::uint64_t& s) {
  s ^= s << 13;
  s ^= s >> 7;
  s ^= s << 17;
  return s;
}

struct test_case {
  const char* name;
  std::function<void()> body;
};

std::vector<test_case>& registry() {
  static std::vector<test_case> r;
  return r;
}

struct registrar {
  registrar(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};

#define TEST(id, title) \
  static void id();     \
  static registrar reg_##id(title, id); \
  static void id()

// ---------------------------------------------------------------------------

TEST(roster, "backend roster is well formed (test_lookup.cpp:34-51)") {
  const auto rs = utf8v::lookup_backends();
  CHECK(!rs.empty());
  CHECK(std::string(rs.front().name) == "cuda");
  for (const auto& b : rs) {
    CHECK(b.width >= 32);
    CHECK(b.validate && b.classify_lanes && b.length_error_lanes && b.incomplete_lanes &&
          b.ops_self_test);
    CHECK(utf8v::find_lookup_backend(b.name) == &b);
  }
  for (std::size_t i = 1; i < rs.size(); ++i) CHECK(rs[i - 1].width >= rs[i].width);
  CHECK(utf8v::find_lookup_backend("no-such-backend") == nullptr);
}

TEST(self_test, "every backend passes the vector-operation self test (:53-60)") {
  for (const auto& b : utf8v::lookup_backends())
    for (std::uint64_t seed : {1ull, 2ull, 0x9E3779B97F4A7C15ull, 12345ull}) CHECK(b.ops_self_test(seed));
}

TEST(lanes, "lane entry points equal the restated kernels on random and structured vectors (:62-187)") {
  std::uint64_t s = 0x1234567;
  for (const auto& b : utf8v::lookup_backends()) {
    const std::size_t w = b.width;
    bytes in(w), prev(w), got(w), want(w);
    for (int round = 0; round < 300; ++round) {
      for (std::size_t i = 0; i < w; ++i) {
        const std::uint64_t r = xorshift(s);
        // Mix of uniform bytes and bytes near the interesting thresholds.
        static const int pick[] = {0x00, 0x41, 0x7F, 0x80, 0x8F, 0x90, 0x9F, 0xA0, 0xBF, 0xC0, 0xC1,
                                   0xC2, 0xDF, 0xE0, 0xED, 0xEF, 0xF0, 0xF4, 0xF5, 0xFF};
        in[i] = (r & 3) ? static_cast<std::uint8_t>(r >> 8) : pick[(r >> 16) % 20];
        prev[i] = static_cast<std::uint8_t>(r >> 24);
      }
      b.classify_lanes(in.data(), prev.data(), got.data());
      orc_classify_lanes(in.data(), prev.data(), want.data(), w);
      CHECK(got == want);
      b.length_error_lanes(in.data(), prev.data(), got.data());
      orc_length_error_lanes(in.data(), prev.data(), want.data(), w);
      CHECK(got == want);
      b.incomplete_lanes(in.data(), got.data());
      orc_incomplete_lanes(in.data(), want.data(), w);
      CHECK(got == want);
    }
    // Pure ASCII classifies to zero (:81-90).
    for (std::size_t i = 0; i < w; ++i) in[i] = prev[i] = static_cast<std::uint8_t>(0x20 + i % 90);
    b.classify_lanes(in.data(), prev.data(), got.data());
    CHECK(got == bytes(w, 0));
  }
}

TEST(known, "whole-buffer verdicts on known inputs (:189-201)") {
  CHECK(utf8v::validate_lookup(utf8v::bytes_view{}));
  CHECK(utf8v::lookup_backends().front().validate(nullptr, 0));
  const std::vector<std::pair<bytes, bool>> cases = {
      {B({'h', 'i'}), true},
      {B({0xC3, 0xA9}), true},
      {B({0xE2, 0x82, 0xAC}), true},
      {B({0xF0, 0x9F, 0x98, 0x80}), true},
      {B({0xF4, 0x8F, 0xBF, 0xBF}), true},
      {B({0xEF, 0xBF, 0xBF}), true},
      {B({0xC0, 0x80}), false},
      {B({0xC1, 0xBF}), false},
      {B({0xE0, 0x9F, 0xBF}), false},
      {B({0xED, 0xA0, 0x80}), false},
      {B({0xF0, 0x8F, 0xBF, 0xBF}), false},
      {B({0xF4, 0x90, 0x80, 0x80}), false},
      {B({0xF5, 0x80, 0x80, 0x80}), false},
      {B({0xFF}), false},
      {B({0x80}), false},
      {B({0xC3}), false},
      {B({0xE2, 0x82}), false},
      {B({0xF0, 0x9F, 0x98}), false},
      {B({0xC3, 0x41}), false},
      {B({0xE0, 0x30, 0x30}), false},
  };
  for (const auto& [b, want] : cases) {
    CHECK(oracle_ok(b) == want);
    CHECK(utf8v::validate_lookup(b) == want);
    CHECK(utf8v::validate_lookup_fallback(b) == want);
    CHECK(utf8v::validate_lookup_verdict(b) == oracle_verdict(b));
  }
}

TEST(sticky, "errors survive any number of later clean blocks (:203-214)") {
  for (std::size_t clean : {0u, 1u, 63u, 64u, 4096u, 1u << 20}) {
    bytes b = B({0xC0, 0x80});
    b.resize(2 + clean, 'a');
    CHECK(!utf8v::validate_lookup(b));
    bytes c(clean, 'a');
    c.push_back(0xE2);  // error at the very end after clean data
    CHECK(!utf8v::validate_lookup(c));
  }
}

TEST(tails, "block boundaries and tails for every length (:216-254)") {
  const bytes euro = B({0xE2, 0x82, 0xAC});
  for (std::size_t len = 0; len < 300; ++len) {
    bytes b(len, 'x');
    for (std::size_t i = 0; i + 3 <= len; i += 7) std::memcpy(&b[i], euro.data(), 3);
    CHECK(utf8v::validate_lookup(b) == oracle_ok(b));
    for (std::size_t cut = 1; cut <= 3 && len >= cut; ++cut) {
      bytes t = b;
      // Truncated 4-byte sequence in the last `cut` bytes.
      static const std::uint8_t four[4] = {0xF0, 0x9F, 0x98, 0x80};
      std::memcpy(&t[len - cut], four, cut);
      CHECK(utf8v::validate_lookup(t) == oracle_ok(t));
      CHECK(utf8v::validate_lookup_verdict(t) == oracle_verdict(t));
    }
  }
}

TEST(ascii_between, "ascii blocks between multibyte blocks keep the checks sound (:256-285)") {
  for (std::size_t gap : {0u, 1u, 31u, 32u, 64u, 65u, 4096u, 4097u, 70000u}) {
    bytes b;
    b.insert(b.end(), {0xE2, 0x82});  // pending lead at the end of a block...
    b.resize(b.size() + gap, 'a');    // ...then ASCII
    b.insert(b.end(), {0xE2, 0x82, 0xAC});
    CHECK(utf8v::validate_lookup(b) == oracle_ok(b));
    bytes v = B({0xE2, 0x82, 0xAC});
    v.resize(3 + gap, 'a');
    v.insert(v.end(), {0xF0, 0x9F, 0x98, 0x80});
    CHECK(utf8v::validate_lookup(v));
  }
}

TEST(seams, "all byte pairs at every seam offset match the reference (:287-311)") {
  // One record per pair, embedded at offset `o` of a 96-byte ASCII record;
  // checked through the batch entry point (one launch per offset).
  for (std::size_t o : {0u, 1u, 2u, 3u, 14u, 15u, 30u, 31u, 32u, 33u, 62u, 63u, 64u, 94u}) {
    const std::size_t len = 96;
    bytes data(65536 * len, 'a');
    std::vector<std::uint64_t> offs(65537);
    std::vector<std::uint8_t> want(65536);
    for (std::size_t p = 0; p < 65536; ++p) {
      offs[p] = p * len;
      std::uint8_t* r = &data[p * len];
      r[o] = static_cast<std::uint8_t>(p >> 8);
      if (o + 1 < len) r[o + 1] = static_cast<std::uint8_t>(p & 0xFF);
      std::uint64_t off;
      int kind;
      want[p] = static_cast<std::uint8_t>(orc_validate(r, len, &off, &kind));
    }
    offs[65536] = data.size();
    const auto got = utf8v::validate_lookup_batch(data, offs);
    CHECK(got == want);
  }
}

TEST(corpora, "verdicts and first errors on generated corpora (:338-360, test_oracle.cpp:46-79)") {
  bytes buf(1 << 16);
  for (std::uint64_t seed = 1; seed <= 60; ++seed) {
    for (int strategy = -1; strategy < 7; ++strategy) {
      const std::size_t target = 1 + (seed * 977) % 20000;
      std::size_t n = strategy < 0 ? orc_generate_valid(0xF, target, seed, buf.data(), buf.size())
                                   : orc_generate_invalid(0xF, target, seed, strategy, buf.data(), buf.size());
      if (n == static_cast<std::size_t>(-1)) continue;
      const bytes b(buf.begin(), buf.begin() + static_cast<std::ptrdiff_t>(n));
      const auto want = oracle_verdict(b);
      CHECK(utf8v::validate_lookup(b) == want.valid());
      CHECK(utf8v::validate_lookup_verdict(b) == want);
    }
  }
}

TEST(batch, "record batches: empty, ragged, every error class") {
  CHECK(utf8v::validate_lookup_batch({}, {}).empty());
  std::uint64_t s = 99;
  bytes data;
  std::vector<std::uint64_t> offs = {0};
  std::vector<std::uint8_t> want;
  bytes buf(1 << 14);
  for (int r = 0; r < 5000; ++r) {
    const std::uint64_t x = xorshift(s);
    std::size_t n = 0;
    if (x % 7 == 0) {
      n = 0;  // empty record
    } else if (x % 3 == 0) {
      n = orc_generate_invalid(0xF, 1 + (x >> 8) % 3000, x, static_cast<int>((x >> 40) % 7), buf.data(),
                               buf.size());
    } else {
      n = orc_generate_valid(0xF, 1 + (x >> 8) % 3000, x, buf.data(), buf.size());
    }
    if (n == static_cast<std::size_t>(-1)) n = 0;
    data.insert(data.end(), buf.begin(), buf.begin() + static_cast<std::ptrdiff_t>(n));
    offs.push_back(data.size());
    const bytes rec(buf.begin(), buf.begin() + static_cast<std::ptrdiff_t>(n));
    want.push_back(oracle_ok(rec) ? 1 : 0);
  }
  CHECK(utf8v::validate_lookup_batch(data, offs) == want);
}

TEST(stream, "a stream fed in pieces gives the verdict of the whole (fsm.hpp:15-20)") {
  bytes buf(1 << 14);
  std::uint64_t s = 7;
  utf8v::lookup_stream ls;
  CHECK(ls.finish());
  for (std::uint64_t seed = 1; seed <= 40; ++seed) {
    for (int strategy = -1; strategy < 7; ++strategy) {
      const std::size_t n = strategy < 0 ? orc_generate_valid(0xF, 3000, seed, buf.data(), buf.size())
                                         : orc_generate_invalid(0xF, 3000, seed, strategy, buf.data(), buf.size());
      if (n == static_cast<std::size_t>(-1)) continue;
      const bytes b(buf.begin(), buf.begin() + static_cast<std::ptrdiff_t>(n));
      std::size_t at = 0;
      while (at < n) {
        const std::size_t len = std::min<std::size_t>(n - at, xorshift(s) % 9 == 0 ? 0 : 1 + xorshift(s) % 700);
        ls.feed(utf8v::bytes_view(b.data() + at, len));
        at += len;
      }
      CHECK(ls.bytes_fed() == n);
      CHECK(ls.finish() == oracle_ok(b));
    }
  }
}

TEST(states, "segment states merged in any grouping give the verdict of the whole (fsm.hpp:15-20)") {
  bytes buf(1 << 14);
  std::uint64_t s = 11;
  for (std::uint64_t seed = 1; seed <= 25; ++seed) {
    for (int strategy = -1; strategy < 7; ++strategy) {
      const std::size_t n = strategy < 0 ? orc_generate_valid(0xF, 2000, seed, buf.data(), buf.size())
                                         : orc_generate_invalid(0xF, 2000, seed, strategy, buf.data(), buf.size());
      if (n == static_cast<std::size_t>(-1)) continue;
      const bytes b(buf.begin(), buf.begin() + static_cast<std::ptrdiff_t>(n));
      // cut into pieces of 0..600 bytes, validated one by one (in reverse)
      std::vector<std::pair<std::size_t, std::size_t>> cuts;
      for (std::size_t at = 0; at < n;) {
        const std::size_t len = std::min<std::size_t>(n - at, xorshift(s) % 601);
        cuts.emplace_back(at, len);
        at += len;
      }
      std::vector<utf8v::segment_state> st(cuts.size());
      for (std::size_t i = cuts.size(); i-- > 0;)
        st[i] = utf8v::segment_state::of(utf8v::bytes_view(b.data() + cuts[i].first, cuts[i].second));
      // right fold and left fold must agree (associativity) and give the verdict
      utf8v::segment_state left, right;
      for (const auto& x : st) left = left.then(x);
      for (std::size_t i = st.size(); i-- > 0;) right = st[i].then(right);
      CHECK(left.valid() == oracle_ok(b));
      CHECK(right.valid() == oracle_ok(b));
      CHECK(left.len == n && right.len == n);
      // the pieces as records of a batch: per-record states equal the segment states
      std::vector<std::uint64_t> offs{0};
      for (const auto& c : cuts) offs.push_back(c.first + c.second);
      const auto bs = utf8v::batch_states(b, offs);
      CHECK(bs.size() == st.size());
      for (std::size_t i = 0; i < bs.size() && i < st.size(); ++i)
        CHECK(std::memcmp(&bs[i], &st[i], sizeof(utf8v::segment_state)) == 0);
    }
  }
}

TEST(shard_comm, "a one-rank NCCL shard communicator gives the stream's verdict and first error") {
  const auto id = utf8v::shard_comm::unique_id();
  utf8v::shard_comm comm(id, 1, 0);
  bytes buf(1 << 16);
  for (std::uint64_t seed = 1; seed <= 6; ++seed) {
    for (int strategy = -1; strategy < 7; ++strategy) {
      const std::size_t n = strategy < 0 ? orc_generate_valid(0xF, 30000, seed, buf.data(), buf.size())
                                         : orc_generate_invalid(0xF, 30000, seed, strategy, buf.data(), buf.size());
      if (n == static_cast<std::size_t>(-1)) continue;
      const bytes b(buf.begin(), buf.begin() + static_cast<std::ptrdiff_t>(n));
      CHECK(comm.validate(b, 0, n + 3) == oracle_ok(b));
      CHECK(comm.validate_verdict(b, 0, n + 3, 0) == oracle_verdict(b));
    }
  }
}

TEST(threads, "validators are callable concurrently (bench.cpp:112-118)") {
  std::vector<bytes> inputs;
  std::vector<utf8v::verdict> want;
  bytes buf(1 << 20);
  for (int t = 0; t < 8; ++t) {
    const std::size_t n = t % 2 ? orc_generate_invalid(0xF, 500000, 77 + t, t % 7, buf.data(), buf.size())
                                : orc_generate_valid(0xF, 500000, 77 + t, buf.data(), buf.size());
    inputs.emplace_back(buf.begin(), buf.begin() + static_cast<std::ptrdiff_t>(n));
    want.push_back(oracle_verdict(inputs.back()));
  }
  std::vector<int> ok(8, 0);
  std::vector<std::thread> th;
  for (int t = 0; t < 8; ++t)
    th.emplace_back([&, t] {
      int good = 1;
      for (int k = 0; k < 20; ++k) {
        good &= utf8v::validate_lookup(inputs[t]) == want[t].valid();
        good &= utf8v::validate_lookup_verdict(inputs[t]) == want[t];
      }
      ok[t] = good;
    });
  for (auto& x : th) x.join();
  for (int t = 0; t < 8; ++t) CHECK(ok[t] == 1);
}

}  // namespace

int main(int argc, char** argv) {
  const char* only = argc > 1 ? argv[1] : nullptr;
  int ran = 0;
  for (const auto& tc : registry()) {
    if (only && std::strstr(tc.name, only) == nullptr) continue;
    const int before = g_failures;
    try {
      tc.body();
    } catch (const std::exception& e) {
      ++g_failures;
      std::fprintf(stderr, "  EXCEPTION %s\n", e.what());
    }
    std::printf("%s %s\n", g_failures == before ? "PASS" : "FAIL", tc.name);
    ++ran;
  }
  std::printf("%d cases, %d checks, %d failures\n", ran, g_checks, g_failures);
  return g_failures == 0 && ran > 0 ? 0 : 1;
}
