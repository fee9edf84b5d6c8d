// utf8v-cuda -- the reference CLI's `validate` and `bench` commands
// (proj/tools/main.cpp) on the B200 Lookup path.
//
//   utf8v-cuda validate [--algo cuda] [--json] [FILE]     (stdin when omitted)
//   utf8v-cuda bench [--algo cuda] [--file F | --size N --seed S]
//                    [--repeats R] [--device] [--compensate] [--json]
//
// Exit codes as proj/tools/main.cpp:28-31: 0 valid / success, 1 malformed
// input, 2 usage or I/O error, 3 internal inconsistency.  `validate` prints
// "valid" or "invalid: <kind> at offset <n>" (JSON: {"valid":..,"offset":..,
// "kind":..}); the fast verdict (K1) is cross-checked against the exact one
// (K3), and a disagreement is an internal error, as in main.cpp:129-147.
// A missing device or CUDA failure exits 2 (environment error).
// `bench` reports with the schema of proj/src/bench.cpp:127-139.  Host input
// is timed end to end (host buffer in, verdict out, PCIe included), --device
// times the device-resident path.  --compensate times the input and the
// input doubled and reports the difference (bench.cpp:70-78,92-99: fixed
// per-call overhead cancels; well-formed input only).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <iterator>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "utf8v/lookup.hpp"
#include "utf8v_cuda.h"
#include "utf8v_gen.h"

namespace {

constexpr int k_exit_ok = 0;
constexpr int k_exit_invalid = 1;
constexpr int k_exit_usage = 2;
constexpr int k_exit_inconsistent = 3;

int usage(const char* why) {
  if (why) std::cerr << "error: " << why << "\n";
  std::cerr << "usage: utf8v-cuda validate [--algo cuda] [--json] [FILE]\n"
               "       utf8v-cuda bench [--algo cuda] [--file F | --size N --seed S] [--repeats R]"
               " [--device] [--compensate] [--json]\n";
  return k_exit_usage;
}

bool read_input(const std::string& path, std::vector<std::uint8_t>& out) {
  if (path.empty() || path == "-") {
    out.assign(std::istreambuf_iterator<char>(std::cin), std::istreambuf_iterator<char>());
    return true;
  }
  std::ifstream f(path, std::ios::binary);
  if (!f) {
    std::cerr << "error: cannot open '" << path << "'\n";
    return false;
  }
  out.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
  return true;
}

std::string json_escape(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o;
}

int run_validate(const std::string& path, bool as_json) {
  std::vector<std::uint8_t> bytes;
  if (!read_input(path, bytes)) return k_exit_usage;
  try {
    const bool fast = utf8v::validate_lookup(bytes);
    const utf8v::verdict v = utf8v::validate_lookup_verdict(bytes);
    if (fast != v.valid()) {
      std::cerr << "error: 'cuda' verdict and exact scan disagree\n";
      return k_exit_inconsistent;
    }
    if (v.valid()) {
      std::cout << (as_json ? "{\"valid\":true}" : "valid") << "\n";
      return k_exit_ok;
    }
    const std::string kind(utf8v::to_string(v.error->kind));
    if (as_json)
      std::cout << "{\"kind\":\"" << kind << "\",\"offset\":" << v.error->offset << ",\"valid\":false}\n";
    else
      std::cout << "invalid: " << kind << " at offset " << v.error->offset << "\n";
    return k_exit_invalid;
  } catch (const utf8v::cuda_error& e) {
    // No device / CUDA failure: an environment error, not a verdict.
    std::cerr << "error: " << e.what() << "\n";
    return k_exit_usage;
  }
}

struct timing {
  double best, mean;
};

// A CUDA / environment failure inside `bench` (exit 2, as `validate`).
struct env_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Device copies of the bench input, freed on every return path.
struct dev_buffers {
  std::vector<std::uint8_t*> v;
  ~dev_buffers() {
    for (std::uint8_t* d : v) cudaFree(d);
  }
};

int run_bench_impl(const std::string& file, std::uint64_t size, std::uint64_t seed, int repeats, bool device,
                   bool compensate, bool as_json) {
  std::vector<std::uint8_t> bytes;
  std::string input_name;
  bool expect_valid = true;
  if (!file.empty()) {
    if (!read_input(file, bytes)) return k_exit_usage;
    input_name = file;
    expect_valid = utf8v::validate_lookup_verdict(bytes).valid();
  } else {
    bytes.resize(size);
    if (utf8v_gen_stream_host(bytes.data(), size, seed, 0, 0) != UTF8V_OK) {
      std::cerr << "error: generator: " << utf8v_cuda_last_error() << "\n";
      return k_exit_usage;
    }
    input_name = "c1-mix seed=" + std::to_string(seed);
  }
  if (compensate && !expect_valid) {
    std::cerr << "error: compensated timing needs well-formed input\n";
    return k_exit_usage;
  }
  // Host or device copies of the input (and of the input doubled).
  std::vector<std::uint8_t> doubled;
  if (compensate) {
    doubled.reserve(bytes.size() * 2);
    doubled.insert(doubled.end(), bytes.begin(), bytes.end());
    doubled.insert(doubled.end(), bytes.begin(), bytes.end());
  }
  dev_buffers dev_bufs;
  auto place = [&](const std::vector<std::uint8_t>& b) -> const std::uint8_t* {
    if (!device) return b.data();
    std::uint8_t* d = nullptr;
    cudaError_t e = cudaMalloc(&d, b.size() ? b.size() : 1);
    if (e == cudaSuccess) {
      dev_bufs.v.push_back(d);
      e = cudaMemcpy(d, b.data(), b.size(), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) throw env_error(std::string("device buffer: ") + cudaGetErrorString(e));
    return d;
  };
  const std::uint8_t* p1 = place(bytes);
  const std::uint8_t* p2 = compensate ? place(doubled) : nullptr;
  auto once = [&](const std::uint8_t* p, std::size_t n) -> int {
    std::uint8_t ok = 0;
    if (utf8v_cuda_validate(p, n, device ? 1 : 0, &ok) != UTF8V_OK) throw env_error(utf8v_cuda_last_error());
    return ok;
  };
  // Correctness gate before timing (proj/src/bench.cpp:80-86).
  int gate = once(p1, bytes.size());
  if (gate >= 0 && compensate) gate = once(p2, doubled.size()) == 1 && gate == 1 ? 1 : -1;
  if (gate < 0 || (gate == 1) != expect_valid) {
    std::cerr << "error: validator_mismatch on '" << input_name << "'\n";
    return k_exit_inconsistent;
  }
  auto passes = [&](const std::uint8_t* p, std::size_t n, timing& t) -> bool {
    t.best = std::numeric_limits<double>::infinity();
    double sum = 0.0;
    for (int r = 0; r < repeats; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      if (once(p, n) < 0) return false;
      const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      t.best = s < t.best ? s : t.best;
      sum += s;
    }
    t.mean = sum / repeats;
    return true;
  };
  timing t{};
  if (!passes(p1, bytes.size(), t)) return k_exit_inconsistent;
  if (compensate) {
    timing td{};
    if (!passes(p2, doubled.size(), td)) return k_exit_inconsistent;
    // Difference of the two runs, clamped to 0 <= best <= mean (bench.cpp:92-99).
    t.best = std::max(td.best - t.best, 0.0);
    t.mean = std::max(td.mean - t.mean, t.best);
  }
  const double best = t.best, mean = t.mean;
  const double n = (double)bytes.size();
  const std::string name = device ? "cuda-device" : "cuda";
  std::cerr << "lookup backend: cuda (" << UTF8V_CUDA_WIDTH << "-byte lanes, sm_100a)\n";
  if (as_json) {
    std::printf(
        "[\n  {\n    \"best_seconds\": %.9g,\n    \"best_throughput\": %.9g,\n    \"compensated\": %s,\n"
        "    \"input_bytes\": %zu,\n    \"input_name\": \"%s\",\n    \"mean_seconds\": %.9g,\n"
        "    \"mean_throughput\": %.9g,\n    \"repeats\": %d,\n    \"validator\": \"%s\"\n  }\n]\n",
        best, n / best, compensate ? "true" : "false", bytes.size(), json_escape(input_name).c_str(), mean,
        n / mean, repeats, name.c_str());
  } else {
    std::printf("%-13s%-22s%12s%12s%12s\n", "validator", "input", "bytes", "best GB/s", "mean GB/s");
    std::printf("%-13s%-22s%12zu%12.3f%12.3f\n", name.c_str(), input_name.c_str(), bytes.size(),
                n / best / 1e9, n / mean / 1e9);
  }
  return k_exit_ok;
}

int run_bench(const std::string& file, std::uint64_t size, std::uint64_t seed, int repeats, bool device,
              bool compensate, bool as_json) {
  try {
    return run_bench_impl(file, size, seed, repeats, device, compensate, as_json);
  } catch (const utf8v::cuda_error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return k_exit_usage;
  } catch (const env_error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return k_exit_usage;
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage(nullptr);
  const std::string cmd = argv[1];
  if (cmd == "-h" || cmd == "--help") {
    usage(nullptr);
    return k_exit_ok;
  }
  std::string file, algo = "cuda";
  bool as_json = false, device = false, compensate = false;
  std::uint64_t size = 1ull << 26, seed = 2;
  int repeats = 20;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    auto value = [&](const char* what) -> const char* {
      if (i + 1 >= argc) return nullptr;
      (void)what;
      return argv[++i];
    };
    if (a == "--json") {
      as_json = true;
    } else if (a == "--device") {
      device = true;
    } else if (a == "--compensate") {
      compensate = true;
    } else if (a == "--algo" || a.rfind("--algo=", 0) == 0) {
      const char* v = a == "--algo" ? value("--algo") : a.c_str() + 7;
      if (!v) return usage("--algo needs a value");
      algo = v;
    } else if (a == "--file") {
      const char* v = value("--file");
      if (!v) return usage("--file needs a value");
      file = v;
    } else if (a == "--size" || a == "--seed" || a == "--repeats") {
      const char* v = value(a.c_str());
      if (!v) return usage("option needs a value");
      char* end = nullptr;
      const unsigned long long x = std::strtoull(v, &end, 10);
      if (!end || *end) return usage("not a number");
      if (a == "--size") size = x;
      else if (a == "--seed") seed = x;
      else repeats = (int)x;
    } else if (!a.empty() && a[0] == '-' && a != "-") {
      return usage(("unknown option " + a).c_str());
    } else {
      file = a;
    }
  }
  if (algo != "cuda" && algo != "lookup") return usage("--algo: only 'cuda' (alias 'lookup') is built here");
  if (cmd == "validate") return run_validate(file, as_json);
  if (cmd == "bench") {
    if (repeats < 1) return usage("--repeats must be >= 1");
    return run_bench(file, size, seed, repeats, device, compensate, as_json);
  }
  return usage(("unknown command " + cmd).c_str());
}
