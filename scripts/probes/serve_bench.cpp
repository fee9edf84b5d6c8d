// serve_bench.cpp -- per-call latency of the C-ABI on pageable host input
// (no Python in the loop): min / median over back-to-back calls.
// g++ -O2 -std=c++17 -Iinclude serve_bench.cpp -Lpaper_2010_03090_b200 -lutf8v_cuda -Wl,-rpath,...
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <chrono>
#include <vector>

#include "utf8v_cuda.h"

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  std::vector<uint8_t> buf(1 << 20);
  for (size_t i = 0; i < buf.size(); ++i) buf[i] = (uint8_t)('a' + i % 26);
  uint8_t ok = 0;
  uint64_t off = 0;
  int kind = 0;
  if (utf8v_cuda_validate(buf.data(), 16, 0, &ok) != 0) {
    printf("error: %s\n", utf8v_cuda_last_error());
    return 1;
  }
  for (size_t n : {16, 256, 4096, 16384, 65536, 262144}) {
    for (int mode = 0; mode < 2; ++mode) {
      std::vector<double> t;
      for (int i = 0; i < 3000; ++i) {
        const double a = now_us();
        if (mode == 0)
          utf8v_cuda_validate(buf.data(), n, 0, &ok);
        else
          utf8v_cuda_validate_verdict(buf.data(), n, 0, &ok, &off, &kind);
        t.push_back(now_us() - a);
      }
      std::sort(t.begin(), t.end());
      printf("%-8s %7zu B: min %6.2f med %6.2f p99 %6.2f us  valid=%d\n", mode ? "verdict" : "validate", n, t[0],
             t[t.size() / 2], t[t.size() * 99 / 100], ok);
    }
  }
  uint64_t l = 0, r = 0;
  utf8v_cuda_serve_stats(&l, &r);
  printf("server launches %llu requests %llu\n", (unsigned long long)l, (unsigned long long)r);
  return 0;
}
