// pageable_copy.cpp -- host copy throughput from pageable memory into pinned
// memory with T threads (the CopyPool's job), regular vs non-temporal stores,
// and the whole pageable e2e of utf8v_cuda_validate for comparison.
// g++ -O3 -mavx2 -std=c++17 -Iinclude pageable_copy.cpp -lcudart -lutf8v_cuda ...
#include <cuda_runtime.h>
#include <immintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <chrono>
#include <thread>
#include <vector>

#include "utf8v_cuda.h"

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void copy_nt(uint8_t* dst, const uint8_t* src, size_t n) {
  size_t i = 0;
  for (; i + 128 <= n; i += 128) {
    __m256i a = _mm256_loadu_si256((const __m256i*)(src + i));
    __m256i b = _mm256_loadu_si256((const __m256i*)(src + i + 32));
    __m256i c = _mm256_loadu_si256((const __m256i*)(src + i + 64));
    __m256i d = _mm256_loadu_si256((const __m256i*)(src + i + 96));
    _mm256_stream_si256((__m256i*)(dst + i), a);
    _mm256_stream_si256((__m256i*)(dst + i + 32), b);
    _mm256_stream_si256((__m256i*)(dst + i + 64), c);
    _mm256_stream_si256((__m256i*)(dst + i + 96), d);
  }
  memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}

int main() {
  const size_t n = 1ull << 30;
  std::vector<uint8_t> src(n);
  for (size_t i = 0; i < n; i += 4096) src[i] = 'a';
  memset(src.data(), 'a', n);
  uint8_t* dst = nullptr;
  const cudaError_t e = cudaHostAlloc((void**)&dst, n, 0);
  if (e != cudaSuccess || !dst) {
    printf("cudaHostAlloc: %s\n", cudaGetErrorString(e));
    return 1;
  }
  printf("pinned buffer ok\n");
  fflush(stdout);
  for (int nt = 0; nt < 2; ++nt) {
    for (int T : {1, 4, 8, 12, 16}) {
      double best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        const double t0 = now_s();
        std::vector<std::thread> th;
        const size_t seg = (n / T) & ~size_t(4095);  // NT stores need aligned destinations
        for (int k = 0; k < T; ++k)
          th.emplace_back([&, k] {
            const size_t len = k == T - 1 ? n - k * seg : seg;
            if (nt) copy_nt(dst + k * seg, src.data() + k * seg, len);
            else memcpy(dst + k * seg, src.data() + k * seg, len);
          });
        for (auto& t : th) t.join();
        best = std::min(best, now_s() - t0);
      }
      printf("%s copy, %2d threads: %.1f GB/s\n", nt ? "non-temporal" : "memcpy      ", T, n / best / 1e9);
    }
  }
  uint8_t ok = 0;
  utf8v_cuda_validate(src.data(), n, 0, &ok);
  double best = 1e9;
  for (int rep = 0; rep < 5; ++rep) {
    const double t0 = now_s();
    utf8v_cuda_validate(src.data(), n, 0, &ok);
    best = std::min(best, now_s() - t0);
  }
  printf("utf8v_cuda_validate(pageable 1 GiB): %.1f GB/s valid=%d\n", n / best / 1e9, ok);
  return 0;
}
