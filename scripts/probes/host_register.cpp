// host_register.cpp -- cost of cudaHostRegister / Unregister on ordinary
// (pageable) memory, per piece size: could the pageable path pin the
// caller's pages in place instead of copying them into a pinned ring?
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <chrono>

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  const size_t n = 1ull << 30;
  uint8_t* src = (uint8_t*)aligned_alloc(4096, n);
  memset(src, 'a', n);
  uint8_t* d;
  if (cudaMalloc(&d, n) != cudaSuccess) return 1;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (size_t piece : {size_t(2) << 20, size_t(8) << 20, size_t(32) << 20, size_t(128) << 20, n}) {
    double reg = 0, unreg = 0;
    const double t0 = now_s();
    for (size_t off = 0; off < n; off += piece) {
      double a = now_s();
      cudaError_t e = cudaHostRegister(src + off, piece, cudaHostRegisterDefault);
      if (e != cudaSuccess) {
        printf("register: %s\n", cudaGetErrorString(e));
        return 1;
      }
      reg += now_s() - a;
      cudaMemcpyAsync(d + off, src + off, piece, cudaMemcpyHostToDevice, s);
      cudaStreamSynchronize(s);
      a = now_s();
      cudaHostUnregister(src + off);
      unreg += now_s() - a;
    }
    const double total = now_s() - t0;
    printf("piece %5zu MiB: register %.1f GB/s, unregister %.1f GB/s, serial register+copy+unregister %.1f GB/s\n",
           piece >> 20, n / reg / 1e9, n / unreg / 1e9, n / total / 1e9);
  }
  return 0;
}
