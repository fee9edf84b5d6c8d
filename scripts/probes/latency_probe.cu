// latency_probe.cu -- where does a small validate call's time go?
// (round 2 probe; nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lp latency_probe.cu)
//   A: empty kernel launch + cudaStreamSynchronize
//   B: kernel storing a mapped host word + host spin on it (no stream sync)
//   C: kernel reading N bytes of mapped pinned memory (zero copy) + host spin
//   D: a resident doorbell kernel: host memcpy into mapped pinned memory, one
//      sequence store, the kernel polls it (1 or 32 pollers), reads N bytes
//      over PCIe, stores the reply word; the host spins on the reply.
// Prints min / median / p99 in microseconds over R calls.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_));     \
      return 1;                                                                \
    }                                                                          \
  } while (0)

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void k_empty() {}
__global__ void k_store(volatile uint32_t* f, uint32_t v) {
  if (threadIdx.x == 0) *f = v;
}
__global__ void k_read(const uint4* p, int n16, volatile uint32_t* f, uint32_t v) {
  uint32_t acc = 0;
  for (int i = threadIdx.x; i < n16; i += blockDim.x) {
    uint4 q = __ldcv(p + i);
    acc |= q.x | q.y | q.z | q.w;
  }
  acc = __syncthreads_or(acc & 0x80808080u);
  if (threadIdx.x == 0) *f = v | (acc ? 0x80000000u : 0);
}

__device__ __forceinline__ unsigned long long ld_acq_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct Box {
  unsigned long long req;   // seq << 32 | n
  unsigned long long pad0[15];
  unsigned long long resp;  // seq << 1 | flag
  unsigned long long pad1[15];
  unsigned long long stop;
  unsigned long long pad2[15];
};

// D: one CTA; `pollers` threads of warp 0 poll the request word (staggered).
__global__ void k_server(Box* b, const uint4* data, int pollers, unsigned long long idle_ns) {
  __shared__ unsigned long long s_req;
  unsigned long long last = 0;
  unsigned long long t0 = gtimer();
  for (;;) {
    if (threadIdx.x < 32) {
      unsigned long long r = 0;
      for (;;) {
        if ((int)threadIdx.x < pollers) r = ld_acq_sys(&b->req);
        const bool fresh = (r >> 32) != (last >> 32) && r != 0;
        const unsigned m = __ballot_sync(0xffffffffu, fresh);
        if (m) {
          r = __shfl_sync(0xffffffffu, r, __ffs(m) - 1);
          break;
        }
        unsigned long long st = 0;
        if (threadIdx.x == 0) st = ld_acq_sys(&b->stop);
        st = __shfl_sync(0xffffffffu, st, 0);
        if (st || gtimer() - t0 > idle_ns) {
          r = ~0ull;
          break;
        }
      }
      if (threadIdx.x == 0) s_req = r;
    }
    __syncthreads();
    const unsigned long long r = s_req;
    if (r == ~0ull) return;
    last = r;
    const int n16 = (int)((r & 0xffffffffu) + 15) / 16;
    uint32_t acc = 0;
    for (int i = threadIdx.x; i < n16; i += blockDim.x) {
      uint4 q = __ldcv(data + i);
      acc |= q.x | q.y | q.z | q.w;
    }
    acc = __syncthreads_or(acc & 0x80808080u);
    if (threadIdx.x == 0) st_rel_sys(&b->resp, ((r >> 32) << 1) | (acc ? 1 : 0));
    t0 = gtimer();
  }
}


__device__ __forceinline__ unsigned long long ld_rlx_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rlx_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// F: variants. poll_warps warps poll (lane 0 each), warp w starts w*stagger_ns late;
// relaxed loads for polls, relaxed store for the reply when rlx_reply; each
// thread loads `per` uint4 before using them.
__global__ void k_server2(Box* b, const uint4* data, int poll_warps, int stagger_ns, int rlx_reply,
                          unsigned long long idle_ns) {
  __shared__ unsigned long long s_req;
  __shared__ int s_go;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long last = 0;
  if (threadIdx.x == 0) { s_go = 0; s_req = 0; }
  __syncthreads();
  unsigned long long t0 = gtimer();
  for (;;) {
    if (warp < poll_warps) {
      if (lane == 0) {
        const unsigned long long ts = gtimer();
        while (gtimer() - ts < (unsigned long long)(warp * stagger_ns)) {}
        for (;;) {
          if (*(volatile int*)&s_go) break;
          const unsigned long long r = ld_rlx_sys(&b->req);
          if ((r >> 32) != (last >> 32) && r != 0) {
            if (atomicCAS((int*)&s_go, 0, 1) == 0) s_req = r;
            break;
          }
          if (warp == 0 && (ld_rlx_sys(&b->stop) || gtimer() - t0 > idle_ns)) {
            if (atomicCAS((int*)&s_go, 0, 1) == 0) s_req = ~0ull;
            break;
          }
        }
      }
    }
    __syncthreads();
    const unsigned long long r = s_req;
    if (r == ~0ull) return;
    last = r;
    const int n16 = (int)((r & 0xffffffffu) + 15) / 16;
    uint32_t acc = 0;
    uint4 q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = threadIdx.x + j * blockDim.x;
      q[j] = i < n16 ? __ldcv(data + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) acc |= q[j].x | q[j].y | q[j].z | q[j].w;
    for (int i = threadIdx.x + 4 * blockDim.x; i < n16; i += blockDim.x) {
      uint4 x = __ldcv(data + i);
      acc |= x.x | x.y | x.z | x.w;
    }
    acc = __syncthreads_or(acc & 0x80808080u);
    if (threadIdx.x == 0) {
      s_go = 0;
      const unsigned long long v = ((r >> 32) << 1) | (acc ? 1 : 0);
      if (rlx_reply) st_rlx_sys(&b->resp, v); else st_rel_sys(&b->resp, v);
    }
    __syncthreads();
    t0 = gtimer();
  }
}


// k_server2 with the request/stop words and the data in one (write-combined)
// buffer and the reply in another.
__global__ void k_server3(Box* b, Box* rb, const uint4* data, int poll_warps, int stagger_ns,
                          unsigned long long idle_ns) {
  __shared__ unsigned long long s_req;
  __shared__ int s_go;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long last = 0;
  if (threadIdx.x == 0) { s_go = 0; s_req = 0; }
  __syncthreads();
  unsigned long long t0 = gtimer();
  for (;;) {
    if (warp < poll_warps) {
      if (lane == 0) {
        const unsigned long long ts = gtimer();
        while (gtimer() - ts < (unsigned long long)(warp * stagger_ns)) {}
        for (;;) {
          if (*(volatile int*)&s_go) break;
          const unsigned long long r = ld_rlx_sys(&b->req);
          if ((r >> 32) != (last >> 32) && r != 0) {
            if (atomicCAS((int*)&s_go, 0, 1) == 0) s_req = r;
            break;
          }
          if (warp == 0 && (ld_rlx_sys(&b->stop) || gtimer() - t0 > idle_ns)) {
            if (atomicCAS((int*)&s_go, 0, 1) == 0) s_req = ~0ull;
            break;
          }
        }
      }
    }
    __syncthreads();
    const unsigned long long r = s_req;
    if (r == ~0ull) return;
    last = r;
    const int n16 = (int)((r & 0xffffffffu) + 15) / 16;
    uint32_t acc = 0;
    uint4 q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = threadIdx.x + j * blockDim.x;
      q[j] = i < n16 ? __ldcv(data + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) acc |= q[j].x | q[j].y | q[j].z | q[j].w;
    for (int i = threadIdx.x + 4 * blockDim.x; i < n16; i += blockDim.x) {
      uint4 x = __ldcv(data + i);
      acc |= x.x | x.y | x.z | x.w;
    }
    acc = __syncthreads_or(acc & 0x80808080u);
    if (threadIdx.x == 0) {
      s_go = 0;
      st_rlx_sys(&rb->resp, ((r >> 32) << 1) | (acc ? 1 : 0));
    }
    __syncthreads();
    t0 = gtimer();
  }
}


// J: G CTAs each read 1/G of the bytes (zero copy); the last CTA to finish
// (global counter) stores the flag.
__global__ void k_read_multi(const uint4* p, int n16, volatile uint32_t* f, uint32_t v, unsigned* count) {
  uint32_t acc = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += gridDim.x * blockDim.x) {
    uint4 q = __ldcv(p + i);
    acc |= q.x | q.y | q.z | q.w;
  }
  acc = __syncthreads_or(acc & 0x80808080u);
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0;
      *f = v | (acc ? 0x80000000u : 0);
    }
  }
}

static void report(const char* what, std::vector<double>& v) {
  std::sort(v.begin(), v.end());
  printf("%-58s min %7.2f  med %7.2f  p99 %7.2f us\n", what, v[0], v[v.size() / 2], v[v.size() * 99 / 100]);
}

int main(int argc, char** argv) {
  const int R = 3000;
  CK(cudaSetDevice(0));
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  uint8_t* h;
  CK(cudaHostAlloc(&h, 1 << 21, cudaHostAllocMapped));
  uint8_t* dh;
  CK(cudaHostGetDevicePointer((void**)&dh, h, 0));
  Box* box = (Box*)h;
  Box* dbox = (Box*)dh;
  uint8_t* hdata = h + 4096;
  const uint4* ddata = (const uint4*)(dh + 4096);
  std::vector<uint8_t> user(1 << 20, 'a');
  volatile uint32_t* hflag = (volatile uint32_t*)(h + 2048);
  uint32_t* dflag = (uint32_t*)(dh + 2048);
  std::vector<double> t;

  for (int it = 0; it < 100; ++it) k_empty<<<1, 32, 0, s>>>();
  CK(cudaStreamSynchronize(s));
  t.clear();
  for (int i = 0; i < R; ++i) {
    double a = now_us();
    k_empty<<<1, 32, 0, s>>>();
    cudaStreamSynchronize(s);
    t.push_back(now_us() - a);
  }
  report("A  empty launch + cudaStreamSynchronize", t);

  t.clear();
  for (int i = 0; i < R; ++i) {
    double a = now_us();
    k_store<<<1, 32, 0, s>>>(dflag, i + 1);
    while (*hflag != (uint32_t)(i + 1)) {
    }
    t.push_back(now_us() - a);
  }
  CK(cudaStreamSynchronize(s));
  report("B  store-mapped-word launch + host spin", t);

  for (int n : {16, 1024, 16384, 65536}) {
    for (int thr : {256, 1024}) {
      t.clear();
      for (int i = 0; i < R; ++i) {
        double a = now_us();
        memcpy(hdata, user.data(), n);
        const uint32_t v = (uint32_t)(i + 1) & 0x7fffffffu;
        k_read<<<1, thr, 0, s>>>(ddata, (n + 15) / 16, dflag, v);
        while ((*hflag & 0x7fffffffu) != v) {
        }
        t.push_back(now_us() - a);
      }
      CK(cudaStreamSynchronize(s));
      char w[96];
      snprintf(w, sizeof w, "C  memcpy+zero-copy read %6d B, %4d thr + spin", n, thr);
      report(w, t);
    }
  }

  for (int pollers : {1, 32}) {
    for (int thr : {512, 1024}) {
      memset(box, 0, sizeof(Box));
      k_server<<<1, thr, 0, s>>>(dbox, ddata, pollers, 2000000000ull);
      CK(cudaGetLastError());
      volatile unsigned long long* vreq = &box->req;
      volatile unsigned long long* vresp = &box->resp;
      unsigned long long seq = 0;
      for (int n : {16, 1024, 16384, 65536}) {
        t.clear();
        for (int i = 0; i < R; ++i) {
          double a = now_us();
          memcpy(hdata, user.data(), n);
          ++seq;
          __atomic_thread_fence(__ATOMIC_RELEASE);
          *vreq = (seq << 32) | (unsigned)n;
          while ((*vresp >> 1) != seq) {
          }
          t.push_back(now_us() - a);
        }
        char w[96];
        snprintf(w, sizeof w, "D  server %2d poller(s) %4d thr, %6d B", pollers, thr, n);
        report(w, t);
      }
      box->stop = 1;
      CK(cudaStreamSynchronize(s));
    }
  }

  struct V { int thr, pw, stag, rlx; };
  for (V v : {V{256, 1, 0, 0}, V{256, 1, 0, 1}, V{256, 4, 250, 1}, V{256, 8, 125, 1}, V{512, 8, 125, 1},
              V{1024, 8, 125, 1}, V{256, 8, 250, 1}}) {
    memset(box, 0, sizeof(Box));
    k_server2<<<1, v.thr, 0, s>>>(dbox, ddata, v.pw, v.stag, v.rlx, 2000000000ull);
    CK(cudaGetLastError());
    volatile unsigned long long* vreq = &box->req;
    volatile unsigned long long* vresp = &box->resp;
    unsigned long long seq = 0;
    for (int n : {16, 4096, 16384, 65536}) {
      t.clear();
      for (int i = 0; i < R; ++i) {
        double a = now_us();
        memcpy(hdata, user.data(), n);
        ++seq;
        __atomic_thread_fence(__ATOMIC_RELEASE);
        *vreq = (seq << 32) | (unsigned)n;
        while ((*vresp >> 1) != seq) {
        }
        t.push_back(now_us() - a);
      }
      char w[96];
      snprintf(w, sizeof w, "F  thr %4d pollwarps %d stagger %3d rlx %d, %6d B", v.thr, v.pw, v.stag, v.rlx, n);
      report(w, t);
    }
    box->stop = 1;
    CK(cudaStreamSynchronize(s));
  }
  {
    t.clear();
    for (int i = 0; i < 200000; ++i) {
      double a = now_us();
      memcpy(hdata, user.data(), 16384);
      t.push_back(now_us() - a);
    }
    report("G  host memcpy 16 KiB into pinned", t);
  }

  // H: request word + data in write-combined pinned memory (not snooped),
  // the reply in cached pinned memory.
  {
    uint8_t* hw;
    CK(cudaHostAlloc(&hw, 1 << 21, cudaHostAllocMapped | cudaHostAllocWriteCombined));
    uint8_t* dhw;
    CK(cudaHostGetDevicePointer((void**)&dhw, hw, 0));
    Box* wbox = (Box*)hw;
    Box* dwbox = (Box*)dhw;
    uint8_t* wdata = hw + 4096;
    const uint4* dwdata = (const uint4*)(dhw + 4096);
    struct V { int thr, pw, stag; };
    for (V v : {V{256, 1, 0}, V{1024, 1, 0}, V{256, 2, 800}, V{256, 4, 400}}) {
      memset(box, 0, sizeof(Box));
      memset(wbox, 0, sizeof(Box));
      __builtin_ia32_sfence();
      k_server3<<<1, v.thr, 0, s>>>(dwbox, dbox, dwdata, v.pw, v.stag, 2000000000ull);
      CK(cudaGetLastError());
      volatile unsigned long long* vreq = &wbox->req;
      volatile unsigned long long* vresp = &box->resp;
      unsigned long long seq = 0;
      for (int n : {16, 4096, 16384, 65536}) {
        t.clear();
        for (int i = 0; i < R; ++i) {
          double a = now_us();
          memcpy(wdata, user.data(), n);
          ++seq;
          __builtin_ia32_sfence();
          *vreq = (seq << 32) | (unsigned)n;
          __builtin_ia32_sfence();
          while ((*vresp >> 1) != seq) {
          }
          t.push_back(now_us() - a);
        }
        char w[96];
        snprintf(w, sizeof w, "H  WC thr %4d pollwarps %d stagger %3d, %6d B", v.thr, v.pw, v.stag, n);
        report(w, t);
      }
      wbox->stop = 1;
      __builtin_ia32_sfence();
      CK(cudaStreamSynchronize(s));
    }
    t.clear();
    for (int i = 0; i < 20000; ++i) {
      double a = now_us();
      memcpy(wdata, user.data(), 16384);
      __builtin_ia32_sfence();
      t.push_back(now_us() - a);
    }
    report("G  host memcpy 16 KiB into WC pinned + sfence", t);
  }

  // I: the launch path with a large dynamic shared-memory request (the
  // server's 86 KB), after a grid that used little shared memory, vs none.
  {
    cudaFuncSetAttribute(k_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 << 10);
    uint8_t* dbig;
    CK(cudaMalloc(&dbig, 64 << 20));
    for (int smem : {0, 86 << 10}) {
      for (int after_grid : {0, 1}) {
        t.clear();
        for (int i = 0; i < 400; ++i) {
          if (after_grid) {
            CK(cudaMemsetAsync(dbig, i, 64 << 20, s));  // a grid-wide kernel of the runtime
            CK(cudaStreamSynchronize(s));
          }
          double a = now_us();
          memcpy(hdata, user.data(), 16384);
          const uint32_t v = (uint32_t)(i + 1) & 0x7fffffffu;
          k_read<<<1, 1024, smem, s>>>(ddata, 16384 / 16, dflag, v);
          while ((*hflag & 0x7fffffffu) != v) {
          }
          t.push_back(now_us() - a);
        }
        CK(cudaStreamSynchronize(s));
        char w[96];
        snprintf(w, sizeof w, "I  16 KiB launch+spin, dyn smem %6d, after grid %d", smem, after_grid);
        report(w, t);
      }
    }
  }

  // J: the read part spread over G SMs (is one SM's outstanding sysmem
  // read count the limit?)
  {
    unsigned* cnt;
    CK(cudaMalloc(&cnt, 4));
    CK(cudaMemset(cnt, 0, 4));
    for (int n : {16384, 65536}) {
      for (int G : {1, 2, 4, 8, 16}) {
        t.clear();
        for (int i = 0; i < 1000; ++i) {
          double a = now_us();
          memcpy(hdata, user.data(), n);
          const uint32_t v = (uint32_t)(i + 1) & 0x7fffffffu;
          k_read_multi<<<G, 1024, 0, s>>>(ddata, n / 16, dflag, v, cnt);
          while ((*hflag & 0x7fffffffu) != v) {
          }
          t.push_back(now_us() - a);
        }
        CK(cudaStreamSynchronize(s));
        char w[96];
        snprintf(w, sizeof w, "J  %6d B over %2d CTAs, launch + spin", n, G);
        report(w, t);
      }
    }
  }
  // idle exit: the server returns by itself after idle_ns
  memset(box, 0, sizeof(Box));
  double a = now_us();
  k_server<<<1, 512, 0, s>>>(dbox, ddata, 32, 100000ull);
  CK(cudaStreamSynchronize(s));
  printf("E  idle server (100 us idle limit) launch..exit: %.1f us\n", now_us() - a);
  return 0;
}
