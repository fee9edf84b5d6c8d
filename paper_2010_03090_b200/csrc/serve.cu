// serve.cu -- the small-call server: per-call latency of the drop-in
// validate_lookup on host inputs of at most kServeMax bytes.
//
// Reference path: validate_lookup / oracle-position verdicts called on short
// buffers (proj/src/lookup.cpp:39-41; the paper's throughput numbers are for
// 16 KiB in-cache inputs, and the reference's acceptance
// gate times 16 KiB calls, proj/tests/acceptance.cpp:346-383).
//
// A kernel launch plus a stream synchronisation costs 7-9 us on a B200 host
// before any byte is read (scripts/probes/latency_probe.cu, A/B).  Here one
// resident CTA (k_serve) instead waits for requests in a mailbox of mapped
// pinned host memory:
//
//   host:   memcpy the bytes into the mailbox's data area, store the request
//           word (sequence, n, lane range, mode) -- x86 stores are ordered,
//           so the data is visible before the word;
//   server: thread 0 polls the request word (ld.relaxed.sys, one PCIe round
//           trip per poll), every thread then fetches its share of the bytes
//           with ld.global.cv (never from a stale cached line) into shared
//           memory, zero-extends past n, evaluates the lead-form lane
//           predicate of chunk.cuh per 32-byte chunk, and thread 0 stores one
//           reply word (sequence, flag, and for the verdict mode the first
//           error's offset and kind from locate.cuh);
//   host:   spins on the reply word (no cudaStreamSynchronize).
//
// Measured (latency_probe D/F): 16 B calls 2.7-4.4 us, 16 KiB calls 4.8-6 us,
// against 13-15 us for a launch of K1 over zero-copy memory.
//
// Lifetime: the server exits by itself after `idle` ns without a request
// (UTF8V_CUDA_SERVE_IDLE_US, default 100 us), so a device-wide
// synchronisation by the application waits at most that long for it.  Every
// other kernel launch of this library first bumps a per-device epoch word the
// servers poll (serve_quiesce): K1/K2 size their grids to one CTA per SM and
// must not find an SM held by a server.  A server that exited (idle or
// epoch) writes its generation to the mailbox's exit word; a caller that sees
// it without its reply relaunches the server, which takes the pending request
// first.  UTF8V_CUDA_SERVE=0 disables the server (capi.cu then launches K1 over
// zero-copy memory per call).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>

#include "capi_internal.h"
#include "chunk.cuh"
#include "kernels.cuh"
#include "locate.cuh"
#include "serve.h"

namespace u8v {

namespace {

constexpr int kServeThreads = 1024;
// Bytes staged per request: chunks [0, ceil(L1/32)] (the chunk after the last
// evaluated one supplies its `next` word), L1 <= n + 3.
constexpr unsigned kStageBytes = kServeMax + 2 * kChunkBytes;
constexpr int kLoads = (kStageBytes / 16 + kServeThreads - 1) / kServeThreads;  // uint4 per thread

// Request word: n (bits 0-16), lane_lo or the record count (17-33), lane_hi
// (34-50), mode (51-52), sequence (53-63, never 0).
enum { kModeFlag = 0, kModeVerdict = 1, kModeBatch = 2 };
constexpr unsigned kSeqMax = 2047;
__host__ __device__ __forceinline__ unsigned req_seq(unsigned long long r) { return (unsigned)(r >> 53); }
__host__ __device__ __forceinline__ unsigned req_n(unsigned long long r) { return (unsigned)(r & 0x1FFFF); }
__host__ __device__ __forceinline__ unsigned req_lo(unsigned long long r) { return (unsigned)((r >> 17) & 0x1FFFF); }
__host__ __device__ __forceinline__ unsigned req_hi(unsigned long long r) { return (unsigned)((r >> 34) & 0x1FFFF); }
__host__ __device__ __forceinline__ unsigned req_mode(unsigned long long r) { return (unsigned)((r >> 51) & 3); }
// Reply word: flag (bit 0), kind + 1 (bits 1-4, 0 = none), offset (5-21),
// sequence (53-63).

// Mailbox layout in the mapped pinned buffer (one 64-byte line per word;
// batch mode: the records' 32-bit offsets and the verdicts the server
// writes back).
constexpr size_t kReqOff = 0, kRespOff = 64, kExitOff = 128, kDataOff = 256;
constexpr size_t kOffsOff = kDataOff + kStageBytes + 64;
constexpr size_t kVerOff = kOffsOff + 4 * (kServeMaxRecords + 1 + 15);
constexpr size_t kMailboxBytes = kVerOff + kServeMaxRecords + 64;
// Shared memory: the staged bytes, then (batch mode) offsets and verdicts.
constexpr size_t kSmemOffs = kStageBytes;
constexpr size_t kSmemVer = kSmemOffs + 4 * (kServeMaxRecords + 1 + 3);
constexpr size_t kSmemBytes = kSmemVer + kServeMaxRecords;

struct ServeArgs {
  const unsigned long long* req;
  unsigned long long* resp;
  unsigned long long* exit_word;
  const uint4* data;
  const uint32_t* offs;  // batch mode: R + 1 offsets (relative to the data)
  uint32_t* verdicts;    // batch mode: R verdict bytes (mapped host memory)
  const unsigned long long* epoch;
  unsigned long long epoch0;
  unsigned long long idle_ns;
  unsigned long long gen;
  unsigned long long first_req;  // the request pending at launch (taken without a poll)
  unsigned last_seq;
  u8v_consts k;
};

__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Batch mode (the K2 decomposition of batch.cu over shared memory; proven
// against per-record validation by tests/test_swar.py::test_k2_*): every
// flagged lane of the unbounded stream is attributed to its record unless
// it is one of that record's first three lanes or lies past the data, and
// every record start (and the data end) runs u8v_boundary_errors on the
// bytes around it.  R records, offsets s_off[0..R] relative to the staged
// bytes (s_off[0] = 0, s_off[R] = n); verdicts in s_ver.
__device__ __forceinline__ unsigned last_start_le(const uint32_t* s_off, unsigned R, unsigned q) {
  unsigned a = 0, b = R - 1;  // largest r in [0, R-1] with s_off[r] <= q (s_off[0] = 0 <= q)
  while (a < b) {
    const unsigned m = (a + b + 1) >> 1;
    if (s_off[m] <= q) a = m;
    else b = m - 1;
  }
  return a;
}

__device__ void serve_batch(const uint8_t* s_bytes, const uint32_t* sw, const uint32_t* s_off, uint8_t* s_ver,
                            unsigned n, unsigned R, u8v_consts k) {
  const unsigned t = threadIdx.x;
  const unsigned c_end = (n + kChunkBytes - 1) / kChunkBytes;
  for (unsigned c = t; c < c_end; c += kServeThreads) {
    Chunk v;
#pragma unroll
    for (int j = 0; j < kChunkWords; ++j) v.w[j] = sw[c * kChunkWords + j];
    const uint32_t prev = c ? sw[c * kChunkWords - 1] : 0u;
    const uint32_t next = sw[(c + 1) * kChunkWords];
    uint32_t hi7;
    uint32_t e = chunk_errors<true>(v, prev, next, k, (int64_t)c * kChunkBytes, 0, n, &hi7);
    while (e) {  // natural order: bit i = lane 32c + i
      const unsigned q = c * kChunkBytes + (unsigned)(__ffs(e) - 1);
      e &= e - 1;
      const unsigned r = last_start_le(s_off, R, q);
      if (q - s_off[r] >= 3) s_ver[r] = 0;
    }
  }
  for (unsigned rr = t; rr <= R; rr += kServeThreads) {
    const unsigned o = s_off[rr];
    uint64_t w8 = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int q = (int)o - 4 + j;
      if (q >= 0 && q < (int)n) w8 |= (uint64_t)s_bytes[q] << (8 * j);
    }
    int ka = rr > 0 ? (int)s_off[rr - 1] - ((int)o - 4) : 4;
    int kb = rr < R ? (int)s_off[rr + 1] - ((int)o - 4) : 4;
    ka = ka < 0 ? 0 : (ka > 4 ? 4 : ka);
    kb = kb < 4 ? 4 : (kb > 8 ? 8 : kb);
    const uint32_t f = u8v_boundary_errors(w8, (unsigned)ka, (unsigned)kb, k);
    if ((f & 1u) && rr > 0) s_ver[rr - 1] = 0;
    if ((f & 2u) && rr < R) s_ver[rr] = 0;
  }
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Bytes [keep, 16) of q set to zero.
__device__ __forceinline__ uint4 keep_bytes(uint4 q, unsigned keep) {
  uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = (int)keep - 4 * j;  // bytes of word j to keep
    w[j] = k >= 4 ? w[j] : (k <= 0 ? 0u : (w[j] & (0xFFFFFFFFu >> (32 - 8 * k))));
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__global__ void __launch_bounds__(kServeThreads, 1) k_serve(ServeArgs a) {
  extern __shared__ uint4 s_buf[];
  uint32_t* const s_off = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(s_buf) + kSmemOffs);
  uint8_t* const s_ver = reinterpret_cast<uint8_t*>(s_buf) + kSmemVer;
  __shared__ unsigned long long s_req;
  __shared__ unsigned s_first;
  const unsigned t = threadIdx.x;
  unsigned last = a.last_seq;
  unsigned long long t0 = global_ns();
  for (bool first = true;; first = false) {
    if (t == 0) {
      unsigned long long r = 0;
      if (first && req_seq(a.first_req) != last && req_seq(a.first_req) != 0) r = a.first_req;
      while (!r) {
        const unsigned long long q = ld_relaxed_sys(a.req);
        const unsigned long long ep = ld_relaxed_sys(a.epoch);
        if (req_seq(q) != last && req_seq(q) != 0) {
          r = q;
          break;
        }
        if (ep != a.epoch0 || global_ns() - t0 > a.idle_ns) break;
      }
      s_req = r;
      s_first = 0xFFFFFFFFu;
    }
    __syncthreads();
    const unsigned long long r = s_req;
    if (r == 0) {
      if (t == 0) st_relaxed_sys(a.exit_word, a.gen);
      return;
    }
    last = req_seq(r);
    const unsigned mode = req_mode(r);
    const unsigned n = req_n(r), L0 = mode == kModeBatch ? 0u : req_lo(r), L1 = mode == kModeBatch ? n : req_hi(r);
    const unsigned c_end = (L1 + kChunkBytes - 1) / kChunkBytes;
    const unsigned lim16 = (c_end + 1) * (kChunkBytes / 16);  // uint4 words staged
    // Every load is issued before any is used: one PCIe round trip for up
    // to kServeThreads x kLoads x 16 bytes.
    uint4 q[kLoads];
#pragma unroll
    for (int j = 0; j < kLoads; ++j) {
      const unsigned i = t + j * kServeThreads;
      q[j] = (i < lim16 && i * 16 < n) ? __ldcv(a.data + i) : make_uint4(0, 0, 0, 0);
    }
    if (mode == kModeBatch) {  // offsets in (their loads overlap the bytes'), verdicts initialised
      const unsigned R = req_lo(r);
      for (unsigned i = t; i <= R; i += kServeThreads) s_off[i] = __ldcv(a.offs + i);
      for (unsigned i = t; i < R; i += kServeThreads) s_ver[i] = 1;
    }
#pragma unroll
    for (int j = 0; j < kLoads; ++j) {
      const unsigned i = t + j * kServeThreads;
      if (i < lim16) {
        const int rem = (int)n - (int)(i * 16);  // bytes of this word inside the input
        if (rem < 16 && rem > 0) q[j] = keep_bytes(q[j], (unsigned)rem);  // the one straddling word
        s_buf[i] = q[j];
      }
    }
    __syncthreads();
    const uint32_t* sw = reinterpret_cast<const uint32_t*>(s_buf);
    if (mode == kModeBatch) {
      const unsigned R = req_lo(r);
      serve_batch(reinterpret_cast<const uint8_t*>(s_buf), sw, s_off, s_ver, n, R, a.k);
      __syncthreads();
      uint32_t bad = 0;
      for (unsigned i = t; i < (R + 3) / 4; i += kServeThreads) {
        const uint32_t w = reinterpret_cast<const uint32_t*>(s_ver)[i];
        bad |= ~w & 0x01010101u & (i * 4 + 4 <= R ? 0xFFFFFFFFu : (0xFFFFFFFFu >> (8 * (i * 4 + 4 - R))));
        a.verdicts[i] = w;  // mapped host memory
      }
      bad = __syncthreads_or(bad);
      if (t == 0) st_release_sys(a.resp, ((unsigned long long)last << 53) | (bad ? 1 : 0));  // after every verdict store
      t0 = global_ns();
      __syncthreads();
      continue;
    }
    uint32_t any = 0;
    for (unsigned c = L0 / kChunkBytes + t; c < c_end; c += kServeThreads) {
      Chunk v;
#pragma unroll
      for (int j = 0; j < kChunkWords; ++j) v.w[j] = sw[c * kChunkWords + j];
      const uint32_t prev = c ? sw[c * kChunkWords - 1] : 0u;
      const uint32_t next = sw[(c + 1) * kChunkWords];
      uint32_t hi7;
      // Interior chunks (every lane inside [L0, L1)) take the unranged form.
      const bool inside = c * kChunkBytes >= L0 && c * kChunkBytes + kChunkBytes <= L1;
      const uint32_t e = inside ? chunk_errors<false>(v, prev, next, a.k, 0, 0, 0, &hi7)
                                : chunk_errors<true>(v, prev, next, a.k, (int64_t)c * kChunkBytes, L0, L1, &hi7);
      if (e) {
        any = 1;
        atomicMin(&s_first, c);  // a thread's chunks ascend: its first is its least
        break;
      }
    }
    any = __syncthreads_or(any);
    if (t == 0) {
      unsigned long long w = ((unsigned long long)last << 53) | any;
      if (any && mode == kModeVerdict) {
        unsigned long long off = 0;
        int kind = -1;
        locate_chunk(reinterpret_cast<const uint8_t*>(s_buf), n, 0, L0, s_first, &off, &kind);
        if (kind >= 0) w |= ((unsigned long long)(kind + 1) << 1) | ((off & 0x1FFFF) << 5);
      }
      st_relaxed_sys(a.resp, w);
    }
    t0 = global_ns();
    __syncthreads();  // s_req, s_first and s_buf are rewritten for the next request
  }
}

// Per-device epoch words (mapped pinned, one line each), allocated on the
// first server launch of the device and kept for the process.
constexpr int kMaxDev = 64;
std::atomic<bool> g_any_server{false};
std::mutex g_epoch_mu;
std::atomic<unsigned long long*> g_epoch_h[kMaxDev];  // host view (set once)
unsigned long long* g_epoch_d[kMaxDev];  // device view
std::once_flag g_attr_once[kMaxDev];
std::atomic<int> g_servers[kMaxDev];  // threads holding a server, per device

bool env_disabled() {
  const char* e = getenv("UTF8V_CUDA_SERVE");
  return e && e[0] == '0';
}

unsigned long long env_idle_ns() {
  const char* e = getenv("UTF8V_CUDA_SERVE_IDLE_US");
  long v = e ? atol(e) : 100;
  if (v < 1) v = 1;
  if (v > 1000000) v = 1000000;
  return (unsigned long long)v * 1000ull;
}

int epoch_words(int dev, unsigned long long** h, unsigned long long** d) {
  std::lock_guard<std::mutex> g(g_epoch_mu);
  if (!g_epoch_h[dev].load()) {
    void* p = nullptr;
    CK(cudaHostAlloc(&p, 64, cudaHostAllocMapped | cudaHostAllocPortable));
    memset(p, 0, 64);
    void* dp = nullptr;
    CK(cudaHostGetDevicePointer(&dp, p, 0));
    g_epoch_d[dev] = static_cast<unsigned long long*>(dp);
    g_epoch_h[dev].store(static_cast<unsigned long long*>(p));
  }
  *h = g_epoch_h[dev].load();
  *d = g_epoch_d[dev];
  return UTF8V_OK;
}

}  // namespace

bool serve_enabled() {
  static const bool off = env_disabled();
  return !off;
}

void serve_quiesce() {
  if (!g_any_server.load(std::memory_order_relaxed)) return;
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return;
  unsigned long long* e = g_epoch_h[dev].load(std::memory_order_acquire);
  if (e) __atomic_fetch_add(e, 1ull, __ATOMIC_RELEASE);
}

int Server::launch() {
  unsigned long long *eh = nullptr, *ed = nullptr;
  int st = epoch_words(dev, &eh, &ed);
  if (st) return st;
  std::call_once(g_attr_once[dev], [] {
    cudaFuncSetAttribute(k_serve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
  });
  uint8_t* dh = mailbox_d;
  ServeArgs a;
  a.req = reinterpret_cast<const unsigned long long*>(dh + kReqOff);
  a.resp = reinterpret_cast<unsigned long long*>(dh + kRespOff);
  a.exit_word = reinterpret_cast<unsigned long long*>(dh + kExitOff);
  a.data = reinterpret_cast<const uint4*>(dh + kDataOff);
  a.offs = reinterpret_cast<const uint32_t*>(dh + kOffsOff);
  a.verdicts = reinterpret_cast<uint32_t*>(dh + kVerOff);
  a.epoch = ed;
  a.epoch0 = __atomic_load_n(eh, __ATOMIC_ACQUIRE);
  a.idle_ns = idle_ns;
  a.gen = ++gen;
  a.last_seq = seq == 1 ? kSeqMax : seq - 1;  // the pending request (seq) is new to it
  a.first_req = __atomic_load_n(reinterpret_cast<unsigned long long*>(mailbox_h + kReqOff), __ATOMIC_ACQUIRE);
  a.k = u8v_make_consts();
  g_any_server.store(true, std::memory_order_relaxed);
  k_serve<<<1, kServeThreads, kSmemBytes, stream>>>(a);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return u8v_capi::fail(UTF8V_ERR_CUDA, "server launch", e);
  ++launches;
  alive = true;
  return UTF8V_OK;
}

int Server::ensure(int device, bool* usable) {
  *usable = false;
  if (mailbox_h) {
    *usable = true;
    return UTF8V_OK;
  }
  if (device < 0 || device >= kMaxDev) return UTF8V_OK;
  // At most kMaxServersPerDevice threads hold a server on a device (each
  // server CTA fills an SM); the others launch a kernel per call.
  if (g_servers[device].fetch_add(1) >= kMaxServersPerDevice) {
    g_servers[device].fetch_sub(1);
    return UTF8V_OK;
  }
  dev = device;
  idle_ns = env_idle_ns();
  void* p = nullptr;
  void* dp = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaHostAlloc(&p, kMailboxBytes, cudaHostAllocMapped);
  if (e == cudaSuccess) e = cudaHostGetDevicePointer(&dp, p, 0);
  if (e != cudaSuccess) {
    if (p) cudaFreeHost(p);
    if (stream) cudaStreamDestroy(stream);
    stream = nullptr;
    g_servers[device].fetch_sub(1);
    return u8v_capi::fail(UTF8V_ERR_CUDA, "small-call server set-up", e);
  }
  memset(p, 0, kMailboxBytes);
  mailbox_h = static_cast<uint8_t*>(p);
  mailbox_d = static_cast<uint8_t*>(dp);
  *usable = true;
  return UTF8V_OK;
}

int Server::post(unsigned long long w, unsigned long long* reply) {
  seq = seq % kSeqMax + 1;
  w |= (unsigned long long)seq << 53;
  auto* req = reinterpret_cast<unsigned long long*>(mailbox_h + kReqOff);
  auto* resp = reinterpret_cast<unsigned long long*>(mailbox_h + kRespOff);
  auto* exit_word = reinterpret_cast<unsigned long long*>(mailbox_h + kExitOff);
  __atomic_store_n(req, w, __ATOMIC_RELEASE);
  if (!alive) {
    const int st = launch();
    if (st) return st;
  }
  ++requests;
  for (unsigned long long spins = 1;; ++spins) {
    unsigned long long r = __atomic_load_n(resp, __ATOMIC_ACQUIRE);
    if ((unsigned)(r >> 53) != seq && __atomic_load_n(exit_word, __ATOMIC_ACQUIRE) == gen) {
      // The server exited (idle or epoch); it wrote any reply before that.
      r = __atomic_load_n(resp, __ATOMIC_ACQUIRE);
      if ((unsigned)(r >> 53) != seq) {
        alive = false;
        const int st = launch();
        if (st) return st;
        continue;
      }
    }
    if ((unsigned)(r >> 53) == seq) {
      *reply = r;
      return UTF8V_OK;
    }
    if ((spins & 0xFFFFF) == 0) {  // a failed server never replies
      const cudaError_t e = cudaStreamQuery(stream);
      if (e != cudaSuccess && e != cudaErrorNotReady) return u8v_capi::fail(UTF8V_ERR_CUDA, "server", e);
    }
  }
}

int Server::call(const uint8_t* p, size_t n, uint64_t lane_lo, uint64_t lane_hi, bool verdict, ServeReply* out) {
  if (n == 0 || n > kServeMax || lane_hi > n + 3 || lane_lo > lane_hi)
    return u8v_capi::fail(UTF8V_ERR_ARG, "server request out of range");
  memcpy(mailbox_h + kDataOff, p, n);
  const unsigned long long w = (unsigned long long)n | ((unsigned long long)lane_lo << 17) |
                               ((unsigned long long)lane_hi << 34) |
                               ((unsigned long long)(verdict ? kModeVerdict : kModeFlag) << 51);
  unsigned long long r = 0;
  const int st = post(w, &r);
  if (st) return st;
  out->flag = (uint32_t)(r & 1);
  out->kind = (int)((r >> 1) & 0xF) - 1;
  out->offset = (r >> 5) & 0x1FFFF;
  return UTF8V_OK;
}

int Server::call_batch(const uint8_t* data, const uint64_t* offsets, size_t n_records, uint8_t* verdicts) {
  const uint64_t base = offsets[0], n = offsets[n_records] - base;
  if (n_records == 0 || n_records > kServeMaxRecords || n > kServeMax)
    return u8v_capi::fail(UTF8V_ERR_ARG, "server batch out of range");
  if (n) memcpy(mailbox_h + kDataOff, data + base, n);
  auto* offs = reinterpret_cast<uint32_t*>(mailbox_h + kOffsOff);
  for (size_t r = 0; r <= n_records; ++r) offs[r] = (uint32_t)(offsets[r] - base);
  const unsigned long long w = n | ((unsigned long long)n_records << 17) | ((unsigned long long)kModeBatch << 51);
  unsigned long long r = 0;
  const int st = post(w, &r);
  if (st) return st;
  memcpy(verdicts, mailbox_h + kVerOff, n_records);
  return UTF8V_OK;
}

void Server::release() {
  if (!mailbox_h) return;
  if (alive) {
    serve_quiesce();
    alive = false;
  }
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
  cudaFreeHost(mailbox_h);
  cudaGetLastError();
  g_servers[dev].fetch_sub(1);
  *this = Server();
}

}  // namespace u8v
