// capi.cu -- the extern "C" boundary (include/utf8v_cuda.h) over the sm_100a
// kernels: per-thread/per-device context, H2D pipelining for host inputs,
// status mapping.  No CPU fallback: without a CUDA device every compute entry
// point returns UTF8V_ERR_NO_DEVICE.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/utf8v_cuda.h"
#include "capi_internal.h"
#include "kernels.cuh"
#include "serve.h"

namespace u8v_capi {

thread_local std::string t_err;
thread_local int t_launches = 0;

int fail(int code, const std::string& what, cudaError_t e) {
  t_err = what;
  if (e != cudaSuccess) {
    t_err += ": ";
    t_err += cudaGetErrorString(e);
  }
  return code;
}

}  // namespace u8v_capi

using namespace u8v_capi;

namespace {

constexpr int kMaxDevices = 64;
constexpr size_t kPiece = 32ull << 20;  // H2D pipeline piece (multiple of 16)

// The reference's eight 2-byte error patterns -> three nibble tables
// (proj/include/utf8v/tables.hpp:60-99, same construction).
void build_tables(uint8_t t1[16], uint8_t t2[16], uint8_t t3[16]) {
  auto nib = [](unsigned lo, unsigned hi) {
    uint16_t m = 0;
    for (unsigned v = lo; v <= hi; ++v) m = (uint16_t)(m | (1u << v));
    return m;
  };
  struct P {
    uint8_t bit;
    uint16_t h1, l1, h2;
  };
  const P pat[8] = {
      {0, nib(0xC, 0xF), 0xFFFF, (uint16_t)(nib(0x0, 0x7) | nib(0xC, 0xF))},
      {1, nib(0x0, 0x7), 0xFFFF, nib(0x8, 0xB)},
      {2, nib(0xE, 0xE), nib(0x0, 0x0), nib(0x8, 0x9)},
      {3, nib(0xF, 0xF), nib(0x4, 0xF), nib(0x9, 0xB)},
      {4, nib(0xE, 0xE), nib(0xD, 0xD), nib(0xA, 0xB)},
      {5, nib(0xC, 0xC), nib(0x0, 0x1), nib(0x8, 0xB)},
      {6, nib(0xF, 0xF), (uint16_t)(nib(0x0, 0x0) | nib(0x5, 0xF)), nib(0x8, 0x8)},
      {7, nib(0x8, 0xB), 0xFFFF, nib(0x8, 0xB)},
  };
  memset(t1, 0, 16);
  memset(t2, 0, 16);
  memset(t3, 0, 16);
  for (const P& p : pat)
    for (unsigned n = 0; n < 16; ++n) {
      if (p.h1 & (1u << n)) t1[n] |= (uint8_t)(1u << p.bit);
      if (p.l1 & (1u << n)) t2[n] |= (uint8_t)(1u << p.bit);
      if (p.h2 & (1u << n)) t3[n] |= (uint8_t)(1u << p.bit);
    }
}

std::once_flag g_dev_once[kMaxDevices];

// Host input crosses PCIe through a bounded ring of device slots: piece k
// (about n/8 bytes, 2..32 MiB) goes to slot k % kRing together with kHalo
// bytes on either side, so K1 validates each piece's lanes as soon as its own
// copy has landed and the HBM a host call holds is kRing x (32 MiB + 2 kHalo)
// whatever n is.  Inputs of at most kSmall bytes take one copy into a
// dedicated buffer (fewer API calls: the per-call latency path).
constexpr size_t kHalo = 16;                   // >= 6 look-back (decode), >= 3 lookahead
constexpr int kRing = 4;
constexpr size_t kSlotBytes = kPiece + 2 * kHalo;
constexpr size_t kSmall = 1u << 20;
constexpr size_t kZeroCopy = 256u << 10;       // K1 reads host memory in place up to this size
constexpr size_t kKeepStage = 256ull << 20;    // batch staging kept across calls up to this size

// Per thread and device: streams, small result buffers, the device ring for
// host input, the pinned ring for pageable input, and the batch stage.
// Released when the thread exits or on utf8v_cuda_release_thread_resources().
struct Ctx {
  bool ready = false;
  int dev = -1;
  cudaStream_t s_comp = nullptr, s_copy = nullptr;
  uint32_t* d_flag = nullptr;               // [0] verdict flag
  unsigned long long* d_pos = nullptr;      // [0] first flagged step (chunk index), [1] offset
  int* d_kind = nullptr;
  uint8_t* d_lanes = nullptr;               // 3 x UTF8V_CUDA_WIDTH
  int* d_ok = nullptr;
  uint32_t* h_res = nullptr;                // pinned result words
  // Device ring (kRing slots of slot_bytes) and its events: full = the H2D
  // copy of the slot's piece landed (s_copy), free = the K1 that read the
  // slot finished (s_comp).
  uint8_t* d_ring = nullptr;
  size_t slot_bytes = 0;
  cudaEvent_t ring_full[kRing] = {}, ring_free[kRing] = {};
  // Per-piece flags of a host call (the verdict path finds its first
  // flagged piece), device and pinned host copies.
  uint32_t* d_pflags = nullptr;
  uint32_t* h_pflags = nullptr;
  size_t pflags_cap = 0;
  // Pageable input: pinned ring (kRing slots of slot_bytes) and the event of
  // the DMA that last read each slot.
  uint8_t* h_ring = nullptr;
  size_t h_slot_bytes = 0;
  cudaEvent_t hslot_done[kRing] = {};
  // Small inputs.
  uint8_t* h_small = nullptr;   // mapped pinned: K1 reads it over PCIe (zero copy)
  uint8_t* dh_small = nullptr;  // its device address
  uint8_t* d_small = nullptr;   // device copy for the small verdict path
  u8v::Server srv;              // the small-call server (serve.cu), <= kServeMax bytes
  // Batch from host memory: the whole data array (kept up to kKeepStage).
  uint8_t* d_stage = nullptr;
  size_t stage_cap = 0;
  cudaEvent_t ev_legacy = nullptr;          // see after_legacy()

  ~Ctx() { release(); }
  // Errors are ignored: at process exit the runtime may already be gone.
  void release() {
    if (dev < 0) return;
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(dev);
    srv.release();
    if (s_comp) cudaStreamSynchronize(s_comp);
    if (s_copy) cudaStreamSynchronize(s_copy);
    for (void* p : {(void*)d_flag, (void*)d_pos, (void*)d_kind, (void*)d_lanes, (void*)d_ok, (void*)d_stage,
                    (void*)d_ring, (void*)d_pflags, (void*)d_small})
      if (p) cudaFree(p);
    for (void* p : {(void*)h_res, (void*)h_ring, (void*)h_pflags, (void*)h_small})
      if (p) cudaFreeHost(p);
    for (int i = 0; i < kRing; ++i)
      for (cudaEvent_t e : {ring_full[i], ring_free[i], hslot_done[i]})
        if (e) cudaEventDestroy(e);
    if (ev_legacy) cudaEventDestroy(ev_legacy);
    if (s_comp) cudaStreamDestroy(s_comp);
    if (s_copy) cudaStreamDestroy(s_copy);
    if (cur >= 0) cudaSetDevice(cur);
    cudaGetLastError();
    *this = Ctx();
  }
  Ctx() = default;
  Ctx& operator=(const Ctx&) = default;
};
thread_local Ctx t_ctx[kMaxDevices];

int get_ctx(Ctx** out) {
  int dev = -1, count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(UTF8V_ERR_NO_DEVICE, "no CUDA device");
  }
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices)
    return fail(UTF8V_ERR_NO_DEVICE, "cudaGetDevice failed");
  std::call_once(g_dev_once[dev], [] {
    uint8_t t1[16], t2[16], t3[16];
    build_tables(t1, t2, t3);
    u8v::set_tables(t1, t2, t3);
  });
  Ctx& c = t_ctx[dev];
  if (!c.ready) {
    c.release();  // a failed earlier initialisation
    c.dev = dev;
    CK(cudaStreamCreateWithFlags(&c.s_comp, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c.s_copy, cudaStreamNonBlocking));
    CK(cudaMalloc(&c.d_flag, 64));
    CK(cudaMalloc(&c.d_pos, 64));
    CK(cudaMalloc(&c.d_kind, 64));
    CK(cudaMalloc(&c.d_lanes, 4 * UTF8V_CUDA_WIDTH));
    CK(cudaMalloc(&c.d_ok, 64));
    CK(cudaMallocHost(&c.h_res, 256));
    CK(cudaEventCreateWithFlags(&c.ev_legacy, cudaEventDisableTiming));
    for (int i = 0; i < kRing; ++i) {
      CK(cudaEventCreateWithFlags(&c.ring_full[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c.ring_free[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c.hslot_done[i], cudaEventDisableTiming));
    }
    c.ready = true;
  }
  *out = &c;
  return UTF8V_OK;
}

// Device input to the synchronous entry points is ordered like a
// synchronous cudaMemcpy: after all work issued before the call to the legacy
// default stream (and, through it, to every blocking stream).  The library
// streams are non-blocking, so the order is made explicit with one event.
int after_legacy(cudaStream_t s, cudaEvent_t ev) {
  CK(cudaEventRecord(ev, cudaStreamLegacy));
  CK(cudaStreamWaitEvent(s, ev, 0));
  return UTF8V_OK;
}

int ensure_stage(Ctx& c, size_t n) {
  if (c.stage_cap >= n) return UTF8V_OK;
  if (c.d_stage) cudaFree(c.d_stage);
  c.d_stage = nullptr;
  c.stage_cap = 0;
  size_t cap = (n + 0xFFFFF) & ~size_t(0xFFFFF);
  CK(cudaMalloc(&c.d_stage, cap));
  c.stage_cap = cap;
  return UTF8V_OK;
}

// A batch stage larger than kKeepStage is not kept past its call.
void trim_stage(Ctx& c) {
  if (c.stage_cap <= kKeepStage) return;
  cudaStreamSynchronize(c.s_comp);
  cudaFree(c.d_stage);
  c.d_stage = nullptr;
  c.stage_cap = 0;
}

// The device ring with slots of at least `slot` bytes (grown, never beyond
// kSlotBytes: pieces are at most kPiece).
int ensure_ring_dev(Ctx& c, size_t slot) {
  if (c.slot_bytes >= slot) return UTF8V_OK;
  if (c.d_ring) {
    CK(cudaStreamSynchronize(c.s_comp));
    cudaFree(c.d_ring);
  }
  c.d_ring = nullptr;
  c.slot_bytes = 0;
  CK(cudaMalloc(&c.d_ring, kRing * slot));
  c.slot_bytes = slot;
  return UTF8V_OK;
}

int ensure_pflags(Ctx& c, size_t k) {
  if (c.pflags_cap >= k) return UTF8V_OK;
  CK(cudaStreamSynchronize(c.s_comp));
  if (c.d_pflags) cudaFree(c.d_pflags);
  if (c.h_pflags) cudaFreeHost(c.h_pflags);
  c.d_pflags = nullptr;
  c.h_pflags = nullptr;
  c.pflags_cap = 0;
  const size_t cap = (k + 255) & ~size_t(255);
  CK(cudaMalloc(&c.d_pflags, cap * 4));
  CK(cudaMallocHost(&c.h_pflags, cap * 4));
  c.pflags_cap = cap;
  return UTF8V_OK;
}

int ensure_small(Ctx& c) {
  if (c.d_small) return UTF8V_OK;
  CK(cudaHostAlloc(&c.h_small, kSmall + 64, cudaHostAllocMapped));
  CK(cudaHostGetDevicePointer((void**)&c.dh_small, c.h_small, 0));
  CK(cudaMalloc(&c.d_small, kSmall + 64));
  return UTF8V_OK;
}

// Stream-ordered scratch of the batch entry points from a per-device pool
// that keeps up to kPoolKeep bytes mapped between calls: the default pool
// returns its memory at every synchronisation, and mapping it again cost
// ~0.4 ms per small host batch call.
constexpr uint64_t kPoolKeep = 256ull << 20;
cudaMemPool_t g_pool[kMaxDevices];
std::once_flag g_pool_once[kMaxDevices];

int pool_alloc(void** p, size_t bytes, cudaStream_t s) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  cudaError_t err = cudaSuccess;
  std::call_once(g_pool_once[dev], [dev, &err] {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    err = cudaMemPoolCreate(&g_pool[dev], &props);
    if (err == cudaSuccess) {
      uint64_t keep = kPoolKeep;
      err = cudaMemPoolSetAttribute(g_pool[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
  });
  if (err != cudaSuccess) return fail(UTF8V_ERR_CUDA, "cudaMemPoolCreate", err);
  if (!g_pool[dev]) return fail(UTF8V_ERR_CUDA, "no memory pool (an earlier creation failed)");
  CK(cudaMallocFromPoolAsync(p, bytes, g_pool[dev], s));
  return UTF8V_OK;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(UTF8V_ERR_CUDA, what, e);
  return UTF8V_OK;
}

// Host copy pool for pageable inputs: a pageable cudaMemcpyAsync is staged by
// the driver at ~11 GB/s on the GPU box (one CPU thread); copying each piece
// into a pinned slot with several threads and then DMA-ing the slot runs the
// PCIe link at its rate.  Workers are persistent (created once per process).
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool* pool = new CopyPool();  // never destroyed: workers outlive exit
    return *pool;
  }
  // dst[0..n) = src[0..n), split over the workers and the calling thread.
  // Concurrent callers (the API is re-entrant) take turns.
  void copy(uint8_t* dst, const uint8_t* src, size_t n) {
    const size_t parts = workers_.size() + 1;
    if (n < (4u << 20) || parts == 1) {
      memcpy(dst, src, n);
      return;
    }
    std::lock_guard<std::mutex> turn(call_m_);
    const size_t seg = ((n + parts - 1) / parts + 4095) & ~size_t(4095);
    {
      std::lock_guard<std::mutex> g(m_);
      dst_ = dst;
      src_ = src;
      n_ = n;
      seg_ = seg;
      next_.store(1);
      pending_ = parts - 1;
      ++gen_;
    }
    cv_.notify_all();
    run_segment(0);
    for (;;) {
      const size_t k = next_.fetch_add(1);
      if (k >= parts) break;
      run_segment(k);
      std::lock_guard<std::mutex> g(m_);
      --pending_;
    }
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    const unsigned n = hw > 2 ? std::min(hw - 1, 11u) : 0u;
    for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    for (auto& t : workers_) t.detach();
  }
  void run_segment(size_t k) {
    const size_t a = k * seg_;
    if (a >= n_) return;
    const size_t len = std::min(seg_, n_ - a);
    memcpy(dst_ + a, src_ + a, len);
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
      }
      for (;;) {
        const size_t k = next_.fetch_add(1);
        if (k >= workers_.size() + 1) break;
        run_segment(k);
        std::lock_guard<std::mutex> g(m_);
        if (--pending_ == 0) done_cv_.notify_all();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_m_, m_;
  std::condition_variable cv_, done_cv_;
  uint64_t gen_ = 0;
  std::atomic<size_t> next_{0};
  size_t pending_ = 0;
  uint8_t* dst_ = nullptr;
  const uint8_t* src_ = nullptr;
  size_t n_ = 0, seg_ = 0;
};

// Shard workers for utf8v_cuda_validate_sharded: worker g runs shard slot g
// of every call and persists, so its per-thread device contexts (stage,
// pinned ring) are built once, not per call.  Concurrent calls take turns.
class ShardPool {
 public:
  static ShardPool& get() {
    static ShardPool* pool = new ShardPool();  // never destroyed: workers outlive exit
    return *pool;
  }
  // Workers created so far (0 if the pool was never used).
  int size() {
    std::lock_guard<std::mutex> turn(call_m_);
    return (int)workers_.size();
  }
  // fn(g) for g in [0, n), slot g on worker g; returns when all are done.
  void run(int n, const std::function<void(int)>& fn) {
    std::lock_guard<std::mutex> turn(call_m_);
    while ((int)workers_.size() < n) {
      const int id = (int)workers_.size();
      uint64_t gen;
      {
        std::lock_guard<std::mutex> g(m_);
        gen = gen_;
      }
      workers_.emplace_back([this, id, gen] { loop(id, gen); });
      workers_.back().detach();
    }
    {
      std::lock_guard<std::mutex> g(m_);
      fn_ = &fn;
      n_ = n;
      pending_ = n;
      ++gen_;
    }
    cv_.notify_all();
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  void loop(int id, uint64_t seen) {
    for (;;) {
      const std::function<void(int)>* fn;
      int n;
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        fn = fn_;
        n = n_;
      }
      if (id >= n) continue;
      (*fn)(id);
      std::lock_guard<std::mutex> g(m_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_m_, m_;
  std::condition_variable cv_, done_cv_;
  uint64_t gen_ = 0;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0, pending_ = 0;
};

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeDevice ||
         a.type == cudaMemoryTypeManaged;
}

// The pinned ring for pageable input, slots of at least `slot` bytes.
int ensure_ring_host(Ctx& c, size_t slot) {
  if (c.h_slot_bytes >= slot) return UTF8V_OK;
  if (c.h_ring) {
    CK(cudaStreamSynchronize(c.s_copy));
    cudaFreeHost(c.h_ring);
  }
  c.h_ring = nullptr;
  c.h_slot_bytes = 0;
  CK(cudaMallocHost(&c.h_ring, kRing * slot));
  c.h_slot_bytes = slot;
  return UTF8V_OK;
}

// Piece size: about n/8 (so small inputs still pipeline), 2..32 MiB, a
// multiple of 1 MiB.
size_t piece_size(size_t n) {
  size_t p = ((n / 8) + 0xFFFFF) & ~size_t(0xFFFFF);
  if (p < (2u << 20)) p = 2u << 20;
  if (p > kPiece) p = kPiece;
  return p;
}

// Host bytes p[a, b) -> device dst on s_copy; pageable memory goes through
// the pinned ring slot `slot` (copied by the CopyPool threads; the slot is
// reused once the DMA that last read it has finished).
int h2d(Ctx& c, uint8_t* dst, const uint8_t* p, size_t a, size_t b, bool pageable, int slot) {
  if (pageable) {
    uint8_t* h = c.h_ring + (size_t)slot * c.h_slot_bytes;
    CK(cudaEventSynchronize(c.hslot_done[slot]));
    CopyPool::get().copy(h, p + a, b - a);
    CK(cudaMemcpyAsync(dst, h, b - a, cudaMemcpyHostToDevice, c.s_copy));
    CK(cudaEventRecord(c.hslot_done[slot], c.s_copy));
  } else {
    CK(cudaMemcpyAsync(dst, p + a, b - a, cudaMemcpyHostToDevice, c.s_copy));
  }
  return UTF8V_OK;
}

// Lanes [lane_lo, lane_hi) of the host stream p[0..n): piece k is copied,
// with kHalo bytes on either side, into ring slot k % kRing on s_copy and its
// own lanes are validated there by K1 on s_comp as soon as it has landed,
// while the next pieces are in flight.  Pieces holding none of the lanes are
// skipped.  Errors are ORed into c.d_flag, or, with per_piece, into
// c.d_pflags[k] (zeroed here; *n_pieces = the piece count).
int validate_host_lanes(Ctx& c, const uint8_t* p, size_t n, uint64_t lane_lo, uint64_t lane_hi,
                        bool per_piece = false, size_t* n_pieces = nullptr) {
  const size_t piece = piece_size(n);
  const size_t pieces = (n + piece - 1) / piece;
  if (n_pieces) *n_pieces = pieces;
  int st = ensure_ring_dev(c, piece + 2 * kHalo);
  if (st) return st;
  const bool pageable = !is_pinned(p);
  if (pageable) {
    st = ensure_ring_host(c, piece + 2 * kHalo);
    if (st) return st;
  }
  if (per_piece) {
    st = ensure_pflags(c, pieces);
    if (st) return st;
    CK(cudaMemsetAsync(c.d_pflags, 0, pieces * 4, c.s_comp));
  }
  for (size_t k = 0; k < pieces; ++k) {
    const size_t off = k * piece;
    const size_t end = off + piece < n ? off + piece : n;
    // This piece's lanes (the last piece also holds the end-of-input lanes).
    const uint64_t lhi_piece = k + 1 == pieces ? (uint64_t)n + 3 : (uint64_t)end;
    const uint64_t llo = off > lane_lo ? off : lane_lo, lhi = lhi_piece < lane_hi ? lhi_piece : lane_hi;
    if (llo >= lhi) continue;
    const size_t a = off - (off < kHalo ? off : kHalo);
    const size_t b = end + kHalo < n ? end + kHalo : n;
    const int slot = (int)(k % kRing);
    uint8_t* dst = c.d_ring + (size_t)slot * c.slot_bytes;
    CK(cudaStreamWaitEvent(c.s_copy, c.ring_free[slot], 0));
    st = h2d(c, dst, p, a, b, pageable, slot);
    if (st) return st;
    CK(cudaEventRecord(c.ring_full[slot], c.s_copy));
    CK(cudaStreamWaitEvent(c.s_comp, c.ring_full[slot], 0));
    u8v::launch_validate(u8v::make_desc(dst, b - a, llo - a, lhi - a), per_piece ? c.d_pflags + k : c.d_flag,
                         c.s_comp);
    ++t_launches;
    CK(cudaEventRecord(c.ring_free[slot], c.s_comp));
    st = check_launch("validate kernel");
    if (st) return st;
  }
  return UTF8V_OK;
}

// Inputs of at most kZeroCopy bytes (the per-call latency path): one host copy
// into the mapped pinned buffer, and K1 reads it there over PCIe and stores
// its flag into a mapped word -- one launch and one synchronisation, no
// copies or memsets on the stream.
int validate_small(Ctx& c, const uint8_t* p, size_t n, uint64_t lane_lo, uint64_t lane_hi, uint32_t* out) {
  int st = ensure_small(c);
  if (st) return st;
  volatile uint32_t* hflag = reinterpret_cast<volatile uint32_t*>(c.h_small + kSmall + 32);
  *hflag = 0;
  memcpy(c.h_small, p, n);
  u8v::StreamDesc d = u8v::make_desc(c.dh_small, n, lane_lo, lane_hi);
  d.flag_store = 1;
  u8v::launch_validate(d, reinterpret_cast<uint32_t*>(c.dh_small + kSmall + 32), c.s_comp);
  ++t_launches;
  st = check_launch("validate kernel");
  if (st) return st;
  CK(cudaStreamSynchronize(c.s_comp));
  *out = *hflag;
  return UTF8V_OK;
}

// Batch from host memory: the whole data array staged on the device in
// pieces (records may span any bytes).
int stage_h2d(Ctx& c, const uint8_t* p, size_t n) {
  int st = ensure_stage(c, n);
  if (st) return st;
  const size_t piece = piece_size(n);
  const bool pageable = !is_pinned(p);
  if (pageable) {
    st = ensure_ring_host(c, piece);
    if (st) return st;
  }
  for (size_t off = 0, k = 0; off < n; off += piece, ++k) {
    const size_t end = off + piece < n ? off + piece : n;
    st = h2d(c, c.d_stage + off, p, off, end, pageable, (int)(k % kRing));
    if (st) return st;
  }
  CK(cudaEventRecord(c.ring_full[0], c.s_copy));
  CK(cudaStreamWaitEvent(c.s_comp, c.ring_full[0], 0));
  return UTF8V_OK;
}

}  // namespace

extern "C" {

int utf8v_cuda_abi_version(void) { return 6; }

const char* utf8v_cuda_last_error(void) { return t_err.c_str(); }

int utf8v_cuda_last_launch_count(void) { return t_launches; }

int utf8v_cuda_serve_stats(uint64_t* out_launches, uint64_t* out_requests) {
  if (!out_launches || !out_requests) return fail(UTF8V_ERR_ARG, "NULL output");
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    cudaGetLastError();
    return fail(UTF8V_ERR_NO_DEVICE, "no CUDA device");
  }
  *out_launches = t_ctx[dev].srv.launches;
  *out_requests = t_ctx[dev].srv.requests;
  return UTF8V_OK;
}

void utf8v_cuda_release_thread_resources(void) {
  for (int d = 0; d < kMaxDevices; ++d) t_ctx[d].release();
  // Unused batch scratch the per-device pools keep mapped goes back too
  // (memory other threads still hold stays allocated).
  for (int d = 0; d < kMaxDevices; ++d)
    if (g_pool[d]) cudaMemPoolTrimTo(g_pool[d], 0);
  cudaGetLastError();
  // The persistent shard workers of utf8v_cuda_validate_sharded hold
  // per-thread contexts too: release theirs as well.
  ShardPool& pool = ShardPool::get();
  const int n = pool.size();
  if (n > 0)
    pool.run(n, [](int) {
      for (int d = 0; d < kMaxDevices; ++d) t_ctx[d].release();
    });
}

}  // extern "C"

namespace {

// The error flag of lanes [lane_lo, lane_hi) of p[0..n) (host or device),
// synchronously: device input in place, host input over the bounded ring
// (or the small-input path).
int flag_lanes(const uint8_t* p, uint64_t n, uint64_t lane_lo, uint64_t lane_hi, int is_device, uint32_t* out) {
  Ctx* c;
  int st = get_ctx(&c);
  if (st) return st;
  bool serve = false;
  if (!is_device && n <= u8v::kServeMax && u8v::serve_enabled()) {
    st = c->srv.ensure(c->dev, &serve);
    if (st) return st;
  }
  if (serve) {
    u8v::ServeReply r;
    st = c->srv.call(p, n, lane_lo, lane_hi, false, &r);
    if (st) return st;
    *out = r.flag;
    return UTF8V_OK;
  }
  if (!is_device && n <= kZeroCopy) return validate_small(*c, p, n, lane_lo, lane_hi, out);
  CK(cudaMemsetAsync(c->d_flag, 0, 4, c->s_comp));
  if (is_device) {
    st = after_legacy(c->s_comp, c->ev_legacy);
    if (st) return st;
    u8v::launch_validate(u8v::make_desc(p, n, lane_lo, lane_hi), c->d_flag, c->s_comp);
    ++t_launches;
    st = check_launch("validate kernel");
  } else if (n <= kSmall) {
    // one staged copy: host memcpy into pinned memory, one DMA, K1
    st = ensure_small(*c);
    if (st) return st;
    memcpy(c->h_small, p, n);
    CK(cudaMemcpyAsync(c->d_small, c->h_small, n, cudaMemcpyHostToDevice, c->s_comp));
    u8v::launch_validate(u8v::make_desc(c->d_small, n, lane_lo, lane_hi), c->d_flag, c->s_comp);
    ++t_launches;
    st = check_launch("validate kernel");
  } else {
    st = validate_host_lanes(*c, p, n, lane_lo, lane_hi);
  }
  if (st) return st;
  CK(cudaMemcpyAsync(c->h_res, c->d_flag, 4, cudaMemcpyDeviceToHost, c->s_comp));
  CK(cudaStreamSynchronize(c->s_comp));
  *out = c->h_res[0];
  return UTF8V_OK;
}

// Verdict of lanes [lane_lo, lane_hi) of DEVICE bytes d[0..n) on s_comp (the
// caller orders d): one K1 pass that also records its first flagged step;
// only a flagged input then runs K3, one warp that recomputes that step and
// decodes the window around its first flagged chunk.
int device_verdict(Ctx* c, const uint8_t* d, uint64_t n, uint64_t lane_lo, uint64_t lane_hi, uint8_t* out_valid,
                   uint64_t* out_offset, int* out_kind) {
  // d_pos[0] = ~0: "no flagged step" is also the verdict (K1's flag word is
  // not read here, so it needs no reset).
  CK(cudaMemsetAsync(c->d_pos, 0xFF, 8, c->s_comp));
  u8v::StreamDesc sd = u8v::make_desc(d, n, lane_lo, lane_hi);
  sd.first_step = c->d_pos;
  u8v::launch_validate(sd, c->d_flag, c->s_comp);
  ++t_launches;
  int st = check_launch("validate kernel");
  if (st) return st;
  CK(cudaMemcpyAsync(c->h_res, c->d_pos, 8, cudaMemcpyDeviceToHost, c->s_comp));
  CK(cudaStreamSynchronize(c->s_comp));
  if (c->h_res[0] == ~0u && c->h_res[1] == ~0u) return UTF8V_OK;
  u8v::launch_locate(u8v::make_desc(d, n, lane_lo, lane_hi), n, c->d_pos, c->d_pos + 1, c->d_kind, c->s_comp);
  ++t_launches;
  st = check_launch("locate kernel");
  if (st) return st;
  CK(cudaMemcpyAsync(c->h_res + 2, c->d_pos + 1, 8, cudaMemcpyDeviceToHost, c->s_comp));
  CK(cudaMemcpyAsync(c->h_res + 4, c->d_kind, 4, cudaMemcpyDeviceToHost, c->s_comp));
  CK(cudaStreamSynchronize(c->s_comp));
  uint64_t off;
  memcpy(&off, c->h_res + 2, 8);
  const int kind = (int)c->h_res[4];
  if (kind < 0) return fail(UTF8V_ERR_CUDA, "flagged input but the window decode found no error");
  *out_valid = 0;
  *out_offset = off;
  *out_kind = kind;
  return UTF8V_OK;
}

// Verdict of lanes [lane_lo, lane_hi) of p[0..n).  Host input of more than
// kSmall bytes: the ring pass records one flag per piece; the first flagged
// piece holds the first error (every lane before it is clean), so only that
// piece, with its halos, is copied again and decoded on the device.
int verdict_lanes(const uint8_t* p, uint64_t n, uint64_t lane_lo, uint64_t lane_hi, int is_device,
                  uint8_t* out_valid, uint64_t* out_offset, int* out_kind) {
  t_launches = 0;
  if (!out_valid || !out_offset || !out_kind) return fail(UTF8V_ERR_ARG, "NULL output");
  if (lane_hi > n + 3 || lane_lo > lane_hi) return fail(UTF8V_ERR_ARG, "bad lane range");
  *out_offset = 0;
  *out_kind = -1;
  *out_valid = 1;
  if (n == 0 || lane_lo == lane_hi) return UTF8V_OK;
  if (!p) return fail(UTF8V_ERR_ARG, "NULL data with n > 0");
  Ctx* c;
  int st = get_ctx(&c);
  if (st) return st;
  if (is_device) {
    st = after_legacy(c->s_comp, c->ev_legacy);
    if (st) return st;
    return device_verdict(c, p, n, lane_lo, lane_hi, out_valid, out_offset, out_kind);
  }
  bool serve = false;
  if (n <= u8v::kServeMax && u8v::serve_enabled()) {
    st = c->srv.ensure(c->dev, &serve);
    if (st) return st;
  }
  if (serve) {
    u8v::ServeReply r;
    st = c->srv.call(p, n, lane_lo, lane_hi, true, &r);
    if (st) return st;
    if (!r.flag) return UTF8V_OK;
    if (r.kind < 0) return fail(UTF8V_ERR_CUDA, "flagged input but the window decode found no error");
    *out_valid = 0;
    *out_offset = r.offset;
    *out_kind = r.kind;
    return UTF8V_OK;
  }
  if (n <= kSmall) {
    st = ensure_small(*c);
    if (st) return st;
    memcpy(c->h_small, p, n);
    CK(cudaMemcpyAsync(c->d_small, c->h_small, n, cudaMemcpyHostToDevice, c->s_comp));
    return device_verdict(c, c->d_small, n, lane_lo, lane_hi, out_valid, out_offset, out_kind);
  }
  size_t pieces = 0;
  st = validate_host_lanes(*c, p, n, lane_lo, lane_hi, true, &pieces);
  if (st) return st;
  CK(cudaMemcpyAsync(c->h_pflags, c->d_pflags, pieces * 4, cudaMemcpyDeviceToHost, c->s_comp));
  CK(cudaStreamSynchronize(c->s_comp));
  size_t k = 0;
  while (k < pieces && c->h_pflags[k] == 0) ++k;
  if (k == pieces) return UTF8V_OK;
  const size_t piece = piece_size(n);
  const size_t off = k * piece;
  const size_t end = off + piece < n ? off + piece : n;
  const uint64_t lhi_piece = k + 1 == pieces ? (uint64_t)n + 3 : (uint64_t)end;
  const uint64_t llo = off > lane_lo ? off : lane_lo, lhi = lhi_piece < lane_hi ? lhi_piece : lane_hi;
  const size_t a = off - (off < kHalo ? off : kHalo);
  const size_t b = end + kHalo < n ? end + kHalo : n;
  uint8_t* dst = c->d_ring;  // slot 0; the ring pass has finished (synchronised above)
  st = h2d(*c, dst, p, a, b, !is_pinned(p), 0);
  if (st) return st;
  CK(cudaEventRecord(c->ring_full[0], c->s_copy));
  CK(cudaStreamWaitEvent(c->s_comp, c->ring_full[0], 0));
  st = device_verdict(c, dst, b - a, llo - a, lhi - a, out_valid, out_offset, out_kind);
  if (st) return st;
  if (!*out_valid) *out_offset += a;
  else return fail(UTF8V_ERR_CUDA, "flagged piece but its decode found no error");
  return UTF8V_OK;
}

}  // namespace

extern "C" {

int utf8v_cuda_validate(const uint8_t* p, size_t n, int is_device, uint8_t* out_valid) {
  t_launches = 0;
  if (!out_valid) return fail(UTF8V_ERR_ARG, "out_valid is NULL");
  if (n == 0) {
    *out_valid = 1;
    return UTF8V_OK;
  }
  if (!p) return fail(UTF8V_ERR_ARG, "NULL data with n > 0");
  uint32_t flag = 0;
  const int st = flag_lanes(p, n, 0, (uint64_t)n + 3, is_device, &flag);
  if (st) return st;
  *out_valid = flag == 0 ? 1 : 0;
  return UTF8V_OK;
}

int utf8v_cuda_validate_verdict(const uint8_t* p, size_t n, int is_device, uint8_t* out_valid,
                                uint64_t* out_offset, int* out_kind) {
  return verdict_lanes(p, n, 0, (uint64_t)n + 3, is_device, out_valid, out_offset, out_kind);
}

int utf8v_cuda_validate_verdict_lanes(const uint8_t* p, uint64_t n, uint64_t lane_lo, uint64_t lane_hi,
                                      int is_device, uint8_t* out_valid, uint64_t* out_offset,
                                      int* out_kind) {
  return verdict_lanes(p, n, lane_lo, lane_hi, is_device, out_valid, out_offset, out_kind);
}

int utf8v_cuda_validate_lanes_async(const uint8_t* d_p, uint64_t n, uint64_t lane_lo,
                                    uint64_t lane_hi, uint32_t* d_flag, void* stream) {
  t_launches = 0;
  if (lane_hi > n + 3 || lane_lo > lane_hi || !d_flag) return fail(UTF8V_ERR_ARG, "bad lane range");
  if (lane_lo == lane_hi || n == 0) return UTF8V_OK;
  if (!d_p) return fail(UTF8V_ERR_ARG, "NULL data");
  Ctx* c;
  int st = get_ctx(&c);
  if (st) return st;
  u8v::launch_validate(u8v::make_desc(d_p, n, lane_lo, lane_hi), d_flag, (cudaStream_t)stream);
  ++t_launches;
  return check_launch("validate kernel");
}

int utf8v_cuda_validate_lanes(const uint8_t* p, uint64_t n, uint64_t lane_lo, uint64_t lane_hi,
                              int is_device, uint32_t* out_flag) {
  t_launches = 0;
  if (!out_flag) return fail(UTF8V_ERR_ARG, "out_flag is NULL");
  if (lane_hi > n + 3 || lane_lo > lane_hi) return fail(UTF8V_ERR_ARG, "bad lane range");
  *out_flag = 0;
  if (lane_lo == lane_hi || n == 0) return UTF8V_OK;
  if (!p) return fail(UTF8V_ERR_ARG, "NULL data");
  return flag_lanes(p, n, lane_lo, lane_hi, is_device, out_flag);
}

int utf8v_cuda_validate_batch_async(const uint8_t* d_data, uint64_t n, const uint64_t* d_offsets,
                                    uint64_t n_records, uint8_t* d_verdicts, void* stream) {
  t_launches = 0;
  if (n_records == 0) return UTF8V_OK;
  if (!d_offsets || !d_verdicts) return fail(UTF8V_ERR_ARG, "NULL offsets/verdicts");
  Ctx* c;
  int st = get_ctx(&c);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (n > 0 && !d_data) return fail(UTF8V_ERR_ARG, "NULL data");
  // No host round trip: the kernel reads the first/last offsets itself.
  u8v::launch_batch(d_data, n, d_offsets, n_records, d_verdicts, s);
  t_launches += n > 0 ? 2 : 1;  // verdict initialisation + K2 / K2L
  return check_launch("batch kernel");
}

int utf8v_cuda_validate_batch(const uint8_t* data, size_t n, const uint64_t* offsets,
                              size_t n_records, int is_device, uint8_t* verdicts) {
  t_launches = 0;
  if (n_records == 0) return UTF8V_OK;
  if (!offsets || !verdicts) return fail(UTF8V_ERR_ARG, "NULL offsets/verdicts");
  if (is_device) {
    Ctx* c;
    int st = get_ctx(&c);
    if (st) return st;
    st = after_legacy(c->s_comp, c->ev_legacy);
    if (st) return st;
    st = utf8v_cuda_validate_batch_async(data, n, offsets, n_records, verdicts, c->s_comp);
    if (st) return st;
    CK(cudaStreamSynchronize(c->s_comp));
    return UTF8V_OK;
  }
  // Host arrays: validate the offsets here (cheap), stage everything.
  for (size_t r = 0; r < n_records; ++r)
    if (offsets[r + 1] < offsets[r]) return fail(UTF8V_ERR_ARG, "offsets not non-decreasing");
  if (offsets[n_records] > n) return fail(UTF8V_ERR_ARG, "offsets exceed data size");
  Ctx* c;
  int st = get_ctx(&c);
  if (st) return st;
  if (u8v::serve_enabled() && n_records <= u8v::kServeMaxRecords &&
      offsets[n_records] - offsets[0] <= u8v::kServeMax) {  // small batch: the server
    bool serve = false;
    st = c->srv.ensure(c->dev, &serve);
    if (st) return st;
    if (serve) return c->srv.call_batch(data, offsets, n_records, verdicts);
  }
  uint64_t* d_off = nullptr;
  uint8_t* d_ver = nullptr;
  st = pool_alloc((void**)&d_off, (n_records + 1) * 8, c->s_comp);
  if (st) return st;
  st = pool_alloc((void**)&d_ver, n_records, c->s_comp);
  if (st) {
    cudaFreeAsync(d_off, c->s_comp);
    return st;
  }
  CK(cudaMemcpyAsync(d_off, offsets, (n_records + 1) * 8, cudaMemcpyHostToDevice, c->s_comp));
  if (n > 0) {
    st = stage_h2d(*c, data, n);
    if (st) return st;
  }
  u8v::launch_batch(n > 0 ? c->d_stage : nullptr, n, d_off, n_records, d_ver, c->s_comp);
  t_launches += n > 0 ? 2 : 1;
  st = check_launch("batch kernel");
  if (st) return st;
  CK(cudaMemcpyAsync(verdicts, d_ver, n_records, cudaMemcpyDeviceToHost, c->s_comp));
  CK(cudaFreeAsync(d_off, c->s_comp));
  CK(cudaFreeAsync(d_ver, c->s_comp));
  CK(cudaStreamSynchronize(c->s_comp));
  trim_stage(*c);
  return UTF8V_OK;
}

static int lanes_call(const uint8_t* input, const uint8_t* previous, uint8_t* out, int mode) {
  t_launches = 0;
  if (!input || !out || (mode != 2 && !previous)) return fail(UTF8V_ERR_ARG, "NULL lane buffer");
  Ctx* c;
  int st = get_ctx(&c);
  if (st) return st;
  const int W = UTF8V_CUDA_WIDTH;
  CK(cudaMemcpyAsync(c->d_lanes, input, W, cudaMemcpyHostToDevice, c->s_comp));
  if (mode != 2)
    CK(cudaMemcpyAsync(c->d_lanes + W, previous, W, cudaMemcpyHostToDevice, c->s_comp));
  u8v::launch_classify_lanes(c->d_lanes, c->d_lanes + W, c->d_lanes + 2 * W, mode, c->s_comp);
  ++t_launches;
  st = check_launch("lanes kernel");
  if (st) return st;
  CK(cudaMemcpyAsync(out, c->d_lanes + 2 * W, W, cudaMemcpyDeviceToHost, c->s_comp));
  CK(cudaStreamSynchronize(c->s_comp));
  return UTF8V_OK;
}

int utf8v_cuda_classify_lanes(const uint8_t* input, const uint8_t* previous, uint8_t* out) {
  return lanes_call(input, previous, out, 0);
}

int utf8v_cuda_length_error_lanes(const uint8_t* input, const uint8_t* previous, uint8_t* out) {
  return lanes_call(input, previous, out, 1);
}

int utf8v_cuda_incomplete_lanes(const uint8_t* input, uint8_t* out) {
  return lanes_call(input, nullptr, out, 2);
}

int utf8v_cuda_ops_self_test(uint64_t seed, int* out_ok) {
  t_launches = 0;
  if (!out_ok) return fail(UTF8V_ERR_ARG, "out_ok is NULL");
  Ctx* c;
  int st = get_ctx(&c);
  if (st) return st;
  u8v::launch_ops_self_test(seed, c->d_ok, c->s_comp);
  ++t_launches;
  st = check_launch("self-test kernel");
  if (st) return st;
  CK(cudaMemcpyAsync(c->h_res, c->d_ok, 4, cudaMemcpyDeviceToHost, c->s_comp));
  CK(cudaStreamSynchronize(c->s_comp));
  *out_ok = (int)c->h_res[0];
  return UTF8V_OK;
}

// ---- composable segment states (utf8v_state.h) -------------------------------
static_assert(sizeof(utf8v_state) == sizeof(u8v_state) && sizeof(utf8v_state) == 24, "utf8v_state layout");

static u8v_state to_u8v(const utf8v_state* s) {
  u8v_state r;
  memcpy(&r, s, sizeof r);
  return r;
}

int utf8v_state_combine(const utf8v_state* a, const utf8v_state* b, utf8v_state* out) {
  if (!a || !b || !out) return fail(UTF8V_ERR_ARG, "NULL state");
  const u8v_state r = u8v_state_combine(to_u8v(a), to_u8v(b));
  memcpy(out, &r, sizeof r);
  return UTF8V_OK;
}

int utf8v_state_valid(const utf8v_state* s) { return s && u8v_state_errors(to_u8v(s)) == 0 ? 1 : 0; }

int utf8v_cuda_segment_state(const uint8_t* p, size_t n, int is_device, utf8v_state* out) {
  t_launches = 0;
  if (!out) return fail(UTF8V_ERR_ARG, "NULL state");
  u8v_state s = u8v_state_empty();
  s.len = n;
  if (n > 0 && !p) return fail(UTF8V_ERR_ARG, "NULL data with n > 0");
  const size_t k = n < 4 ? n : 4;
  if (n > 4) {
    uint32_t flag = 0;
    const int st = flag_lanes(p, n, 3, n - 1, is_device, &flag);  // the interior lanes
    if (st) return st;
    s.flag = flag ? 1u : 0u;
  }
  if (k > 0) {
    if (is_device) {
      Ctx* c;
      const int st = get_ctx(&c);
      if (st) return st;
      uint8_t* h = reinterpret_cast<uint8_t*>(c->h_res);
      CK(cudaMemcpyAsync(h, p, k, cudaMemcpyDeviceToHost, c->s_comp));
      CK(cudaMemcpyAsync(h + 8, p + n - k, k, cudaMemcpyDeviceToHost, c->s_comp));
      CK(cudaStreamSynchronize(c->s_comp));
      memcpy(s.head, h, k);
      memcpy(s.tail + 4 - k, h + 8, k);
    } else {
      memcpy(s.head, p, k);
      memcpy(s.tail + 4 - k, p + n - k, k);
    }
  }
  memcpy(out, &s, sizeof s);
  return UTF8V_OK;
}

int utf8v_cuda_batch_states_async(const uint8_t* d_data, uint64_t n, const uint64_t* d_offsets,
                                  uint64_t n_records, utf8v_state* d_states, void* stream) {
  t_launches = 0;
  if (n_records == 0) return UTF8V_OK;
  if (!d_offsets || !d_states) return fail(UTF8V_ERR_ARG, "NULL offsets/states");
  if (n > 0 && !d_data) return fail(UTF8V_ERR_ARG, "NULL data");
  Ctx* c;
  int st = get_ctx(&c);
  if (st) return st;
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* d_clean = nullptr;
  st = pool_alloc((void**)&d_clean, n_records, s);
  if (st) return st;
  u8v::launch_batch(d_data, n, d_offsets, n_records, d_clean, s, true);
  u8v::launch_record_states(d_data, n, d_offsets, n_records, d_clean, reinterpret_cast<u8v_state*>(d_states), s);
  t_launches += n > 0 ? 3 : 2;
  CK(cudaFreeAsync(d_clean, s));
  return check_launch("batch state kernels");
}

int utf8v_cuda_batch_states(const uint8_t* data, size_t n, const uint64_t* offsets, size_t n_records,
                            int is_device, utf8v_state* states) {
  t_launches = 0;
  if (n_records == 0) return UTF8V_OK;
  if (!offsets || !states) return fail(UTF8V_ERR_ARG, "NULL offsets/states");
  Ctx* c;
  int st = get_ctx(&c);
  if (st) return st;
  if (is_device) {
    st = after_legacy(c->s_comp, c->ev_legacy);
    if (st) return st;
    st = utf8v_cuda_batch_states_async(data, n, offsets, n_records, states, c->s_comp);
    if (st) return st;
    CK(cudaStreamSynchronize(c->s_comp));
    return UTF8V_OK;
  }
  for (size_t r = 0; r < n_records; ++r)
    if (offsets[r + 1] < offsets[r]) return fail(UTF8V_ERR_ARG, "offsets not non-decreasing");
  if (offsets[n_records] > n) return fail(UTF8V_ERR_ARG, "offsets exceed data size");
  uint64_t* d_off = nullptr;
  utf8v_state* d_st = nullptr;
  st = pool_alloc((void**)&d_off, (n_records + 1) * 8, c->s_comp);
  if (st) return st;
  st = pool_alloc((void**)&d_st, n_records * sizeof(utf8v_state), c->s_comp);
  if (st) {
    cudaFreeAsync(d_off, c->s_comp);
    return st;
  }
  CK(cudaMemcpyAsync(d_off, offsets, (n_records + 1) * 8, cudaMemcpyHostToDevice, c->s_comp));
  if (n > 0) {
    st = stage_h2d(*c, data, n);
    if (st) return st;
  }
  st = utf8v_cuda_batch_states_async(n > 0 ? c->d_stage : nullptr, n, d_off, n_records, d_st, c->s_comp);
  if (st) return st;
  CK(cudaMemcpyAsync(states, d_st, n_records * sizeof(utf8v_state), cudaMemcpyDeviceToHost, c->s_comp));
  CK(cudaFreeAsync(d_off, c->s_comp));
  CK(cudaFreeAsync(d_st, c->s_comp));
  CK(cudaStreamSynchronize(c->s_comp));
  trim_stage(*c);
  return UTF8V_OK;
}

int utf8v_cuda_states_reduce_async(const utf8v_state* d_states, uint64_t count, utf8v_state* d_out,
                                   void* stream) {
  t_launches = 0;
  if (!d_out || (count > 0 && !d_states)) return fail(UTF8V_ERR_ARG, "NULL states");
  Ctx* c;
  const int st = get_ctx(&c);
  if (st) return st;
  u8v::launch_states_reduce(reinterpret_cast<const u8v_state*>(d_states), count,
                            reinterpret_cast<u8v_state*>(d_out), (cudaStream_t)stream);
  ++t_launches;
  return check_launch("state reduce kernel");
}

// ---- one process, several GPUs ----
int utf8v_cuda_validate_sharded(const uint8_t* p, size_t n, int n_gpus, int is_device,
                                uint8_t* out_valid) {
  t_launches = 0;
  if (!out_valid) return fail(UTF8V_ERR_ARG, "out_valid is NULL");
  if (n_gpus < 1) return fail(UTF8V_ERR_ARG, "n_gpus must be >= 1");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(UTF8V_ERR_NO_DEVICE, "no CUDA device");
  }
  // Device input lives on one GPU: validated there.  Shards under 1 MiB: one GPU.
  if (is_device || n_gpus == 1 || n < (size_t)n_gpus * (1u << 20))
    return utf8v_cuda_validate(p, n, is_device, out_valid);
  if (!p) return fail(UTF8V_ERR_ARG, "NULL data with n > 0");
  // Shards as sharding.plan: cuts at floor(k n / G) rounded down to 16 bytes,
  // a look-back head of up to 16 bytes, a 1-byte lookahead tail (not on the
  // last shard, which also evaluates the end-of-input lanes n..n+2).
  std::vector<uint64_t> cut(n_gpus + 1);
  for (int k = 0; k <= n_gpus; ++k)
    cut[k] = k == n_gpus ? n : ((uint64_t)k * n / (uint64_t)n_gpus) & ~uint64_t(15);
  std::vector<uint32_t> flags(n_gpus, 0);
  std::vector<int> status(n_gpus, UTF8V_OK);
  std::vector<std::string> errs(n_gpus);
  std::vector<int> launches(n_gpus, 0);
  int caller_dev = 0;
  cudaGetDevice(&caller_dev);
  ShardPool::get().run(n_gpus, [&](int g) {
    // Shards go round-robin over the visible devices.
    if (cudaSetDevice(g % count) != cudaSuccess) {
      status[g] = fail(UTF8V_ERR_CUDA, "cudaSetDevice", cudaGetLastError());
      errs[g] = t_err;
      return;
    }
    const uint64_t s = cut[g], e = cut[g + 1];
    const uint64_t head = s < 16 ? s : 16;
    const bool last = g == n_gpus - 1;
    const uint64_t lo = s - head, hi = last ? e : e + 1;
    const uint64_t lane_hi = last ? (hi - lo) + 3 : head + (e - s);
    status[g] = utf8v_cuda_validate_lanes(p + lo, hi - lo, head, lane_hi, 0, &flags[g]);
    launches[g] = t_launches;
    if (status[g]) errs[g] = t_err;
  });
  cudaSetDevice(caller_dev);
  uint32_t any = 0;
  for (int g = 0; g < n_gpus; ++g) {
    if (status[g]) return fail(status[g], "GPU " + std::to_string(g) + ": " + errs[g]);
    any |= flags[g];
    t_launches += launches[g];
  }
  *out_valid = any == 0 ? 1 : 0;
  return UTF8V_OK;
}

// ---- streaming session (utf8v_stream.h) ------------------------------------
struct utf8v_cuda_stream {
  int dev = 0;
  cudaStream_t s = nullptr;
  uint32_t* d_state = nullptr;  // [0] carry, [1] error flag
  uint32_t* h_res = nullptr;    // pinned
  uint8_t* d_buf = nullptr;     // staging for host pieces
  size_t cap = 0;
  uint64_t total = 0;
  cudaEvent_t ev_legacy = nullptr;  // see after_legacy()
};

int utf8v_cuda_stream_create(utf8v_cuda_stream** out) {
  if (!out) return fail(UTF8V_ERR_ARG, "NULL out");
  *out = nullptr;
  Ctx* c;
  int st = get_ctx(&c);
  if (st) return st;
  utf8v_cuda_stream* s = new utf8v_cuda_stream();
  cudaGetDevice(&s->dev);
  if (cudaStreamCreateWithFlags(&s->s, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&s->d_state, 64) != cudaSuccess || cudaMallocHost(&s->h_res, 64) != cudaSuccess ||
      cudaEventCreateWithFlags(&s->ev_legacy, cudaEventDisableTiming) != cudaSuccess ||
      cudaMemsetAsync(s->d_state, 0, 64, s->s) != cudaSuccess) {
    const cudaError_t e = cudaGetLastError();
    utf8v_cuda_stream_destroy(s);
    return fail(UTF8V_ERR_CUDA, "stream session allocation", e);
  }
  *out = s;
  return UTF8V_OK;
}

int utf8v_cuda_stream_feed(utf8v_cuda_stream* s, const uint8_t* p, size_t n, int is_device) {
  t_launches = 0;
  if (!s) return fail(UTF8V_ERR_ARG, "NULL session");
  if (n == 0) return UTF8V_OK;
  if (!p) return fail(UTF8V_ERR_ARG, "NULL piece");
  DeviceGuard guard;
  CK(cudaSetDevice(s->dev));
  const uint8_t* d = p;
  if (is_device) {
    const int st = after_legacy(s->s, s->ev_legacy);
    if (st) return st;
  } else {
    if (s->cap < n) {
      if (s->d_buf) {
        CK(cudaStreamSynchronize(s->s));
        cudaFree(s->d_buf);
      }
      s->d_buf = nullptr;
      s->cap = 0;
      const size_t cap = (n + 0xFFFFF) & ~size_t(0xFFFFF);
      CK(cudaMalloc(&s->d_buf, cap));
      s->cap = cap;
    }
    CK(cudaMemcpyAsync(s->d_buf, p, n, cudaMemcpyHostToDevice, s->s));
    d = s->d_buf;
  }
  // The piece's own lanes in place; K1's first thread also runs the lanes
  // straddling the previous piece (a piece too short for K1 lanes runs them
  // in the one-thread edge kernel).
  u8v::StreamDesc desc = u8v::make_desc(d, n, 3, n > 4 ? n - 1 : 3);
  if (desc.steps > 0) {
    desc.session = s->d_state;
    // Device pieces overlap the previous feed's K1 (the only other work on
    // the session stream); a host piece's K1 follows its own H2D copy (PDL
    // does not reach across a copy).
    u8v::launch_validate_piece(desc, s->d_state + 1, s->s);
  } else {
    u8v::launch_stream_edge(s->d_state, d, n, 0, s->s);
  }
  ++t_launches;
  s->total += n;
  // A device piece is read asynchronously (and consecutive feeds overlap):
  // it must stay valid and unmodified until finish() returns.  A host piece
  // is consumed here: the caller may reuse its buffer.
  if (!is_device) CK(cudaStreamSynchronize(s->s));
  return check_launch("stream feed");
}

int utf8v_cuda_stream_finish(utf8v_cuda_stream* s, uint8_t* out_valid) {
  t_launches = 0;
  if (!s || !out_valid) return fail(UTF8V_ERR_ARG, "NULL session/out_valid");
  DeviceGuard guard;
  CK(cudaSetDevice(s->dev));
  u8v::launch_stream_edge(s->d_state, nullptr, 0, 1, s->s);
  ++t_launches;
  CK(cudaMemcpyAsync(s->h_res, s->d_state + 1, 4, cudaMemcpyDeviceToHost, s->s));
  CK(cudaMemsetAsync(s->d_state, 0, 8, s->s));  // ready for the next stream
  CK(cudaStreamSynchronize(s->s));
  *out_valid = s->h_res[0] == 0 ? 1 : 0;
  s->total = 0;
  return check_launch("stream finish");
}

uint64_t utf8v_cuda_stream_bytes(const utf8v_cuda_stream* s) { return s ? s->total : 0; }

void utf8v_cuda_stream_destroy(utf8v_cuda_stream* s) {
  if (!s) return;
  if (s->s) cudaStreamSynchronize(s->s);
  if (s->d_buf) cudaFree(s->d_buf);
  if (s->d_state) cudaFree(s->d_state);
  if (s->h_res) cudaFreeHost(s->h_res);
  if (s->ev_legacy) cudaEventDestroy(s->ev_legacy);
  if (s->s) cudaStreamDestroy(s->s);
  delete s;
}

}  // extern "C"
