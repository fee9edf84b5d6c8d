// serve.h -- the small-call server (serve.cu): host inputs of at most
// kServeMax bytes validated by a resident CTA that polls a mailbox in mapped
// pinned memory, so a call costs PCIe round trips instead of a kernel launch
// and a stream synchronisation.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace u8v {

constexpr size_t kServeMax = 64u << 10;
constexpr size_t kServeMaxRecords = 4096;  // batch requests: records per request
constexpr int kMaxServersPerDevice = 32;   // threads holding a server on one device

struct ServeReply {
  uint32_t flag = 0;    // some lane of the range is flagged
  int kind = -1;        // verdict mode: first error's kind (verdict.hpp numbering), -1 if none
  uint64_t offset = 0;  // verdict mode: first error's byte offset
};

// One per host thread and device (capi.cu's Ctx): its mailbox, its stream,
// and what the host knows about its server.
struct Server {
  int dev = -1;
  cudaStream_t stream = nullptr;
  uint8_t* mailbox_h = nullptr;
  uint8_t* mailbox_d = nullptr;
  unsigned seq = 0;                 // last request posted (1..2047)
  unsigned long long gen = 0;       // generation of the last server launched
  unsigned long long idle_ns = 0;
  bool alive = false;               // a server of generation `gen` may be running
  unsigned long long launches = 0;  // server launches by this thread (diagnostics)
  unsigned long long requests = 0;

  // Sets up this thread's server on `device` (mailbox, stream) unless
  // kMaxServersPerDevice other threads hold one there: *usable says whether
  // the caller may use it (else it launches a kernel per call).
  int ensure(int device, bool* usable);
  // Flag of lanes [lane_lo, lane_hi) of p[0..n) (1 <= n <= kServeMax); in
  // verdict mode also the first error's (offset, kind).  Synchronous.
  int call(const uint8_t* p, size_t n, uint64_t lane_lo, uint64_t lane_hi, bool verdict, ServeReply* out);
  // One verdict per record of a host batch whose records span at most
  // kServeMax bytes (offsets[n_records] - offsets[0]), 1 <= n_records <=
  // kServeMaxRecords; offsets already checked non-decreasing.  Synchronous.
  int call_batch(const uint8_t* data, const uint64_t* offsets, size_t n_records, uint8_t* verdicts);
  void release();

 private:
  int launch();
  int post(unsigned long long w, unsigned long long* reply);  // w without its sequence
};

// False when UTF8V_CUDA_SERVE=0.
bool serve_enabled();
// Ask every server on the current device to exit (before a launch that
// needs every SM: K1/K2 grids hold one CTA per SM).  A relaxed host store
// when a server was ever started in this process, nothing otherwise.
void serve_quiesce();

}  // namespace u8v
