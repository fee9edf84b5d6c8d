// comm.cu -- the multi-GPU combine of shard verdicts in the native layer
// (include/utf8v_cuda.h "multi-GPU").
//
// A stream sharded over G GPUs is valid iff no rank's lanes hold an error,
// so the shards' verdicts combine with one 4-byte allreduce(MAX) of the rank
// flags, and the first error with one 8-byte allreduce(MIN) of
// offset * 8 + kind (sharding.py states why both are exact).  Two forms:
//
//   NCCL     utf8v_cuda_comm: K1 on the caller's stream, then
//            ncclAllReduce on the same stream (NVLink / NVSwitch; NVLS when
//            NCCL picks it).  Multi-process (one rank per GPU, unique id
//            passed by the caller's bootstrap) or one process driving
//            several GPUs (ncclCommInitAll).  NCCL is loaded with dlopen on
//            first use (the torch-bundled libnccl.so.2 when torch is already
//            loaded, else the system one), so the library itself never
//            requires it; failures return UTF8V_ERR_NCCL.
//   P2P      utf8v_cuda_p2p: the collective folded into K1.  Every rank's
//            flag word is mapped into every other rank (CUDA IPC over
//            NVLink); a warp of K1 that finds an error ORs 1 into all of
//            them (validate.cu, sweep()).  On valid input nothing crosses
//            NVLink and no collective is launched, so consecutive K1
//            launches keep their programmatic overlap.  A rank's word holds
//            the global verdict once every rank's K1 over the stream has
//            completed (the caller's barrier).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/utf8v_cuda.h"
#include "capi_internal.h"
#include "kernels.cuh"

using namespace u8v_capi;

namespace {

// ---- NCCL, loaded on first use ----------------------------------------------
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;

const NcclApi& nccl() {
  std::call_once(g_nccl_once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      g_nccl.why = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))sym("ncclGetUniqueId");
    g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))sym("ncclCommInitRank");
    g_nccl.CommInitAll = (decltype(g_nccl.CommInitAll))sym("ncclCommInitAll");
    g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))sym("ncclCommDestroy");
    g_nccl.AllReduce = (decltype(g_nccl.AllReduce))sym("ncclAllReduce");
    g_nccl.GroupStart = (decltype(g_nccl.GroupStart))sym("ncclGroupStart");
    g_nccl.GroupEnd = (decltype(g_nccl.GroupEnd))sym("ncclGroupEnd");
    g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))sym("ncclGetErrorString");
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommInitAll && g_nccl.CommDestroy &&
                g_nccl.AllReduce && g_nccl.GroupStart && g_nccl.GroupEnd && g_nccl.GetErrorString;
    if (!g_nccl.ok) g_nccl.why = "libnccl.so.2 lacks a required symbol";
  });
  return g_nccl;
}

int nccl_fail(const char* what, ncclResult_t r) {
  std::string m = what;
  if (g_nccl.GetErrorString) {
    m += ": ";
    m += g_nccl.GetErrorString(r);
  }
  return fail(UTF8V_ERR_NCCL, m);
}

#define NK(call)                                          \
  do {                                                    \
    ncclResult_t _r = (call);                             \
    if (_r != ncclSuccess) return nccl_fail(#call, _r);   \
  } while (0)

#define NEED_NCCL()                                                      \
  do {                                                                   \
    if (!nccl().ok) return fail(UTF8V_ERR_NCCL, nccl().why);             \
  } while (0)

}  // namespace

struct utf8v_cuda_comm {
  int dev = 0, nranks = 1, rank = 0;
  ncclComm_t nccl = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t ev_legacy = nullptr;  // orders device input after the legacy default stream
  uint32_t* d_buf = nullptr;  // [0] local flag, [1] global flag, [2..3] 64-bit MIN key, [4..5] result
  uint32_t* h_buf = nullptr;  // pinned
};

struct utf8v_cuda_p2p {
  int dev = 0, nranks = 1, rank = 0;
  uint32_t* d_flag = nullptr;               // this rank's flag word (64 B allocation)
  std::vector<void*> opened;                // peers' flag words, IPC-mapped
  uint32_t** d_peers = nullptr;             // device array of the nranks-1 peer words
  cudaStream_t s = nullptr;
  uint32_t* h_res = nullptr;
};

namespace {

int comm_alloc(utf8v_cuda_comm* c) {
  CK(cudaStreamCreateWithFlags(&c->s, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_legacy, cudaEventDisableTiming));
  CK(cudaMalloc(&c->d_buf, 64));
  CK(cudaMemset(c->d_buf, 0, 64));
  CK(cudaMallocHost(&c->h_buf, 64));
  return UTF8V_OK;
}

void comm_free(utf8v_cuda_comm* c) {
  if (!c) return;
  DeviceGuard g;
  cudaSetDevice(c->dev);
  if (c->s) cudaStreamSynchronize(c->s);
  if (c->nccl && g_nccl.CommDestroy) g_nccl.CommDestroy(c->nccl);
  if (c->d_buf) cudaFree(c->d_buf);
  if (c->h_buf) cudaFreeHost(c->h_buf);
  if (c->ev_legacy) cudaEventDestroy(c->ev_legacy);
  if (c->s) cudaStreamDestroy(c->s);
  cudaGetLastError();
  delete c;
}

int bad_lanes(uint64_t n, uint64_t lane_lo, uint64_t lane_hi) {
  if (lane_hi > n + 3 || lane_lo > lane_hi) return fail(UTF8V_ERR_ARG, "bad lane range");
  return UTF8V_OK;
}

}  // namespace

extern "C" {

// ---- NCCL communicators --------------------------------------------------------
int utf8v_cuda_comm_unique_id(uint8_t* out_id) {
  if (!out_id) return fail(UTF8V_ERR_ARG, "NULL out_id");
  NEED_NCCL();
  ncclUniqueId id;
  NK(nccl().GetUniqueId(&id));
  memcpy(out_id, id.internal, UTF8V_COMM_ID_BYTES);
  return UTF8V_OK;
}

int utf8v_cuda_comm_init_rank(const uint8_t* id, int nranks, int rank, utf8v_cuda_comm** out) {
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(UTF8V_ERR_ARG, "bad comm arguments");
  *out = nullptr;
  NEED_NCCL();
  utf8v_cuda_comm* c = new utf8v_cuda_comm();
  cudaGetDevice(&c->dev);
  c->nranks = nranks;
  c->rank = rank;
  int st = comm_alloc(c);
  if (st) {
    comm_free(c);
    return st;
  }
  ncclUniqueId uid;
  memcpy(uid.internal, id, UTF8V_COMM_ID_BYTES);
  const ncclResult_t r = nccl().CommInitRank(&c->nccl, nranks, uid, rank);
  if (r != ncclSuccess) {
    c->nccl = nullptr;
    comm_free(c);
    return nccl_fail("ncclCommInitRank", r);
  }
  *out = c;
  return UTF8V_OK;
}

int utf8v_cuda_comm_init_all(int ndev, const int* devices, utf8v_cuda_comm** out_comms) {
  if (ndev < 1 || !out_comms) return fail(UTF8V_ERR_ARG, "bad comm arguments");
  NEED_NCCL();
  std::vector<int> devs(ndev);
  for (int i = 0; i < ndev; ++i) devs[i] = devices ? devices[i] : i;
  std::vector<ncclComm_t> nc(ndev, nullptr);
  NK(nccl().CommInitAll(nc.data(), ndev, devs.data()));
  DeviceGuard g;
  for (int i = 0; i < ndev; ++i) {
    utf8v_cuda_comm* c = new utf8v_cuda_comm();
    c->dev = devs[i];
    c->nranks = ndev;
    c->rank = i;
    c->nccl = nc[i];
    int st = cudaSetDevice(c->dev) == cudaSuccess ? comm_alloc(c) : fail(UTF8V_ERR_CUDA, "cudaSetDevice");
    out_comms[i] = c;
    if (st) {
      for (int j = 0; j <= i; ++j) comm_free(out_comms[j]), out_comms[j] = nullptr;
      for (int j = i + 1; j < ndev; ++j) g_nccl.CommDestroy(nc[j]);
      return st;
    }
  }
  return UTF8V_OK;
}

void utf8v_cuda_comm_destroy(utf8v_cuda_comm* c) { comm_free(c); }

int utf8v_cuda_validate_shard_allreduce_async(utf8v_cuda_comm* c, const uint8_t* d_p, uint64_t n,
                                              uint64_t lane_lo, uint64_t lane_hi, uint32_t* d_local_flag,
                                              uint32_t* d_global_flag, void* stream) {
  t_launches = 0;
  if (!c || !d_local_flag || !d_global_flag) return fail(UTF8V_ERR_ARG, "NULL comm/flag");
  int st = bad_lanes(n, lane_lo, lane_hi);
  if (st) return st;
  if (n > 0 && lane_lo < lane_hi) {
    if (!d_p) return fail(UTF8V_ERR_ARG, "NULL data");
    u8v::launch_validate(u8v::make_desc(d_p, n, lane_lo, lane_hi), d_local_flag, (cudaStream_t)stream);
    ++t_launches;
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(UTF8V_ERR_CUDA, "validate kernel", e);
  }
  NK(nccl().AllReduce(d_local_flag, d_global_flag, 1, ncclUint32, ncclMax, c->nccl, (cudaStream_t)stream));
  return UTF8V_OK;
}

int utf8v_cuda_validate_shard_allreduce(utf8v_cuda_comm* c, const uint8_t* p, uint64_t n, uint64_t lane_lo,
                                        uint64_t lane_hi, int is_device, uint8_t* out_valid) {
  t_launches = 0;
  if (!c || !out_valid) return fail(UTF8V_ERR_ARG, "NULL comm/out_valid");
  int st = bad_lanes(n, lane_lo, lane_hi);
  if (st) return st;
  DeviceGuard g;
  CK(cudaSetDevice(c->dev));
  int launches = 0;
  if (is_device) {
    CK(cudaMemsetAsync(c->d_buf, 0, 8, c->s));
    // Device input is ordered after the legacy default stream (as the other
    // synchronous entry points).
    CK(cudaEventRecord(c->ev_legacy, cudaStreamLegacy));
    CK(cudaStreamWaitEvent(c->s, c->ev_legacy, 0));
    if (n > 0 && lane_lo < lane_hi) {
      if (!p) return fail(UTF8V_ERR_ARG, "NULL data");
      u8v::launch_validate(u8v::make_desc(p, n, lane_lo, lane_hi), c->d_buf, c->s);
      ++launches;
    }
  } else {
    // Host input: the pipelined H2D + K1 path, then the flag goes up.
    uint32_t flag = 0;
    st = utf8v_cuda_validate_lanes(p, n, lane_lo, lane_hi, 0, &flag);
    if (st) return st;
    launches = t_launches;
    c->h_buf[0] = flag;
    CK(cudaMemcpyAsync(c->d_buf, c->h_buf, 4, cudaMemcpyHostToDevice, c->s));
  }
  NK(nccl().AllReduce(c->d_buf, c->d_buf + 1, 1, ncclUint32, ncclMax, c->nccl, c->s));
  CK(cudaMemcpyAsync(c->h_buf + 1, c->d_buf + 1, 4, cudaMemcpyDeviceToHost, c->s));
  CK(cudaStreamSynchronize(c->s));
  *out_valid = c->h_buf[1] == 0 ? 1 : 0;
  t_launches = launches;
  return UTF8V_OK;
}

int utf8v_cuda_verdict_shard_allreduce(utf8v_cuda_comm* c, const uint8_t* p, uint64_t n, uint64_t lane_lo,
                                       uint64_t lane_hi, uint64_t p_stream_offset, int is_device,
                                       uint8_t* out_valid, uint64_t* out_offset, int* out_kind) {
  t_launches = 0;
  if (!c || !out_valid || !out_offset || !out_kind) return fail(UTF8V_ERR_ARG, "NULL argument");
  DeviceGuard g;
  CK(cudaSetDevice(c->dev));
  uint8_t ok = 1;
  uint64_t off = 0;
  int kind = -1;
  int st = utf8v_cuda_validate_verdict_lanes(p, n, lane_lo, lane_hi, is_device, &ok, &off, &kind);
  if (st) return st;
  const int launches = t_launches;
  // (stream offset, kind) as one key; MIN over ranks picks the first error
  // (kinds are 0..5: 3 bits).  A valid shard contributes the maximum key.
  const uint64_t key = ok ? ~0ull : ((p_stream_offset + off) << 3) | (uint64_t)kind;
  memcpy(c->h_buf + 2, &key, 8);
  CK(cudaMemcpyAsync(c->d_buf + 2, c->h_buf + 2, 8, cudaMemcpyHostToDevice, c->s));
  NK(nccl().AllReduce(c->d_buf + 2, c->d_buf + 4, 1, ncclUint64, ncclMin, c->nccl, c->s));
  CK(cudaMemcpyAsync(c->h_buf + 4, c->d_buf + 4, 8, cudaMemcpyDeviceToHost, c->s));
  CK(cudaStreamSynchronize(c->s));
  uint64_t k;
  memcpy(&k, c->h_buf + 4, 8);
  *out_valid = k == ~0ull ? 1 : 0;
  *out_offset = k == ~0ull ? 0 : k >> 3;
  *out_kind = k == ~0ull ? -1 : (int)(k & 7);
  t_launches = launches;
  return UTF8V_OK;
}

int utf8v_cuda_validate_sharded_device(utf8v_cuda_comm* const* comms, int n_gpus, const uint8_t* const* d_shards,
                                       const uint64_t* shard_bytes, const uint64_t* lane_lo,
                                       const uint64_t* lane_hi, uint8_t* out_valid) {
  t_launches = 0;
  if (!comms || n_gpus < 1 || !d_shards || !shard_bytes || !lane_lo || !lane_hi || !out_valid)
    return fail(UTF8V_ERR_ARG, "NULL argument");
  NEED_NCCL();
  for (int g = 0; g < n_gpus; ++g) {
    if (!comms[g] || comms[g]->nranks != n_gpus) return fail(UTF8V_ERR_ARG, "comms must be one utf8v_cuda_comm_init_all set");
    const int st = bad_lanes(shard_bytes[g], lane_lo[g], lane_hi[g]);
    if (st) return st;
  }
  DeviceGuard dg;
  int launches = 0;
  // K1 on every device, each into its own local flag ...
  for (int g = 0; g < n_gpus; ++g) {
    utf8v_cuda_comm* c = comms[g];
    CK(cudaSetDevice(c->dev));
    CK(cudaMemsetAsync(c->d_buf, 0, 8, c->s));
    if (shard_bytes[g] > 0 && lane_lo[g] < lane_hi[g]) {
      if (!d_shards[g]) return fail(UTF8V_ERR_ARG, "NULL shard");
      u8v::launch_validate(u8v::make_desc(d_shards[g], shard_bytes[g], lane_lo[g], lane_hi[g]), c->d_buf, c->s);
      ++launches;
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(UTF8V_ERR_CUDA, "validate kernel", e);
  }
  // ... then one grouped 4-byte allreduce(MAX) over NVLink.
  NK(nccl().GroupStart());
  for (int g = 0; g < n_gpus; ++g) {
    utf8v_cuda_comm* c = comms[g];
    const ncclResult_t r = nccl().AllReduce(c->d_buf, c->d_buf + 1, 1, ncclUint32, ncclMax, c->nccl, c->s);
    if (r != ncclSuccess) {
      nccl().GroupEnd();
      return nccl_fail("ncclAllReduce", r);
    }
  }
  NK(nccl().GroupEnd());
  uint32_t any = 0;
  for (int g = 0; g < n_gpus; ++g) {
    utf8v_cuda_comm* c = comms[g];
    CK(cudaSetDevice(c->dev));
    CK(cudaMemcpyAsync(c->h_buf + 1, c->d_buf + 1, 4, cudaMemcpyDeviceToHost, c->s));
    CK(cudaStreamSynchronize(c->s));
    if (g == 0) any = c->h_buf[1];
    else if (c->h_buf[1] != any) return fail(UTF8V_ERR_NCCL, "ranks disagree after allreduce");
  }
  *out_valid = any == 0 ? 1 : 0;
  t_launches = launches;
  return UTF8V_OK;
}

// ---- P2P: the combine folded into K1 ------------------------------------------
int utf8v_cuda_p2p_create(utf8v_cuda_p2p** out, uint8_t* out_handle) {
  if (!out || !out_handle) return fail(UTF8V_ERR_ARG, "NULL argument");
  *out = nullptr;
  utf8v_cuda_p2p* g = new utf8v_cuda_p2p();
  cudaGetDevice(&g->dev);
  cudaIpcMemHandle_t h;
  if (cudaStreamCreateWithFlags(&g->s, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&g->d_flag, 64) != cudaSuccess || cudaMemset(g->d_flag, 0, 64) != cudaSuccess ||
      cudaMallocHost(&g->h_res, 64) != cudaSuccess || cudaIpcGetMemHandle(&h, g->d_flag) != cudaSuccess) {
    const cudaError_t e = cudaGetLastError();
    utf8v_cuda_p2p_destroy(g);
    return fail(UTF8V_ERR_CUDA, "p2p flag allocation / IPC handle", e);
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == UTF8V_P2P_HANDLE_BYTES, "IPC handle size");
  memcpy(out_handle, &h, UTF8V_P2P_HANDLE_BYTES);
  *out = g;
  return UTF8V_OK;
}

int utf8v_cuda_p2p_connect(utf8v_cuda_p2p* g, const uint8_t* handles, int nranks, int rank) {
  if (!g || !handles || nranks < 1 || rank < 0 || rank >= nranks) return fail(UTF8V_ERR_ARG, "bad p2p arguments");
  if (!g->opened.empty() || g->d_peers) return fail(UTF8V_ERR_ARG, "p2p group already connected");
  DeviceGuard dg;
  CK(cudaSetDevice(g->dev));
  std::vector<uint32_t*> peers;
  for (int r = 0; r < nranks; ++r) {
    if (r == rank) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + (size_t)r * UTF8V_P2P_HANDLE_BYTES, UTF8V_P2P_HANDLE_BYTES);
    void* ptr = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (void* q : g->opened) cudaIpcCloseMemHandle(q);
      g->opened.clear();
      return fail(UTF8V_ERR_CUDA, "cudaIpcOpenMemHandle (rank " + std::to_string(r) + ")", e);
    }
    g->opened.push_back(ptr);
    peers.push_back((uint32_t*)ptr);
  }
  g->nranks = nranks;
  g->rank = rank;
  if (!peers.empty()) {
    CK(cudaMalloc(&g->d_peers, peers.size() * sizeof(uint32_t*)));
    CK(cudaMemcpy(g->d_peers, peers.data(), peers.size() * sizeof(uint32_t*), cudaMemcpyHostToDevice));
  }
  return UTF8V_OK;
}

int utf8v_cuda_p2p_validate_async(utf8v_cuda_p2p* g, const uint8_t* d_p, uint64_t n, uint64_t lane_lo,
                                  uint64_t lane_hi, void* stream) {
  t_launches = 0;
  if (!g) return fail(UTF8V_ERR_ARG, "NULL p2p group");
  const int st = bad_lanes(n, lane_lo, lane_hi);
  if (st) return st;
  if (n == 0 || lane_lo == lane_hi) return UTF8V_OK;
  if (!d_p) return fail(UTF8V_ERR_ARG, "NULL data");
  u8v::StreamDesc d = u8v::make_desc(d_p, n, lane_lo, lane_hi);
  d.peer_flags = g->d_peers;
  d.n_peers = g->d_peers ? g->nranks - 1 : 0;
  u8v::launch_validate(d, g->d_flag, (cudaStream_t)stream);
  ++t_launches;
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? UTF8V_OK : fail(UTF8V_ERR_CUDA, "validate kernel", e);
}

uint32_t* utf8v_cuda_p2p_flag(utf8v_cuda_p2p* g) { return g ? g->d_flag : nullptr; }

int utf8v_cuda_p2p_read(utf8v_cuda_p2p* g, uint32_t* out_flag) {
  if (!g || !out_flag) return fail(UTF8V_ERR_ARG, "NULL argument");
  DeviceGuard dg;
  CK(cudaSetDevice(g->dev));
  CK(cudaMemcpyAsync(g->h_res, g->d_flag, 4, cudaMemcpyDeviceToHost, g->s));
  CK(cudaStreamSynchronize(g->s));
  *out_flag = g->h_res[0];
  return UTF8V_OK;
}

int utf8v_cuda_p2p_reset(utf8v_cuda_p2p* g) {
  if (!g) return fail(UTF8V_ERR_ARG, "NULL p2p group");
  DeviceGuard dg;
  CK(cudaSetDevice(g->dev));
  CK(cudaMemsetAsync(g->d_flag, 0, 4, g->s));
  CK(cudaStreamSynchronize(g->s));
  return UTF8V_OK;
}

void utf8v_cuda_p2p_destroy(utf8v_cuda_p2p* g) {
  if (!g) return;
  DeviceGuard dg;
  cudaSetDevice(g->dev);
  cudaDeviceSynchronize();
  for (void* q : g->opened) cudaIpcCloseMemHandle(q);
  if (g->d_peers) cudaFree(g->d_peers);
  if (g->d_flag) cudaFree(g->d_flag);
  if (g->h_res) cudaFreeHost(g->h_res);
  if (g->s) cudaStreamDestroy(g->s);
  cudaGetLastError();
  delete g;
}

}  // extern "C"
