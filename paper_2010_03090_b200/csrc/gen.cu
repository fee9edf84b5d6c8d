// gen.cu -- deterministic synthetic inputs for the five BASELINE configs,
// generated on the device (a 16 GiB stream in milliseconds, not minutes).
//
// This is bench/test tooling, not the validation path.  It reuses the
// reference corpus primitives (proj/include/utf8v/corpus.hpp:123-146
// splitmix64 + unbiased below(); proj/src/corpus.cpp:68-82 random_code_point;
// proj/src/oracle.cpp:46-70 encode_code_point) and the reference's error
// shapes (proj/src/corpus.cpp:153-184), with the config-specific choices
// pinned in DESIGN.md "Synthetic inputs":
//
//   * A stream is cut into 64 KiB generation chunks; chunk j of a stream with
//     seed S draws from splitmix64(S ^ 0xD1B54A32D192ED03 * (j+1)).  Within a
//     chunk characters are appended while >= 4 bytes remain, then the chunk
//     is padded with printable ASCII, so every chunk (and stream) is exactly
//     sized and valid.  Chunk boundaries are character boundaries.
//   * mix: kind from below(10): 0-3 -> 1 byte, 4-5 -> 2, 6-8 -> 3, 9 -> 4
//     (0.4/0.2/0.3/0.1), code point uniform within the kind's class.
//   * ascii: per byte below(100) < 2 -> 0x0A, else 0x20 + below(95).
//   * patches: fixed byte strings written at given positions; the chunk fill
//     skips them (used to force shard edges inside characters, config 4).
//   * injected errors (configs 2, 3): one of seven classes at the character
//     boundary at or after a drawn offset, overwriting in place (sizes stay
//     exact) and turning orphaned continuation bytes after it into 'A'.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "../../include/utf8v_gen.h"
#include "kernels.cuh"

namespace u8v {

struct Rng {
  uint64_t s;
};

__host__ __device__ __forceinline__ uint64_t rng_next(Rng& r) {
  uint64_t z = (r.s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t rng_below(Rng& r, uint64_t bound) {
  const uint64_t threshold = (0 - bound) % bound;
  for (;;) {
    const uint64_t x = rng_next(r);
    if (x >= threshold) return x % bound;
  }
}

__host__ __device__ __forceinline__ uint32_t random_cp(int kind, Rng& r) {
  switch (kind) {
    case 1: return (uint32_t)rng_below(r, 0x80);
    case 2: return 0x80 + (uint32_t)rng_below(r, 0x800 - 0x80);
    case 3: {
      uint32_t cp = 0x800 + (uint32_t)rng_below(r, 0x10000 - 0x800 - 0x800);
      if (cp >= 0xD800) cp += 0x800;
      return cp;
    }
    default: return 0x10000 + (uint32_t)rng_below(r, 0x110000 - 0x10000);
  }
}

__host__ __device__ __forceinline__ int encode_cp(uint32_t cp, uint8_t* o) {
  if (cp <= 0x7F) {
    o[0] = (uint8_t)cp;
    return 1;
  }
  if (cp <= 0x7FF) {
    o[0] = (uint8_t)(0xC0 | (cp >> 6));
    o[1] = (uint8_t)(0x80 | (cp & 0x3F));
    return 2;
  }
  if (cp <= 0xFFFF) {
    o[0] = (uint8_t)(0xE0 | (cp >> 12));
    o[1] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
    o[2] = (uint8_t)(0x80 | (cp & 0x3F));
    return 3;
  }
  o[0] = (uint8_t)(0xF0 | (cp >> 18));
  o[1] = (uint8_t)(0x80 | ((cp >> 12) & 0x3F));
  o[2] = (uint8_t)(0x80 | ((cp >> 6) & 0x3F));
  o[3] = (uint8_t)(0x80 | (cp & 0x3F));
  return 4;
}

__host__ __device__ __forceinline__ int mix_kind(Rng& r) {
  const uint64_t k = rng_below(r, 10);
  return k < 4 ? 1 : k < 6 ? 2 : k < 9 ? 3 : 4;
}

__host__ __device__ __forceinline__ uint64_t chunk_seed(uint64_t seed, uint64_t j) {
  return seed ^ (0xD1B54A32D192ED03ull * (j + 1));
}

__host__ __device__ __forceinline__ Rng plan_rng(uint64_t seed, uint64_t tag) {
  return Rng{seed ^ (0xA24BAED4963EE407ull * tag)};
}

// Byte writer that turns a thread's sequential byte stream into aligned
// 32-bit stores (a warp's threads write far-apart regions).
struct Writer {
  uint8_t* base;
  uint64_t pos;
  uint32_t acc;
  __host__ __device__ void start(uint8_t* b, uint64_t p) {
    base = b;
    pos = p;
    acc = 0;
  }
  __host__ __device__ __forceinline__ void put(uint8_t v) {
    acc |= (uint32_t)v << (8 * (pos & 3));
    ++pos;
    if ((pos & 3) == 0) {
      *reinterpret_cast<uint32_t*>(base + pos - 4) = acc;
      acc = 0;
    }
  }
  // Flush a partial word (first/last word of a range: byte stores).
  __host__ __device__ void flush() {
    const uint64_t k = pos & 3;
    for (uint64_t i = 0; i < k; ++i) base[pos - k + i] = (uint8_t)(acc >> (8 * i));
    acc = 0;
  }
};

// Fill [lo, hi) of out (valid text, exactly sized) drawing from r.
__host__ __device__ void fill_range(uint8_t* out, uint64_t lo, uint64_t hi, Rng& r, int ascii_only) {
  if (lo >= hi) return;
  // Leading unaligned bytes go through byte stores so the word stores of the
  // writer never clobber a neighbour's bytes.
  Writer w;
  uint8_t buf[4];
  uint64_t p = lo;
  auto emit = [&](uint8_t v) {
    if ((p & ~3ull) == (lo & ~3ull) && (lo & 3)) {
      out[p] = v;  // shares its word with bytes before lo
    } else if ((p & ~3ull) == ((hi - 1) & ~3ull) && (hi & 3)) {
      out[p] = v;  // shares its word with bytes at/after hi
    } else {
      if ((p & 3) == 0) w.start(out, p);
      w.put(v);
    }
    ++p;
  };
  if (ascii_only) {
    while (p < hi) emit(rng_below(r, 100) < 2 ? (uint8_t)0x0A : (uint8_t)(0x20 + rng_below(r, 95)));
  } else {
    while (hi - p >= 4) {
      const int len = encode_cp(random_cp(mix_kind(r), r), buf);
      for (int i = 0; i < len; ++i) emit(buf[i]);
    }
    while (p < hi) emit((uint8_t)(0x20 + rng_below(r, 95)));
  }
}

struct DevPatch {
  uint64_t pos;
  uint32_t len;
  uint8_t bytes[12];
};

// One thread per 64 KiB chunk; patches (sorted, non-overlapping) are skipped.
__global__ void k_gen_stream(uint8_t* __restrict__ out, uint64_t n, uint64_t seed, int ascii_only,
                             const DevPatch* __restrict__ patches, int npatches) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t cs = j * kGenChunk;
  if (cs >= n) return;
  const uint64_t ce = cs + kGenChunk < n ? cs + kGenChunk : n;
  Rng r{chunk_seed(seed, j)};
  uint64_t p = cs;
  for (int k = 0; k < npatches; ++k) {
    const uint64_t ps = patches[k].pos, pe = ps + patches[k].len;
    if (pe <= cs || ps >= ce) continue;
    if (ps > p) fill_range(out, p, ps, r, ascii_only);
    p = pe;
  }
  if (p < ce) fill_range(out, p, ce, r, ascii_only);
}

// Host twin of k_gen_stream (no patches): same bytes, for CPU-only callers
// (the reference arm of bench.py needs no GPU).
void gen_chunks_host(uint8_t* out, uint64_t n, uint64_t seed, int ascii_only, uint64_t j0,
                     uint64_t j1) {
  for (uint64_t j = j0; j < j1; ++j) {
    const uint64_t cs = j * kGenChunk;
    const uint64_t ce = cs + kGenChunk < n ? cs + kGenChunk : n;
    Rng r{chunk_seed(seed, j)};
    fill_range(out, cs, ce, r, ascii_only);
  }
}

// Bytes [lo, hi) of the n-byte stream (lo % 4 == 0) into out[0 .. hi-lo):
// chunks inside the window write through the aligned writer, the (at most
// two) chunks cut by the window regenerate the chunk and keep their part.
__global__ void k_gen_stream_range(uint8_t* __restrict__ out, uint64_t n, uint64_t lo, uint64_t hi,
                                   uint64_t seed, int ascii_only) {
  const uint64_t j = lo / kGenChunk + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t cs = j * kGenChunk;
  if (cs >= hi || cs >= n) return;
  const uint64_t ce = cs + kGenChunk < n ? cs + kGenChunk : n;
  Rng r{chunk_seed(seed, j)};
  if (cs >= lo && ce <= hi) {
    fill_range(out - lo, cs, ce, r, ascii_only);
    return;
  }
  // Cut chunk: generate sequentially, store only the window's bytes.
  uint8_t buf[4];
  uint64_t p = cs;
  auto put = [&](uint8_t v) {
    if (p >= lo && p < hi) out[p - lo] = v;
    ++p;
  };
  if (ascii_only) {
    while (p < ce) put(rng_below(r, 100) < 2 ? (uint8_t)0x0A : (uint8_t)(0x20 + rng_below(r, 95)));
  } else {
    while (ce - p >= 4) {
      const int len = encode_cp(random_cp(mix_kind(r), r), buf);
      for (int i = 0; i < len; ++i) put(buf[i]);
    }
    while (p < ce) put((uint8_t)(0x20 + rng_below(r, 95)));
  }
}

__global__ void k_write_patches(uint8_t* __restrict__ out, const DevPatch* __restrict__ patches,
                                int npatches) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= npatches) return;
  for (uint32_t i = 0; i < patches[k].len; ++i) out[patches[k].pos + i] = patches[k].bytes[i];
}

// One thread per record: record r is its own mix stream of exactly its length.
__global__ void k_gen_records(uint8_t* __restrict__ out, const uint64_t* __restrict__ offsets,
                              uint64_t n_records, uint64_t seed) {
  const uint64_t rix = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rix >= n_records) return;
  Rng r{chunk_seed(seed, rix)};
  fill_range(out, offsets[rix], offsets[rix + 1], r, 0);
}

// ---- error injection (host+device) ----------------------------------------
__host__ __device__ __forceinline__ bool is_cont(uint8_t b) { return (b & 0xC0) == 0x80; }

// Inject one error of class cls into the valid text [lo, hi), at the
// character boundary at or after lo + u (u <= hi - lo - 8), or at the end
// (class 6).  Returns the offset the oracle will report.
__host__ __device__ uint64_t inject_error(uint8_t* s, uint64_t lo, uint64_t hi, int cls,
                                          uint64_t u, Rng& r) {
  uint8_t piece[8];
  int m = 0;
  auto cont = [&r]() { return (uint8_t)(0x80 + rng_below(r, 0x40)); };
  if (cls == kErrTruncatedEnd) {
    const int len = 2 + (int)rng_below(r, 3);
    uint8_t enc[4];
    encode_cp(random_cp(len, r), enc);
    const uint64_t q = hi - (uint64_t)(len - 1);
    uint64_t t = q;
    while (t > lo && is_cont(s[t])) --t;  // start of the character holding q
    for (uint64_t i = t; i < q; ++i) s[i] = 'A';
    for (int i = 0; i < len - 1; ++i) s[q + i] = enc[i];
    return q;
  }
  uint64_t q = lo + u;
  while (q < hi && is_cont(s[q])) ++q;
  switch (cls) {
    case kErrOverlong: {
      const uint64_t sub = rng_below(r, 3);
      if (sub == 0) {
        piece[m++] = (uint8_t)(0xC0 + rng_below(r, 2));
        piece[m++] = cont();
      } else if (sub == 1) {
        piece[m++] = 0xE0;
        piece[m++] = (uint8_t)(0x80 + rng_below(r, 0x20));
        piece[m++] = cont();
      } else {
        piece[m++] = 0xF0;
        piece[m++] = (uint8_t)(0x80 + rng_below(r, 0x10));
        piece[m++] = cont();
        piece[m++] = cont();
      }
      break;
    }
    case kErrSurrogate:
      piece[m++] = 0xED;
      piece[m++] = (uint8_t)(0xA0 + rng_below(r, 0x20));
      piece[m++] = cont();
      break;
    case kErrTooLarge:
      piece[m++] = 0xF4;
      piece[m++] = (uint8_t)(0x90 + rng_below(r, 0x30));
      piece[m++] = cont();
      piece[m++] = cont();
      break;
    case kErrBadLead: {
      const uint64_t v = rng_below(r, 13);
      const uint8_t lead = v < 2 ? (uint8_t)(0xC0 + v) : (uint8_t)(0xF5 + (v - 2));
      piece[m++] = lead;
      const int k = lead < 0xE0 ? 1 : 3;
      for (int i = 0; i < k; ++i) piece[m++] = cont();
      break;
    }
    case kErrMissingCont: {
      const int len = 2 + (int)rng_below(r, 3);
      uint8_t enc[4];
      encode_cp(random_cp(len, r), enc);
      piece[m++] = enc[0];
      piece[m++] = 'A';
      break;
    }
    default:  // kErrStrayCont
      piece[m++] = cont();
      break;
  }
  for (int i = 0; i < m; ++i) s[q + i] = piece[i];
  for (uint64_t p = q + m; p < hi && is_cont(s[p]); ++p) s[p] = 'A';
  return q;
}

struct DevInjection {
  uint64_t lo, hi, u, seed;
  int cls;
  int pad;
};

__global__ void k_inject(uint8_t* __restrict__ s, const DevInjection* __restrict__ inj, int count,
                         unsigned long long* __restrict__ where) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  Rng r{inj[k].seed};
  where[k] = inject_error(s, inj[k].lo, inj[k].hi, inj[k].cls, inj[k].u, r);
}

}  // namespace u8v

// ---- C-ABI (include/utf8v_gen.h) ------------------------------------------
using namespace u8v;

namespace {

int cuda_status(cudaError_t e) { return e == cudaSuccess ? 0 : 1; }

int gen_stream_impl(uint8_t* d_out, uint64_t n, uint64_t seed, int ascii_only,
                    std::vector<DevPatch> patches, cudaStream_t st) {
  std::sort(patches.begin(), patches.end(),
            [](const DevPatch& a, const DevPatch& b) { return a.pos < b.pos; });
  DevPatch* d_p = nullptr;
  const int np = (int)patches.size();
  if (np > 0) {
    if (cudaMalloc(&d_p, sizeof(DevPatch) * np) != cudaSuccess) return 1;
    cudaMemcpyAsync(d_p, patches.data(), sizeof(DevPatch) * np, cudaMemcpyHostToDevice, st);
  }
  const uint64_t chunks = (n + kGenChunk - 1) / kGenChunk;
  if (chunks > 0) {
    const unsigned threads = 64;
    k_gen_stream<<<(unsigned)((chunks + threads - 1) / threads), threads, 0, st>>>(
        d_out, n, seed, ascii_only, d_p, np);
  }
  if (np > 0) k_write_patches<<<(np + 63) / 64, 64, 0, st>>>(d_out, d_p, np);
  cudaError_t e = cudaStreamSynchronize(st);
  if (d_p) cudaFree(d_p);
  return cuda_status(e == cudaSuccess ? cudaGetLastError() : e);
}

DevPatch make_patch(uint64_t pos, const uint8_t* b, int len) {
  DevPatch p;
  memset(&p, 0, sizeof p);
  p.pos = pos;
  p.len = (uint32_t)len;
  memcpy(p.bytes, b, len);
  return p;
}

int run_injections(uint8_t* d_s, const std::vector<DevInjection>& inj, uint64_t* h_where,
                   cudaStream_t st) {
  if (inj.empty()) return 0;
  DevInjection* d_inj = nullptr;
  unsigned long long* d_where = nullptr;
  if (cudaMalloc(&d_inj, sizeof(DevInjection) * inj.size()) != cudaSuccess) return 1;
  if (cudaMalloc(&d_where, sizeof(unsigned long long) * inj.size()) != cudaSuccess) return 1;
  cudaMemcpyAsync(d_inj, inj.data(), sizeof(DevInjection) * inj.size(), cudaMemcpyHostToDevice, st);
  k_inject<<<(unsigned)((inj.size() + 127) / 128), 128, 0, st>>>(d_s, d_inj, (int)inj.size(),
                                                                 d_where);
  if (h_where)
    cudaMemcpyAsync(h_where, d_where, sizeof(unsigned long long) * inj.size(),
                    cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  cudaFree(d_inj);
  cudaFree(d_where);
  return cuda_status(e == cudaSuccess ? cudaGetLastError() : e);
}

}  // namespace

extern "C" {

int utf8v_gen_stream(uint8_t* d_out, uint64_t n, uint64_t seed, int ascii_only, void* stream) {
  return gen_stream_impl(d_out, n, seed, ascii_only, {}, (cudaStream_t)stream);
}

int utf8v_gen_stream_range(uint8_t* d_out, uint64_t n, uint64_t lo, uint64_t hi, uint64_t seed,
                           int ascii_only, void* stream) {
  if (lo % 4 != 0 || hi < lo || hi > n) return 2;
  if (hi == lo) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t chunks = (hi + kGenChunk - 1) / kGenChunk - lo / kGenChunk;
  const unsigned threads = 64;
  k_gen_stream_range<<<(unsigned)((chunks + threads - 1) / threads), threads, 0, st>>>(
      d_out, n, lo, hi, seed, ascii_only);
  cudaError_t e = cudaStreamSynchronize(st);
  return cuda_status(e == cudaSuccess ? cudaGetLastError() : e);
}

int utf8v_gen_stream_host(uint8_t* out, uint64_t n, uint64_t seed, int ascii_only, int threads) {
  const uint64_t chunks = (n + kGenChunk - 1) / kGenChunk;
  if (threads < 1) threads = 1;
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    const uint64_t j0 = chunks * (uint64_t)t / (uint64_t)threads;
    const uint64_t j1 = chunks * (uint64_t)(t + 1) / (uint64_t)threads;
    pool.emplace_back([=] { gen_chunks_host(out, n, seed, ascii_only, j0, j1); });
  }
  for (auto& th : pool) th.join();
  return 0;
}

int utf8v_gen_c2(uint8_t* d_out, uint64_t seg_len, uint32_t n_seg, uint64_t seed,
                 uint8_t* h_expected_valid, uint64_t* h_error_offset, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (seg_len < 64 || n_seg == 0) return 2;
  if (gen_stream_impl(d_out, seg_len * n_seg, seed, 0, {}, st)) return 1;
  Rng plan = plan_rng(seed, 2);
  std::vector<uint32_t> perm(n_seg);
  for (uint32_t i = 0; i < n_seg; ++i) perm[i] = i;
  const uint32_t n_bad = n_seg / 2;
  for (uint32_t i = 0; i < n_bad; ++i) {
    const uint32_t j = i + (uint32_t)rng_below(plan, n_seg - i);
    std::swap(perm[i], perm[j]);
  }
  std::vector<uint32_t> bad(perm.begin(), perm.begin() + n_bad);
  std::sort(bad.begin(), bad.end());
  std::vector<DevInjection> inj;
  for (uint32_t s : bad) {
    DevInjection d;
    d.lo = (uint64_t)s * seg_len;
    d.hi = d.lo + seg_len;
    d.cls = (int)rng_below(plan, kErrClasses);
    d.u = rng_below(plan, seg_len - 8);
    d.seed = rng_next(plan);
    d.pad = 0;
    inj.push_back(d);
  }
  std::vector<uint64_t> where(inj.size());
  if (run_injections(d_out, inj, where.data(), st)) return 1;
  for (uint32_t s = 0; s < n_seg; ++s) {
    if (h_expected_valid) h_expected_valid[s] = 1;
    if (h_error_offset) h_error_offset[s] = ~0ull;
  }
  for (size_t k = 0; k < bad.size(); ++k) {
    if (h_expected_valid) h_expected_valid[bad[k]] = 0;
    if (h_error_offset) h_error_offset[bad[k]] = where[k] - (uint64_t)bad[k] * seg_len;
  }
  return 0;
}

int utf8v_gen_c3_offsets(uint64_t n_records, uint64_t seed, double sigma, uint64_t median,
                         uint64_t min_len, uint64_t max_len, uint64_t* h_offsets) {
  Rng plan = plan_rng(seed, 3);
  const double two_pi = 6.283185307179586476925286766559;
  const double mu = log((double)median);
  h_offsets[0] = 0;
  for (uint64_t r = 0; r < n_records; ++r) {
    // Box-Muller on two 53-bit uniforms in (0, 1].
    const double u1 = (double)((rng_next(plan) >> 11) + 1) * (1.0 / 9007199254740992.0);
    const double u2 = (double)((rng_next(plan) >> 11) + 1) * (1.0 / 9007199254740992.0);
    const double z = sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
    double len = floor(exp(mu + sigma * z) + 0.5);
    if (len < (double)min_len) len = (double)min_len;
    if (len > (double)max_len) len = (double)max_len;
    h_offsets[r + 1] = h_offsets[r] + (uint64_t)len;
  }
  return 0;
}

int utf8v_gen_c3(uint8_t* d_out, const uint64_t* d_offsets, const uint64_t* h_offsets,
                 uint64_t n_records, uint64_t seed, uint8_t* h_expected_valid, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_records == 0) return 0;
  k_gen_records<<<(unsigned)((n_records + 127) / 128), 128, 0, st>>>(d_out, d_offsets, n_records,
                                                                     seed);
  Rng plan = plan_rng(seed, 4);
  std::vector<DevInjection> inj;
  for (uint64_t r = 0; r < n_records; ++r) {
    const bool bad = rng_below(plan, 10) == 0 && h_offsets[r + 1] - h_offsets[r] >= 16;
    if (h_expected_valid) h_expected_valid[r] = bad ? 0 : 1;
    if (!bad) continue;
    DevInjection d;
    d.lo = h_offsets[r];
    d.hi = h_offsets[r + 1];
    d.cls = (int)rng_below(plan, kErrClasses);
    d.u = rng_below(plan, (d.hi - d.lo) - 8);
    d.seed = rng_next(plan);
    d.pad = 0;
    inj.push_back(d);
  }
  return run_injections(d_out, inj, nullptr, st);
}

int utf8v_gen_c4(uint8_t* d_out, uint64_t n, uint64_t seed, int variant, uint64_t* h_error_offset,
                 void* stream) {
  if (n < 8 * kGenChunk || n % 8 != 0) return 2;
  Rng plan = plan_rng(seed, 5);
  std::vector<DevPatch> patches;
  uint64_t err_at = ~0ull;
  // Each shard edge k*n/8 (k = 1..7) falls inside a 3- or 4-byte character;
  // bytes before the edge: 1|2, 1|3, 2|1, 2|2, 1|2, 3|1, 2|1 for k = 1..7.
  static const int kLen[8] = {0, 3, 4, 3, 4, 3, 4, 3};
  static const int kBefore[8] = {0, 1, 1, 2, 2, 1, 3, 2};
  for (int k = 1; k < 8; ++k) {
    const uint64_t b = (uint64_t)k * (n / 8);
    uint8_t enc[12];
    const int len = encode_cp(random_cp(kLen[k], plan), enc);
    int before = kBefore[k];
    if (variant == 1 && k == 4) {
      // Variant B: a 3-byte character at [b-2, b+1), then an overlong
      // E0 80..9F 80..BF whose lead is 1 byte after the edge.
      const int l3 = encode_cp(random_cp(3, plan), enc);
      enc[l3 + 0] = 0xE0;
      enc[l3 + 1] = (uint8_t)(0x80 + rng_below(plan, 0x20));
      enc[l3 + 2] = (uint8_t)(0x80 + rng_below(plan, 0x40));
      patches.push_back(make_patch(b - 2, enc, l3 + 3));
      err_at = b + 1;
      continue;
    }
    patches.push_back(make_patch(b - (uint64_t)before, enc, len));
  }
  if (variant == 2) {
    // Variant C: the stream ends with 3 bytes of a 4-byte character.
    uint8_t enc[4];
    encode_cp(random_cp(4, plan), enc);
    patches.push_back(make_patch(n - 3, enc, 3));
    err_at = n - 3;
  }
  if (h_error_offset) *h_error_offset = err_at;
  return gen_stream_impl(d_out, n, seed, 0, patches, (cudaStream_t)stream);
}

}  // extern "C"
