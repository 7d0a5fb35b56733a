// common.cuh — shared device/host helpers for the ASTRA B200 kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <atomic>

#include "../../include/astra_b200.h"

namespace astra {

// ---------------------------------------------------------------- host side

// Thread-local error message for astra_last_error(); returns `code`.
int set_error(int code, const char* fmt, ...);
// Map a CUDA error to ASTRA_ERR_CUDA with a message (0 if ok).
int check_cuda(cudaError_t e, const char* what);
// Count one kernel launch of this library (astra_launch_count()).
void count_launch(uint64_t n = 1);
int num_sms();

// Live kernel timing (astra_kernel_timing_enable / astra_kernel_timing): when
// enabled, a KernelTimer scope records CUDA events on the launching stream
// around the launches it encloses and files the pair under `name`.
bool kernel_timing_on();
cudaEvent_t kernel_timing_event();
void kernel_timing_push(const char* name, cudaEvent_t e0, cudaEvent_t e1);
struct KernelTimer {
  const char* name;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  KernelTimer(const char* n, cudaStream_t s) : name(n), st(s) {
    if (kernel_timing_on()) {
      e0 = kernel_timing_event();
      e1 = kernel_timing_event();
      cudaEventRecord(e0, st);
    }
  }
  ~KernelTimer() {
    if (e0) {
      cudaEventRecord(e1, st);
      kernel_timing_push(name, e0, e1);
    }
  }
};

// Launches of the step's kernel chain (sampler -> counting sort -> passes)
// carry the programmatic-stream-serialization attribute (every chain kernel
// starts with pdl_entry(), ptx.cuh); ASTRA_PDL=0 launches them plainly.
inline bool pdl_on() {
  static const bool v = [] {
    const char* e = getenv("ASTRA_PDL");
    return e == nullptr || atoi(e) != 0;
  }();
  return v;
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
}

#define ASTRA_TRY(expr)            \
  do {                             \
    int _rc = (expr);              \
    if (_rc != ASTRA_OK) return _rc; \
  } while (0)

#define ASTRA_LAUNCHED(what)                                         \
  do {                                                               \
    ::astra::count_launch();                                         \
    cudaError_t _e = cudaGetLastError();                             \
    if (_e != cudaSuccess) return ::astra::check_cuda(_e, what);     \
  } while (0)

__host__ __device__ static inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Carve {
  char* base;
  size_t off = 0;
  size_t cap;
  Carve(void* p, size_t c) : base(static_cast<char*>(p)), cap(c) {}
  template <class T>
  T* take(size_t n) {
    off = align_up(off, 256);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * sizeof(T);
    return p;
  }
  bool ok() const { return off <= cap; }
};

// ---------------------------------------------------------------- keys
// key = (monotone(score) << 32) | (0xFFFFFFFF - id): larger key = higher score,
// ties toward the lower id (anns.py:103-109). 0 = empty.

__host__ __device__ __forceinline__ uint32_t ord_bits(uint32_t b) {
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ uint64_t make_key(float s, uint32_t gid) {
  s = __fadd_rn(s, 0.0f);  // canonicalise -0.0 to +0.0
  return (static_cast<uint64_t>(ord_bits(__float_as_uint(s))) << 32) | (0xFFFFFFFFu - gid);
}

__device__ __forceinline__ float key_score(uint64_t key) {
  uint32_t o = static_cast<uint32_t>(key >> 32);
  uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
  return __uint_as_float(b);
}

__device__ __forceinline__ int32_t key_id(uint64_t key) {
  return static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(key));
}

// Binary search in a sorted int32 list (global or shared).
__device__ __forceinline__ bool sorted_contains(const int32_t* __restrict__ a, int64_t n, int64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo < n && a[lo] == v;
}

// ---------------------------------------------------------------- Philox4x32-10
// Random123 philox4x32-10 (KAT-checked in tests/test_oracle_c.py); counter
// layout documented in oracle/astra_oracle.c and include/astra_b200.h.

struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                           uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return U4{c0, c1, c2, c3};
}

__device__ __forceinline__ uint64_t bounded_u64(U4 r, uint64_t n) {
  uint64_t x = static_cast<uint64_t>(r.x) | (static_cast<uint64_t>(r.y) << 32);
  return __umul64hi(x, n);
}

// ---------------------------------------------------------------- misc

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t h) {
  return __uint_as_float(static_cast<uint32_t>(h) << 16);
}

__device__ __forceinline__ uint16_t f32_to_bf16_bits(float f) {
  __nv_bfloat16 b = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&b);
}

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace astra
