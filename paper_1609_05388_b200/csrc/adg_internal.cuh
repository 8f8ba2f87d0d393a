// adg_internal.cuh -- shared host/device plumbing for libadg.so (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <cstdint>
#include <cstdio>
#include <exception>
#include <new>
#include <string>
#include <vector>

#include "../../include/adg.h"
#include <nvtx3/nvToolsExt.h>

namespace adg {

// NVTX range over a library phase (visible in nsys / ncu --nvtx timelines;
// header-only NVTX 3: no cost without a tool attached).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ----------------------------------------------------------------- errors
struct Error {
  adg_status status;
  std::string msg;
};

void set_last_error(const std::string& msg);

[[noreturn]] inline void fail(adg_status st, const std::string& msg) { throw Error{st, msg}; }

#define ADG_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      ::adg::fail(ADG_ECUDA, std::string("CUDA error ") + cudaGetErrorString(e_) + " at " \
                                 + __FILE__ + ":" + std::to_string(__LINE__));           \
  } while (0)

// Device-side checks of the checked build (build.py --checked ->
// libadg_checked.so, -DADG_DEVICE_CHECKS): index bounds on every list /
// table write of the hot kernels and bounded mbarrier waits, each failure
// printed and trapped.  compute-sanitizer is not available on the GPU pool
// this library is tested on, so this is how the test suite runs checked.
#ifdef ADG_DEVICE_CHECKS
#define ADG_DCHECK(cond)                                                                \
  do {                                                                                  \
    if (!(cond)) {                                                                      \
      printf("ADG_DCHECK failed: %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
             #cond, (int)blockIdx.x, (int)threadIdx.x);                                 \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#define ADG_WAIT_LIMIT (1ull << 31)  // spins before a wait is declared hung
#else
#define ADG_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

#define ADG_REQUIRE(cond, msg)                 \
  do {                                         \
    if (!(cond)) ::adg::fail(ADG_EINVAL, msg); \
  } while (0)

// Run f, mapping exceptions to status codes + the thread-local message.
template <typename F>
inline adg_status guard_call(F&& f) {
  try {
    f();
    return ADG_OK;
  } catch (const Error& e) {
    set_last_error(e.msg);
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return ADG_ENOMEM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return ADG_ECUDA;
  }
}

// ---------------------------------------------------------------- context
}  // namespace adg

struct adg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  double last_screen_ms = -1.0;
  int last_knn_engine = 0;  // adg_last_knn_engine
  int last_orig_passes = 0;  // adg_last_screen_orig_passes (0: no screen finalized yet)
  bool screen_forced3 = false;  // ADG_SCREEN_ORIG3 at the last screen launch
  uint64_t launches = 0;
  void* pinned = nullptr;  // page-locked staging for the finalize read-back
  size_t pinned_bytes = 0;
  cudaStream_t copy_stream = nullptr;  // H2D of the pipelined run_distort flow
  cudaStream_t phase_streams[4] = {};  // its screen phases (round robin)
  void* plan_cache = nullptr;  // adg_eval_plan*: the last device-input SCREEN plan (reused when
                               // the next evaluation has the same operands and shapes)
  void* tile_lists = nullptr;          // std::map<int64_t, DevBuf<uint32_t>>*: device tile lists
};

namespace adg {

// Launch bookkeeping: every kernel launch goes through this so the bench can
// report how many of OUR kernels ran (adg_kernel_launch_count).
inline void after_launch(adg_ctx* ctx) {
  ctx->launches++;
  ADG_CUDA(cudaGetLastError());
}

// ------------------------------------------------------- device buffers
template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t count = 0;
  cudaStream_t stream = nullptr;
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t s) { alloc(n, s); }
  void alloc(size_t n, cudaStream_t s) {
    release();
    stream = s;
    count = n;
    if (n) ADG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ptr), n * sizeof(T), s));
  }
  void zero() {
    if (count) ADG_CUDA(cudaMemsetAsync(ptr, 0, count * sizeof(T), stream));
  }
  void release() {
    if (ptr) cudaFreeAsync(ptr, stream);
    ptr = nullptr;
    count = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), count(o.count), stream(o.stream) {
    o.ptr = nullptr;
    o.count = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    ptr = o.ptr;
    count = o.count;
    stream = o.stream;
    o.ptr = nullptr;
    o.count = 0;
    return *this;
  }
};

inline bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

inline size_t dtype_size(adg_dtype t) { return t == ADG_F64 ? 8 : (t == ADG_F32 ? 4 : 2); }

// Device memory on the current device (managed memory counts as local).
inline bool is_local_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type == cudaMemoryTypeManaged) return true;
  int cur = 0;
  cudaGetDevice(&cur);
  return a.type == cudaMemoryTypeDevice && a.device == cur;
}

// A read-only operand: device pointer usable by kernels (staged if host, or
// if it lives on another device: a peer copy).
struct In {
  const void* dev = nullptr;
  DevBuf<uint8_t> staged;
  In(const void* p, size_t bytes, cudaStream_t s) {
    if (!p || bytes == 0) {
      dev = p;
      return;
    }
    if (is_local_device_ptr(p)) {
      dev = p;
    } else {
      staged.alloc(bytes, s);
      ADG_CUDA(cudaMemcpyAsync(staged.ptr, p, bytes, cudaMemcpyDefault, s));
      dev = staged.ptr;
    }
  }
  template <typename T>
  const T* as() const {
    return reinterpret_cast<const T*>(dev);
  }
};

// A write-only result: kernels write dev; commit() copies back if host.
struct Out {
  void* user = nullptr;
  void* dev = nullptr;
  size_t bytes = 0;
  DevBuf<uint8_t> staged;
  cudaStream_t stream;
  Out(void* p, size_t b, cudaStream_t s) : user(p), bytes(b), stream(s) {
    if (!p || b == 0) {
      dev = p;
      return;
    }
    if (is_device_ptr(p)) {
      dev = p;
    } else {
      staged.alloc(b, s);
      dev = staged.ptr;
    }
  }
  template <typename T>
  T* as() {
    return reinterpret_cast<T*>(dev);
  }
  void commit() {
    if (user && staged.ptr)
      ADG_CUDA(cudaMemcpyAsync(user, staged.ptr, bytes, cudaMemcpyDeviceToHost, stream));
  }
};

inline unsigned blocks_for(int64_t n, int threads, int64_t cap = 1 << 20) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return (unsigned)b;
}

// --------------------------------------------------------- device helpers
template <typename T>
__device__ __forceinline__ double to_f64(T v);
template <>
__device__ __forceinline__ double to_f64<double>(double v) { return v; }
template <>
__device__ __forceinline__ double to_f64<float>(float v) { return (double)v; }
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 v) {
  return (double)__bfloat162float(v);
}

// proj/include/adagio/rng.hpp:11-16
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// proj/include/adagio/rng.hpp:18-32 (host copies for seed bookkeeping)
inline uint64_t fnv1a64(const char* s) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 0x100000001b3ULL;
  }
  return h;
}
inline uint64_t derive_seed(uint64_t seed, const char* purpose) {
  return mix64(mix64(seed) ^ fnv1a64(purpose));
}

// SeededRng::next / below (rng.hpp:53-66), host side (Floyd sampling, ties).
struct HostRng {
  uint64_t state;
  uint64_t next() {
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  uint64_t below(uint64_t bound) {
    const uint64_t limit = bound * ((~uint64_t{0}) / bound);
    uint64_t v = next();
    while (v >= limit) v = next();
    return v % bound;
  }
};

// Dispatch helper over the input dtype.
#define ADG_DISPATCH_DTYPE(dt, T, ...)                        \
  switch (dt) {                                               \
    case ADG_F64: {                                           \
      using T = double;                                       \
      __VA_ARGS__;                                            \
    } break;                                                  \
    case ADG_F32: {                                           \
      using T = float;                                        \
      __VA_ARGS__;                                            \
    } break;                                                  \
    case ADG_BF16: {                                          \
      using T = __nv_bfloat16;                                \
      __VA_ARGS__;                                            \
    } break;                                                  \
    default:                                                  \
      ::adg::fail(ADG_EINVAL, "unsupported dtype");           \
  }

// ------------------------------------------------ shared module interfaces
// (implemented across the .cu files; all launch on ctx->stream)

// column means in fp64 of X (n x d) -> mean[d]; rows [r0, r1) only when
// partial (sum_only=true gives column sums instead of means).
void column_sums(adg_ctx* ctx, const void* X, adg_dtype dt, int64_t n, int64_t d, double* out);

// the context's page-locked staging buffer, grown to >= bytes (callers
// synchronise before reuse)
void* pinned_stage(adg_ctx* ctx, size_t bytes);

}  // namespace adg
