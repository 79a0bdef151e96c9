// common.cuh — shared device/host utilities for librdd (B200, sm_100a, FP64).
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <map>
#include <mutex>
#include <utility>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace rdd {

constexpr int kMaxDim = 4;
constexpr int kMaxJet = 15;  // jet_len(4)

__host__ __device__ constexpr int jet_len(int d) { return 1 + d + d * (d + 1) / 2; }
__host__ __device__ constexpr int hess_index(int i, int j, int d) { return i * d - i * (i - 1) / 2 + (j - i); }

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw CudaError(std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " at " + file + ":" +
                    std::to_string(line));
}
#define RDD_CUDA(x) ::rdd::check_cuda((x), #x, __FILE__, __LINE__)

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: the largest size set so far is
// cached per (kernel, device) under a lock, so contexts on several devices and host threads are safe
inline void ensure_smem_attr(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  RDD_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = done[{kernel, dev}];
  if (bytes > cur) {
    RDD_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    cur = bytes;
  }
}
// every kernel launch of the library goes through this check: it also counts launches
inline int64_t& launch_counter() {
  static thread_local int64_t n = 0;
  return n;
}
#define RDD_LAUNCH_CHECK() (++::rdd::launch_counter(), ::rdd::check_cuda(cudaGetLastError(), "kernel launch", __FILE__, __LINE__))

// Stream that owns temporaries of the current API call: stream-ordered pool allocations
// (cudaMallocAsync / cudaFreeAsync) make per-call scratch buffers cheap.
inline cudaStream_t& alloc_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}

// host<->device bytes moved by the calling thread (e2e accounting)
inline int64_t& h2d_counter() {
  static thread_local int64_t n = 0;
  return n;
}
inline int64_t& d2h_counter() {
  static thread_local int64_t n = 0;
  return n;
}

// Pinned (page-locked) host allocator: the host-built inputs are staged here so the H2D
// copies run at full PCIe/C2C bandwidth.
template <class T>
struct PinnedAlloc {
  using value_type = T;
  PinnedAlloc() = default;
  template <class U>
  PinnedAlloc(const PinnedAlloc<U>&) {}
  T* allocate(size_t n) {
    void* p = nullptr;
    if (cudaMallocHost(&p, n * sizeof(T)) != cudaSuccess) throw std::bad_alloc();
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t) { cudaFreeHost(p); }
  template <class U>
  bool operator==(const PinnedAlloc<U>&) const { return true; }
  template <class U>
  bool operator!=(const PinnedAlloc<U>&) const { return false; }
};
template <class T>
using pinned_vector = std::vector<T, PinnedAlloc<T>>;

// Owning device buffer (pooled, stream-ordered; grows, never shrinks).
// host seconds spent inside DBuf::upload (pageable copies may wait for the stream): diagnostics
inline double& upload_wait_s() {
  static thread_local double t = 0.0;
  return t;
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) {
      if (alloc_stream()) cudaFreeAsync(p, alloc_stream());
      else cudaFree(p);
    }
    p = nullptr;
    n = 0;
  }
  T* ensure(size_t count) {
    if (count > n) {
      release();
      if (count) {
        if (alloc_stream()) RDD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), alloc_stream()));
        else RDD_CUDA(cudaMalloc(&p, count * sizeof(T)));
      }
      n = count;
    }
    return p;
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    ensure(count);
    const auto t0 = std::chrono::steady_clock::now();
    if (count) RDD_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    upload_wait_s() += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    h2d_counter() += static_cast<int64_t>(count * sizeof(T));
  }
  template <class Alloc>
  void upload(const std::vector<T, Alloc>& h, cudaStream_t s) {
    upload(h.data(), h.size(), s);
  }
  void download(T* h, size_t count, cudaStream_t s) const {
    if (count) RDD_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    d2h_counter() += static_cast<int64_t>(count * sizeof(T));
  }
  void zero(size_t count, cudaStream_t s) {
    ensure(count);
    if (count) RDD_CUDA(cudaMemsetAsync(p, 0, count * sizeof(T), s));
  }
};

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// ---- device helpers --------------------------------------------------------------------
#ifdef __CUDACC__
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// sum over a 256-thread CTA in a fixed order (valid in thread 0)
__device__ __forceinline__ double block_sum_256(double v) {
  __shared__ double sh_b256[8];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) sh_b256[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < 8 ? sh_b256[threadIdx.x] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;
}
// Σ part[0..n) by one warp in a fixed order (lane-strided, then the xor tree): every lane of
// every warp that calls it gets the identical value
__device__ __forceinline__ double warp_sum_parts(const double* part, int n) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s += part[i];
  return warp_sum(s);
}
__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Second-order jet in dimension d (value, gradient, packed upper Hessian), jet.hpp:45-156.
struct Jet {
  double c[kMaxJet];
};

__device__ __forceinline__ void jet_zero(Jet& a, int d) {
  for (int i = 0; i < jet_len(d); ++i) a.c[i] = 0.0;
}
// Leibniz product (jet.hpp:107-124), grouped like the reference.
__device__ __forceinline__ Jet jet_mul(const Jet& a, const Jet& b, int d) {
  Jet o;
  o.c[0] = a.c[0] * b.c[0];
  for (int i = 0; i < d; ++i) o.c[1 + i] = a.c[0] * b.c[1 + i] + b.c[0] * a.c[1 + i];
  for (int i = 0; i < d; ++i)
    for (int j = i; j < d; ++j) {
      const int k = 1 + d + hess_index(i, j, d);
      o.c[k] = (a.c[0] * b.c[k] + b.c[0] * a.c[k]) + (a.c[1 + i] * b.c[1 + j] + a.c[1 + j] * b.c[1 + i]);
    }
  return o;
}
// chain rule through a univariate function (jet.hpp:127-138)
__device__ __forceinline__ Jet jet_compose(double f, double df, double d2f, const Jet& a, int d) {
  Jet o;
  o.c[0] = f;
  for (int i = 0; i < d; ++i) o.c[1 + i] = df * a.c[1 + i];
  for (int i = 0; i < d; ++i)
    for (int j = i; j < d; ++j) {
      const int k = 1 + d + hess_index(i, j, d);
      o.c[k] = df * a.c[k] + d2f * a.c[1 + i] * a.c[1 + j];
    }
  return o;
}

#endif  // __CUDACC__

}  // namespace rdd
