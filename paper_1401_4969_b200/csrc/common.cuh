// Shared plumbing for the B200 correction-step library: error taxonomy that
// mirrors the reference's exceptions (errors.hpp:9-21), RAII device buffers,
// launch helpers and the exact-arithmetic helpers used wherever a result must
// be bitwise equal to the reference's scalar C++ (no FMA contraction).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace mlg {

// errors.hpp:9-21 -> C-ABI status codes (mleig_main.cpp:57-66), plus 5 = CUDA.
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SolverError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    throw CudaError(std::string("CUDA error in ") + what + " (" + file + ":" +
                    std::to_string(line) + "): " + cudaGetErrorString(e));
}
// Per-thread message of the last failed C-ABI call (mlg_last_error, capi.cu).
std::string& last_error_slot();

// Process-wide count of this library's kernel launches (bench evidence).
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> n{0};
  return n;
}

#define MLG_CUDA(call) ::mlg::cuda_check((call), #call, __FILE__, __LINE__)
#define MLG_LAUNCH_CHECK()                                                           \
  do {                                                                               \
    ::mlg::launch_counter().fetch_add(1, std::memory_order_relaxed);                 \
    ::mlg::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);      \
  } while (0)

template <class T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(std::size_t n) { alloc(n); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) {
    o.p_ = nullptr;
    o.n_ = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_;
      n_ = o.n_;
      o.p_ = nullptr;
      o.n_ = 0;
    }
    return *this;
  }
  void alloc(std::size_t n) {
    release();
    if (n > 0) MLG_CUDA(cudaMalloc(&p_, n * sizeof(T)));
    n_ = n;
  }
  // Grow-only reallocation (contents not preserved).
  void ensure(std::size_t n) {
    if (n > n_) alloc(n);
  }
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  bool empty() const { return n_ == 0; }
  void zero(cudaStream_t s) {
    if (n_) MLG_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
  }
  void upload(const T* h, std::size_t n, cudaStream_t s) {
    if (n) MLG_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void download(T* h, std::size_t n, cudaStream_t s) const {
    if (n) MLG_CUDA(cudaMemcpyAsync(h, p_, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

inline unsigned grid_for(std::int64_t n, int block) {
  const std::int64_t g = (n + block - 1) / block;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

// Exact-order arithmetic: each op rounded separately, never fused.
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }

// Mesh::lattice_point (mesh.hpp:47-49): x_min + ix * cell_dx, unfused.
__device__ __forceinline__ double lattice_coord(double lo, int i, double d) {
  return xadd(lo, xmul(static_cast<double>(i), d));
}

}  // namespace mlg
