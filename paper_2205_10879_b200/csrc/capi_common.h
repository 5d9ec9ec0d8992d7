// Shared host-side helpers of the C ABI translation units (capi.cu,
// muygps.cu): thread-local error text, argument checks with the reference's
// messages, RAII device buffers and streams.
#pragma once

#include <cstring>

#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/fmgp_b200.h"
#include "fmgp_common.cuh"

namespace fmgp_capi {

inline thread_local std::string g_err;

// Stage timing (fmgp_set_stage_timing, capi.cu): is it on, and record one
// call's events (kNN begin, kNN end = solve begin, solve end; the events
// are destroyed by fmgp_stage_times).
bool stage_timing_on();
void stage_push(cudaEvent_t knn_begin, cudaEvent_t knn_end, cudaEvent_t solve_end);

inline int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

inline int cuda_fail(cudaError_t e, const char* where) {
  return fail(FMGP_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define FMGP_CUDA(call)                                   \
  do {                                                    \
    cudaError_t fmgp_e_ = (call);                         \
    if (fmgp_e_ != cudaSuccess) return cuda_fail(fmgp_e_, #call); \
  } while (0)

inline int num_sms_current() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

inline int require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n < 1)
    return fail(FMGP_ECUDA, std::string("no usable CUDA device (") + cudaGetErrorString(e) +
                                "); the FastMuyGPs B200 path has no CPU fallback");
  // Stage scratch comes from the stream-ordered allocator; keep freed blocks in
  // the device's default pool (release threshold = max) so repeated calls do not
  // re-map tens of MB on the host while the GPU waits.
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && dev < 64 && !(configured.load() & (1ull << dev))) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    configured.fetch_or(1ull << dev);
  }
  return FMGP_OK;
}

// KernelParams (kernel.cpp:13-28) + the device path's nu support; fills KParams.
inline int make_kparams(const fmgp_kernel_params* p, fmgp::KParams* kp) {
  if (p == nullptr) return fail(FMGP_EINVAL, "kernel params must not be null");
  if (!(std::isfinite(p->sigma) && p->sigma > 0.0))
    return fail(FMGP_EINVAL, "KernelParams: sigma must be positive and finite");
  if (!(std::isfinite(p->rho) && p->rho > 0.0))
    return fail(FMGP_EINVAL, "KernelParams: rho must be positive and finite");
  if (!(std::isfinite(p->nu) && p->nu > 0.0))
    return fail(FMGP_EINVAL, "KernelParams: nu must be positive and finite");
  if (!(std::isfinite(p->tau) && p->tau >= 0.0))
    return fail(FMGP_EINVAL, "KernelParams: tau must be non-negative and finite");
  if (p->kind != FMGP_MATERN && p->kind != FMGP_RBF) return fail(FMGP_EINVAL, "unknown kernel kind");
  kp->kind = p->kind;
  kp->nu_code = 0;
  if (p->kind == FMGP_MATERN) {
    if (p->nu == 0.5) kp->nu_code = 0;
    else if (p->nu == 1.5) kp->nu_code = 1;
    else if (p->nu == 2.5) kp->nu_code = 2;
    else kp->nu_code = 3;
  }
  kp->nu = p->nu;
  kp->sqrt2nu = std::sqrt(2.0 * p->nu);
  kp->c0 = (1.0 - p->nu) * 0.69314718055994530942 - std::lgamma(p->nu);
  kp->s2 = p->sigma * p->sigma;
  kp->rho = p->rho;
  kp->inv_rho = 1.0 / p->rho;
  kp->diag = kp->s2 * (1.0 + p->tau * p->tau);
  static const double jit[4] = {0.0, 1e-10, 1e-8, 1e-6};
  kp->diag_jit[0] = kp->diag;
  for (int a = 1; a < 4; ++a) kp->diag_jit[a] = kp->diag_jit[a - 1] + (jit[a] - jit[a - 1]);
  return FMGP_OK;
}

// Every value finite (exponent field not all ones): branch-free over blocks of
// 4096 so the compiler vectorises it (the per-call X check is on the e2e path).
inline bool all_finite(const double* X, int64_t total) {
  constexpr uint64_t kExp = 0x7FF0000000000000ull;
  for (int64_t i0 = 0; i0 < total; i0 += 4096) {
    const int64_t i1 = total < i0 + 4096 ? total : i0 + 4096;
    uint64_t bad = 0;
    for (int64_t i = i0; i < i1; ++i) {
      uint64_t b;
      std::memcpy(&b, X + i, sizeof(b));
      bad |= static_cast<uint64_t>((b & kExp) == kExp);
    }
    if (bad) return false;
  }
  return true;
}

inline int check_points(const double* X, int64_t n, int32_t d) {
  if (n < 1) return fail(FMGP_EINVAL, "NeighborIndex: empty point set");
  if (d < 1) return fail(FMGP_EINVAL, "NeighborIndex: point dimension must be >= 1");
  if (n > INT32_MAX) return fail(FMGP_EINVAL, "NeighborIndex: more than 2^31-1 points (int32 indices)");
  if (X != nullptr && !all_finite(X, n * d)) return fail(FMGP_EINVAL, "NeighborIndex: non-finite coordinates");
  return FMGP_OK;
}

// RAII device buffer on a stream (stream-ordered allocator).
template <typename T>
struct DevBuf {
  T* p = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t alloc(size_t count, cudaStream_t stream) {
    s = stream;
    if (count == 0) count = 1;
    return cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), stream);
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

// Restores the caller's current device on scope exit (entry points that
// switch devices must not leave the calling thread on another GPU).
struct DeviceGuard {
  int dev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&dev) != cudaSuccess) dev = -1;
  }
  ~DeviceGuard() {
    if (dev >= 0) cudaSetDevice(dev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

struct Stream {
  cudaStream_t s = nullptr;
  cudaError_t create() { return cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); }
  ~Stream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
};

}  // namespace fmgp_capi
