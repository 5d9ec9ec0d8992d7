// Small element-wise kernels behind the C ABI: the kernel-arithmetic entry
// points (kernel.cpp:88-119) and helpers for the neighbour table.
#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

// cov_matrix (kernel.cpp:92-104): K(i,j) = kernel(||A_i - B_j||), with the
// nugget firing on exact coordinate equality. cov_matrix_self (:106-119):
// diagonal kernel(0), off-diagonal computed once for i < j and mirrored, so
// the fill is exactly symmetric.
__global__ void cov_kernel(const double* __restrict__ A, int64_t na, const double* __restrict__ B, int64_t nb,
                           int d, KParams kp, double* __restrict__ K) {
  const int64_t total = na * nb;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / nb, j = e - i * nb;
    double v;
    if (B == nullptr) {
      if (i == j) {
        v = kernel_eval(0.0, kp);
      } else {
        const int64_t lo = i < j ? i : j, hi = i < j ? j : i;
        v = kernel_eval(sqrt(dist_sq_dyn(A + lo * d, A + hi * d, d)), kp);
      }
    } else {
      v = kernel_eval(sqrt(dist_sq_dyn(A + i * d, B + j * d, d)), kp);
    }
    K[e] = v;
  }
}

__global__ void kernel_values_kernel(const double* __restrict__ dist, int64_t n, KParams kp,
                                     double* __restrict__ out) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[e] = kernel_eval(dist[e], kp);
}

__global__ void sqrt_kernel(double* __restrict__ v, int64_t n) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[e] = sqrt(v[e]);
}

// Count of non-finite values (exponent field all ones), the device half of
// NeighborIndex::build's finiteness check on the host-buffer path.
__global__ void nonfinite_kernel(const double* __restrict__ v, int64_t n, unsigned int* __restrict__ count) {
  unsigned int bad = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad += (__double2hiint(v[i]) & 0x7ff00000) == 0x7ff00000 ? 1u : 0u;
  bad = __reduce_add_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(count, bad);
}

// The same count on a buffer the caller owns, replacing each non-finite value by 0: the
// kernels that follow (cell sort, walk) then run on valid coordinates, and the caller
// turns a non-zero count into the error return after its final synchronise.
__global__ void nonfinite_zero_kernel(double* __restrict__ v, int64_t n, unsigned int* __restrict__ count) {
  unsigned int bad = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if ((__double2hiint(v[i]) & 0x7ff00000) == 0x7ff00000) {
      v[i] = 0.0;
      ++bad;
    }
  }
  bad = __reduce_add_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(count, bad);
}

__global__ void self_rows_kernel(int32_t* __restrict__ S, int64_t nrows, int64_t row_begin) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < nrows;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    S[e] = static_cast<int32_t>(row_begin + e);
}

// distance_to (nn_index.cpp:344-349): sqrt(dist_sq(q, P[idx[e]])).
__global__ void distances_kernel(const double* __restrict__ P, int d, const double* __restrict__ q,
                                 const int32_t* __restrict__ idx, int64_t cnt, double* __restrict__ out) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < cnt;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[e] = sqrt(dist_sq_dyn(q, P + static_cast<int64_t>(idx[e]) * d, d));
}

unsigned grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

}  // namespace

cudaError_t cov_matrix_launch(const double* A, int64_t na, const double* B, int64_t nb, int d, const KParams& kp,
                              double* K, cudaStream_t stream) {
  if (na * nb == 0) return cudaSuccess;
  cov_kernel<<<grid_for(na * nb), 256, 0, stream>>>(A, na, B, nb, d, kp, K);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t kernel_values_launch(const double* dist, int64_t n, const KParams& kp, double* out,
                                 cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  kernel_values_kernel<<<grid_for(n), 256, 0, stream>>>(dist, n, kp, out);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t sqrt_inplace_launch(double* v, int64_t n, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  sqrt_kernel<<<grid_for(n), 256, 0, stream>>>(v, n);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t distances_launch(const double* P, int d, const double* q, const int32_t* idx, int64_t cnt, double* out,
                             cudaStream_t stream) {
  if (cnt == 0) return cudaSuccess;
  distances_kernel<<<grid_for(cnt), 256, 0, stream>>>(P, d, q, idx, cnt, out);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t nonfinite_count_launch(const double* v, int64_t n, unsigned int* count, int num_sms,
                                   cudaStream_t stream) {
  cudaError_t err = cudaMemsetAsync(count, 0, sizeof(unsigned int), stream);
  if (err != cudaSuccess || n <= 0) return err;
  int64_t blocks = (n + 255) / 256;
  if (blocks > static_cast<int64_t>(num_sms) * 8) blocks = static_cast<int64_t>(num_sms) * 8;
  nonfinite_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(v, n, count);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t nonfinite_zero_launch(double* v, int64_t n, unsigned int* count, int num_sms, cudaStream_t stream) {
  cudaError_t err = cudaMemsetAsync(count, 0, sizeof(unsigned int), stream);
  if (err != cudaSuccess || n <= 0) return err;
  int64_t blocks = (n + 255) / 256;
  if (blocks > static_cast<int64_t>(num_sms) * 8) blocks = static_cast<int64_t>(num_sms) * 8;
  nonfinite_zero_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(v, n, count);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t self_rows_launch(int32_t* S, int64_t nrows, int64_t row_begin, cudaStream_t stream) {
  if (nrows == 0) return cudaSuccess;
  self_rows_kernel<<<grid_for(nrows), 256, 0, stream>>>(S, nrows, row_begin);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace fmgp

// ---------------------------------------------------------------- diagnostics
// The FP64 roofline denominators of this GPU, measured in the caller's
// process (bench.py reports the solve's FP64 fraction against them):
// independent DFMA chains and DMMA m8n8k4 chains over the whole chip.
namespace fmgp {
namespace {

constexpr int kPeakChains = 8;
constexpr int kPeakIters = 4096;

__global__ void peak_dfma_kernel(double* out, double a, double b) {
  double x[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
    for (int c = 0; c < kPeakChains; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kPeakChains; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void peak_dmma_kernel(double* out, double a, double b) {
  double c[kPeakChains][2];
#pragma unroll
  for (int q = 0; q < kPeakChains; ++q) c[q][0] = c[q][1] = threadIdx.x * 1e-3 + q;
  for (int i = 0; i < kPeakIters; ++i) {
#pragma unroll
    for (int q = 0; q < kPeakChains; ++q)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c[q][0]), "+d"(c[q][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < kPeakChains; ++q) s += c[q][0] + c[q][1];
  if (s == 12345.678) out[0] = s;
}

}  // namespace
}  // namespace fmgp

extern "C" int fmgp_diag_fp64_peak(double* dfma_tflops, double* dmma_tflops) {
  using namespace fmgp;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess) return 3;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* sink = nullptr;
  if (cudaMalloc(&sink, sizeof(double)) != cudaSuccess) return 3;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  const double fma_flops = 2.0 * blocks * threads * kPeakChains * double(kPeakIters);
  const double mma_flops = 512.0 * (blocks * threads / 32) * kPeakChains * double(kPeakIters);
  float best_f = 1e30f, best_m = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    float t = 0.f;
    cudaEventRecord(e0);
    peak_dfma_kernel<<<blocks, threads>>>(sink, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t, e0, e1);
    if (rep > 0) best_f = t < best_f ? t : best_f;
    cudaEventRecord(e0);
    peak_dmma_kernel<<<blocks, threads>>>(sink, 0.999, 1e-3);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&t, e0, e1);
    if (rep > 0) best_m = t < best_m ? t : best_m;
  }
  note_launches(8);
  const cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (err != cudaSuccess) return 3;
  if (dfma_tflops) *dfma_tflops = fma_flops / (best_f * 1e-3) / 1e12;
  if (dmma_tflops) *dmma_tflops = mma_flops / (best_m * 1e-3) / 1e12;
  return 0;
}
