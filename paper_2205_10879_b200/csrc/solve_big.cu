// K2-big — the jitter-Cholesky solve for neighbourhoods too large for the
// warp-per-neighbourhood shared-memory kernel (k > kMaxK or m large). One CTA
// per matrix, persistent over rows, with the k x k matrix in a global-memory
// workspace (L2-resident for the sizes this serves). Same semantics as
// solve.cu: lower triangle = working factor, strict upper triangle = the
// untouched kernel matrix for jitter retries (linalg.cpp:13-19), dg = the
// unjittered diagonal. Not on the BASELINE hot path (k <= 100 there); it keeps
// the drop-in complete for any k <= n, like the reference.
#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

constexpr int kBigThreads = 256;
__constant__ double kJit[4] = {0.0, 1e-10, 1e-8, 1e-6};

__device__ __forceinline__ double jittered_big(double v, int a) {
  for (int t = 1; t <= a; ++t) v = __dadd_rn(v, __dsub_rn(kJit[t], kJit[t - 1]));
  return v;
}

__device__ int cta_cholesky_jitter(double* A, const double* dg, int k) {
  __shared__ int ok_s;
  for (int attempt = 0; attempt < 4; ++attempt) {
    if (attempt > 0) {
      for (int64_t e = threadIdx.x; e < static_cast<int64_t>(k) * k; e += blockDim.x) {
        const int a = static_cast<int>(e / k), b = static_cast<int>(e % k);
        if (b < a) A[static_cast<int64_t>(a) * k + b] = A[static_cast<int64_t>(b) * k + a];
      }
    }
    for (int a = threadIdx.x; a < k; a += blockDim.x) A[static_cast<int64_t>(a) * k + a] = jittered_big(dg[a], attempt);
    if (threadIdx.x == 0) ok_s = 1;
    __syncthreads();
    for (int j = 0; j < k; ++j) {
      const double x = A[static_cast<int64_t>(j) * k + j];
      if (!(x > 0.0)) {
        if (threadIdx.x == 0) ok_s = 0;
        break;  // uniform: every thread read the same pivot
      }
      const double ljj = sqrt(x);
      for (int i = j + 1 + threadIdx.x; i < k; i += blockDim.x) A[static_cast<int64_t>(i) * k + j] /= ljj;
      __syncthreads();
      if (threadIdx.x == 0) A[static_cast<int64_t>(j) * k + j] = ljj;
      for (int i = j + 1 + threadIdx.x; i < k; i += blockDim.x) {
        const double lij = A[static_cast<int64_t>(i) * k + j];
        double* rowi = A + static_cast<int64_t>(i) * k;
        for (int l = j + 1; l <= i; ++l) rowi[l] = fma(-lij, A[static_cast<int64_t>(l) * k + j], rowi[l]);
      }
      __syncthreads();
    }
    __syncthreads();
    if (ok_s) return attempt;
    __syncthreads();
  }
  return -1;
}

// L y = b then L^T x = y for each of the m columns of B (k x m, global).
__device__ void cta_llt_solve(const double* A, double* B, int k, int m) {
  for (int c = 0; c < m; ++c) {
    for (int j = 0; j < k; ++j) {
      const double yj = B[static_cast<int64_t>(j) * m + c] / A[static_cast<int64_t>(j) * k + j];
      __syncthreads();
      if (threadIdx.x == 0) B[static_cast<int64_t>(j) * m + c] = yj;
      for (int i = j + 1 + threadIdx.x; i < k; i += blockDim.x)
        B[static_cast<int64_t>(i) * m + c] =
            fma(-A[static_cast<int64_t>(i) * k + j], yj, B[static_cast<int64_t>(i) * m + c]);
      __syncthreads();
    }
    for (int j = k - 1; j >= 0; --j) {
      const double xj = B[static_cast<int64_t>(j) * m + c] / A[static_cast<int64_t>(j) * k + j];
      __syncthreads();
      if (threadIdx.x == 0) B[static_cast<int64_t>(j) * m + c] = xj;
      for (int i = threadIdx.x; i < j; i += blockDim.x)
        B[static_cast<int64_t>(i) * m + c] =
            fma(-A[static_cast<int64_t>(j) * k + i], xj, B[static_cast<int64_t>(i) * m + c]);
      __syncthreads();
    }
  }
}

// Precompute rows with a global-memory neighbourhood (fast_predict.cpp:98-106).
__global__ void __launch_bounds__(kBigThreads)
solve_big_kernel(const double* __restrict__ X, const double* __restrict__ Y, int d, int m,
                 const int32_t* __restrict__ S, int64_t nrows, int64_t row_begin, int k, KParams kp,
                 double* __restrict__ C, unsigned long long* __restrict__ fail_min, double* __restrict__ work) {
  double* A = work + static_cast<int64_t>(blockIdx.x) * (static_cast<int64_t>(k) * k + k + static_cast<int64_t>(k) * m);
  double* dg = A + static_cast<int64_t>(k) * k;
  double* B = dg + k;
  for (int a = threadIdx.x; a < k; a += blockDim.x) dg[a] = kp.diag;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const int32_t* sr = S + r * k;
    for (int e = threadIdx.x; e < k * m; e += blockDim.x) {
      const int t = e / m, c = e - t * m;
      B[e] = Y[static_cast<int64_t>(sr[t]) * m + c];
    }
    for (int64_t e = threadIdx.x; e < static_cast<int64_t>(k) * k; e += blockDim.x) {
      const int a = static_cast<int>(e / k), b = static_cast<int>(e % k);
      if (b < a) {
        const double v = kernel_eval(
            sqrt(dist_sq_dyn(X + static_cast<int64_t>(sr[a]) * d, X + static_cast<int64_t>(sr[b]) * d, d)), kp);
        A[static_cast<int64_t>(a) * k + b] = v;
        A[static_cast<int64_t>(b) * k + a] = v;
      }
    }
    __syncthreads();
    const int used = cta_cholesky_jitter(A, dg, k);
    if (used < 0) {
      if (threadIdx.x == 0) atomicMin(fail_min, static_cast<unsigned long long>(row_begin + r));
      __syncthreads();
      continue;
    }
    cta_llt_solve(A, B, k, m);
    for (int e = threadIdx.x; e < k * m; e += blockDim.x) C[r * k * m + e] = B[e];
    __syncthreads();
  }
}

// solve_spd on given matrices (linalg.cpp:33-36).
__global__ void __launch_bounds__(kBigThreads)
spd_big_kernel(const double* __restrict__ K, const double* __restrict__ Bin, int64_t batch, int k, int m,
               double* __restrict__ Xout, double* __restrict__ jit_out, unsigned long long* __restrict__ fail_min,
               double* __restrict__ work) {
  double* A = work + static_cast<int64_t>(blockIdx.x) * (static_cast<int64_t>(k) * k + k + static_cast<int64_t>(k) * m);
  double* dg = A + static_cast<int64_t>(k) * k;
  double* B = dg + k;
  for (int64_t r = blockIdx.x; r < batch; r += gridDim.x) {
    const double* Kr = K + r * k * k;
    for (int64_t e = threadIdx.x; e < static_cast<int64_t>(k) * k; e += blockDim.x) {
      const int a = static_cast<int>(e / k), b = static_cast<int>(e % k);
      if (b < a) {
        A[static_cast<int64_t>(a) * k + b] = Kr[e];
        A[static_cast<int64_t>(b) * k + a] = Kr[e];
      } else if (a == b) {
        dg[a] = Kr[e];
      }
    }
    for (int e = threadIdx.x; e < k * m; e += blockDim.x) B[e] = Bin[r * k * m + e];
    __syncthreads();
    const int used = cta_cholesky_jitter(A, dg, k);
    if (used < 0) {
      if (threadIdx.x == 0) atomicMin(fail_min, static_cast<unsigned long long>(r));
      __syncthreads();
      continue;
    }
    if (jit_out && threadIdx.x == 0) jit_out[r] = kJit[used];
    cta_llt_solve(A, B, k, m);
    for (int e = threadIdx.x; e < k * m; e += blockDim.x) Xout[r * k * m + e] = B[e];
    __syncthreads();
  }
}

int64_t big_grid(int64_t items, int num_sms) {
  int64_t g = items < static_cast<int64_t>(num_sms) * 2 ? items : static_cast<int64_t>(num_sms) * 2;
  return g < 1 ? 1 : g;
}

}  // namespace

cudaError_t fused_solve_big(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                            int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                            int num_sms, cudaStream_t stream) {
  if (nrows <= 0) return cudaSuccess;
  const int64_t grid = big_grid(nrows, num_sms);
  double* work = nullptr;
  cudaError_t err = cudaMallocAsync(&work, sizeof(double) * grid * (static_cast<int64_t>(k) * k + k + static_cast<int64_t>(k) * m),
                                    stream);
  if (err != cudaSuccess) return err;
  solve_big_kernel<<<static_cast<unsigned>(grid), kBigThreads, 0, stream>>>(X, Y, d, m, S, nrows, row_begin, k, kp, C,
                                                                           fail_min, work);
  note_launches(1);
  err = cudaGetLastError();
  cudaFreeAsync(work, stream);
  return err;
}

cudaError_t spd_solve_big(const double* K, const double* B, int64_t batch, int k, int m, double* X, double* jit_out,
                          unsigned long long* fail_min, int num_sms, cudaStream_t stream) {
  if (batch <= 0) return cudaSuccess;
  const int64_t grid = big_grid(batch, num_sms);
  double* work = nullptr;
  cudaError_t err = cudaMallocAsync(&work, sizeof(double) * grid * (static_cast<int64_t>(k) * k + k + static_cast<int64_t>(k) * m),
                                    stream);
  if (err != cudaSuccess) return err;
  spd_big_kernel<<<static_cast<unsigned>(grid), kBigThreads, 0, stream>>>(K, B, batch, k, m, X, jit_out, fail_min,
                                                                         work);
  note_launches(1);
  err = cudaGetLastError();
  cudaFreeAsync(work, stream);
  return err;
}

}  // namespace fmgp
