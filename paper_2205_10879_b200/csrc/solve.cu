// K2 — fused neighbourhood solve: gather -> kernel matrix -> jitter-Cholesky
// -> two triangular solves, one warp per neighbourhood, all in shared memory.
//
// Replaces, per training row i, the reference's
//   gather xs, ys                      proj/core/src/fast_predict.cpp:98-102
//   cov_matrix_self(xs)                proj/core/src/kernel.cpp:106-119
//   solve_spd / cholesky_with_jitter   proj/core/src/linalg.cpp:10-36
//   C.row(i) = solution                proj/core/src/fast_predict.cpp:104-106
//
// Shared-memory layout per warp (doubles unless noted):
//   A   k x ld (ld = k+1): the kernel matrix. The strict upper triangle keeps
//       an untouched copy of K so a failed factorisation is retried with the
//       next jitter rung (linalg.cpp:13-19) without re-gathering.
//   dg  k: the unjittered diagonal.
//   xs  k x dchunk: neighbour coordinates, streamed dchunk dims at a time.
//   B   k x m: right-hand sides, overwritten by the solution.
//   s   k int32: the neighbour indices S_i.
// Per-pair squared distances are accumulated in ascending dimension order in
// the strict lower triangle, then replaced by kernel values.
#include <cfloat>

#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

__constant__ double kJitters[4] = {0.0, 1e-10, 1e-8, 1e-6};

// The diagonal entry after jitter attempt `a`: the reference adds
// (jitter - previous) to the same matrix on every retry (linalg.cpp:14-18).
__device__ __forceinline__ double jittered(double v, int a) {
  for (int t = 1; t <= a; ++t) v = __dadd_rn(v, __dsub_rn(kJitters[t], kJitters[t - 1]));
  return v;
}

// Factor the warp's matrix (lower triangle + dg, copy in the strict upper
// triangle) under the jitter ladder. Returns the rung used, or -1.
__device__ int warp_cholesky_jitter(double* A, int ld, const double* dg, int k, int lane) {
  for (int attempt = 0; attempt < 4; ++attempt) {
    if (attempt > 0) {
      for (int a = 1; a < k; ++a)
        for (int b = lane; b < a; b += kWarp) A[a * ld + b] = A[b * ld + a];
    }
    for (int a = lane; a < k; a += kWarp) A[a * ld + a] = jittered(dg[a], attempt);
    __syncwarp();
    bool ok = true;
    for (int j = 0; j < k; ++j) {
      const double x = A[j * ld + j];
      if (!(x > 0.0)) {  // Eigen LLT: a pivot <= 0 (or NaN) fails
        ok = false;
        break;
      }
      const double ljj = sqrt(x);
      for (int i = j + 1 + lane; i < k; i += kWarp) A[i * ld + j] = A[i * ld + j] / ljj;
      __syncwarp();
      if (lane == 0) A[j * ld + j] = ljj;
      // trailing update of rows i > j, columns l in (j, i]
      for (int i = j + 1 + lane; i < k; i += kWarp) {
        const double lij = A[i * ld + j];
        double* rowi = A + i * ld;
        for (int l = j + 1; l <= i; ++l) rowi[l] = fma(-lij, A[l * ld + j], rowi[l]);
      }
      __syncwarp();
    }
    __syncwarp();
    if (ok) return attempt;
  }
  return -1;
}

// L y = b, then L^T x = y, for each of the m columns of B (k x m).
__device__ void warp_llt_solve(const double* A, int ld, double* B, int k, int m, int lane) {
  for (int c = 0; c < m; ++c) {
    for (int j = 0; j < k; ++j) {
      const double yj = B[j * m + c] / A[j * ld + j];
      __syncwarp();
      if (lane == 0) B[j * m + c] = yj;
      for (int i = j + 1 + lane; i < k; i += kWarp) B[i * m + c] = fma(-A[i * ld + j], yj, B[i * m + c]);
      __syncwarp();
    }
    for (int j = k - 1; j >= 0; --j) {
      const double xj = B[j * m + c] / A[j * ld + j];
      __syncwarp();
      if (lane == 0) B[j * m + c] = xj;
      for (int i = lane; i < j; i += kWarp) B[i * m + c] = fma(-A[j * ld + i], xj, B[i * m + c]);
      __syncwarp();
    }
  }
}

struct WarpSmem {
  double* A;
  double* dg;
  double* xs;
  double* B;
  int32_t* sr;
};

__device__ __forceinline__ WarpSmem carve(double* smem, int warp, int k, int ld, int dchunk, int m) {
  const size_t per_warp = static_cast<size_t>(k) * ld + k + static_cast<size_t>(k) * dchunk +
                          static_cast<size_t>(k) * m + (k + 1) / 2;
  WarpSmem w;
  w.A = smem + warp * per_warp;
  w.dg = w.A + static_cast<size_t>(k) * ld;
  w.xs = w.dg + k;
  w.B = w.xs + static_cast<size_t>(k) * dchunk;
  w.sr = reinterpret_cast<int32_t*>(w.B + static_cast<size_t>(k) * m);
  return w;
}

__global__ void solve_kernel(const double* __restrict__ X, const double* __restrict__ Y, int d, int m,
                             const int32_t* __restrict__ S, int64_t nrows, int64_t row_begin, int k, int ld,
                             int dchunk, KParams kp, double* __restrict__ C, int32_t* __restrict__ status,
                             unsigned long long* __restrict__ fail_min) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x % kWarp;
  const int warp = threadIdx.x / kWarp;
  const int warps = blockDim.x / kWarp;
  WarpSmem w = carve(smem, warp, k, ld, dchunk, m);
  double* A = w.A;

  for (int a = lane; a < k; a += kWarp) w.dg[a] = kp.diag;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * warps + warp; r < nrows;
       r += static_cast<int64_t>(gridDim.x) * warps) {
    // ---- gather S_i and Y_{S_i} (coalesced row loads)
    for (int t = lane; t < k; t += kWarp) w.sr[t] = S[r * k + t];
    __syncwarp();
    for (int e = lane; e < k * m; e += kWarp) {
      int t = e / m, c = e - t * m;
      w.B[e] = Y[static_cast<int64_t>(w.sr[t]) * m + c];
    }
    // ---- pairwise squared distances, dims streamed in chunks
    for (int c0 = 0; c0 < d; c0 += dchunk) {
      const int dc = min(dchunk, d - c0);
      for (int e = lane; e < k * dc; e += kWarp) {
        int t = e / dc, c = e - t * dc;
        w.xs[t * dc + c] = X[static_cast<int64_t>(w.sr[t]) * d + c0 + c];
      }
      __syncwarp();
      for (int a = 1; a < k; ++a) {
        for (int b = lane; b < a; b += kWarp) {
          double acc = c0 == 0 ? 0.0 : A[a * ld + b];
          const double* xa = w.xs + a * dc;
          const double* xb = w.xs + b * dc;
          for (int c = 0; c < dc; ++c) {
            double diff = __dsub_rn(xa[c], xb[c]);
            acc = __dadd_rn(acc, __dmul_rn(diff, diff));
          }
          A[a * ld + b] = acc;
        }
      }
      __syncwarp();
    }
    // ---- kernel values (cov_matrix_self); mirror into the upper triangle
    for (int a = 1; a < k; ++a) {
      for (int b = lane; b < a; b += kWarp) {
        double v = kernel_eval(sqrt(A[a * ld + b]), kp);
        A[a * ld + b] = v;
        A[b * ld + a] = v;
      }
    }
    __syncwarp();
    const int used = warp_cholesky_jitter(A, ld, w.dg, k, lane);
    if (used < 0) {
      if (lane == 0) {
        if (status) status[r] = -1;
        atomicMin(fail_min, static_cast<unsigned long long>(row_begin + r));
      }
      __syncwarp();
      continue;
    }
    if (status && lane == 0) status[r] = used;
    warp_llt_solve(A, ld, w.B, k, m, lane);
    for (int e = lane; e < k * m; e += kWarp) C[r * k * m + e] = w.B[e];
    __syncwarp();
  }
}

// solve_spd on given matrices (linalg.cpp:33-36): K batch x k x k row-major.
__global__ void spd_kernel(const double* __restrict__ K, const double* __restrict__ Bin, int64_t batch, int k,
                           int m, int ld, double* __restrict__ Xout, double* __restrict__ jit_out,
                           unsigned long long* __restrict__ fail_min) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x % kWarp;
  const int warp = threadIdx.x / kWarp;
  const int warps = blockDim.x / kWarp;
  WarpSmem w = carve(smem, warp, k, ld, 0, m);
  double* A = w.A;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * warps + warp; r < batch;
       r += static_cast<int64_t>(gridDim.x) * warps) {
    const double* Kr = K + r * k * k;
    for (int e = lane; e < k * k; e += kWarp) {
      int a = e / k, b = e - a * k;
      if (b < a) {
        A[a * ld + b] = Kr[e];
        A[b * ld + a] = Kr[e];
      } else if (a == b) {
        w.dg[a] = Kr[e];
      }
    }
    for (int e = lane; e < k * m; e += kWarp) w.B[e] = Bin[r * k * m + e];
    __syncwarp();
    const int used = warp_cholesky_jitter(A, ld, w.dg, k, lane);
    if (used < 0) {
      if (lane == 0) atomicMin(fail_min, static_cast<unsigned long long>(r));
      __syncwarp();
      continue;
    }
    if (jit_out && lane == 0) jit_out[r] = kJitters[used];
    warp_llt_solve(A, ld, w.B, k, m, lane);
    for (int e = lane; e < k * m; e += kWarp) Xout[r * k * m + e] = w.B[e];
    __syncwarp();
  }
}

template <typename Kern>
cudaError_t launch_warp_per_item(Kern kern, size_t per_warp, int64_t items, int num_sms, cudaStream_t stream,
                                 int* warps_out, size_t* smem_out, int64_t* grid_out) {
  const size_t budget = 200 * 1024;
  int warps = static_cast<int>(budget / per_warp);
  if (warps > 8) warps = 8;
  if (warps < 1) return cudaErrorInvalidValue;
  const size_t smem = per_warp * warps;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  int blocks_per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, warps * kWarp, smem);
  if (err != cudaSuccess) return err;
  if (blocks_per_sm < 1) blocks_per_sm = 1;
  const int64_t need = (items + warps - 1) / warps;
  *grid_out = std::min<int64_t>(need, static_cast<int64_t>(num_sms) * blocks_per_sm);
  *warps_out = warps;
  *smem_out = smem;
  (void)stream;
  return cudaSuccess;
}

}  // namespace

size_t solve_smem_per_warp(int k, int d, int m, int* ld, int* dchunk) {
  *ld = k + 1;
  int dc = 1024 / (k > 0 ? k : 1);
  if (dc < 1) dc = 1;
  if (dc > d) dc = d;
  *dchunk = dc;
  return (static_cast<size_t>(k) * *ld + k + static_cast<size_t>(k) * dc + static_cast<size_t>(k) * m +
          (k + 1) / 2) *
         sizeof(double);
}

cudaError_t fused_solve(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                        int64_t row_begin, int k, const KParams& kp, double* C, int32_t* status,
                        unsigned long long* fail_min, int num_sms, cudaStream_t stream) {
  if (nrows <= 0) return cudaSuccess;
  int ld, dchunk, warps;
  size_t smem;
  int64_t grid;
  const size_t per_warp = solve_smem_per_warp(k, d, m, &ld, &dchunk);
  cudaError_t err = launch_warp_per_item(solve_kernel, per_warp, nrows, num_sms, stream, &warps, &smem, &grid);
  if (err != cudaSuccess) return err;
  solve_kernel<<<static_cast<unsigned>(grid), warps * kWarp, smem, stream>>>(
      X, Y, d, m, S, nrows, row_begin, k, ld, dchunk, kp, C, status, fail_min);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t spd_solve_batched(const double* K, const double* B, int64_t batch, int k, int m, double* X,
                              double* jit_out, unsigned long long* fail_min, int num_sms, cudaStream_t stream) {
  if (batch <= 0) return cudaSuccess;
  int ld, dchunk, warps;
  size_t smem;
  int64_t grid;
  size_t per_warp = solve_smem_per_warp(k, 1, m, &ld, &dchunk);
  per_warp -= static_cast<size_t>(k) * dchunk * sizeof(double);
  cudaError_t err = launch_warp_per_item(spd_kernel, per_warp, batch, num_sms, stream, &warps, &smem, &grid);
  if (err != cudaSuccess) return err;
  spd_kernel<<<static_cast<unsigned>(grid), warps * kWarp, smem, stream>>>(K, B, batch, k, m, ld, X, jit_out,
                                                                          fail_min);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace fmgp
