// K2 — fused neighbourhood solve: gather -> kernel matrix -> jitter-Cholesky
// -> two triangular solves, one warp per neighbourhood, all in shared memory.
//
// Replaces, per training row i, the reference's
//   gather xs, ys                      proj/core/src/fast_predict.cpp:98-102
//   cov_matrix_self(xs)                proj/core/src/kernel.cpp:106-119
//   solve_spd / cholesky_with_jitter   proj/core/src/linalg.cpp:10-36
//   C.row(i) = solution                proj/core/src/fast_predict.cpp:104-106
//
// Shared memory per warp (doubles unless noted):
//   A   k(k+1)/2: the lower triangle, packed column-major: column p holds rows
//       p..k-1 contiguously at offset p*k - p(p-1)/2, so a warp reading one
//       column (lanes = rows) is conflict-free and a pivot-row element is a
//       broadcast.
//   xs  k x dchunk: neighbour coordinates, dchunk dims at a time (coalesced
//       row gathers from X).
//   B   k x m right-hand sides -> solution;  s  k int32 neighbour indices.
// Squared distances are accumulated over dims in ascending order in A's
// strict lower triangle, then replaced by kernel values; the diagonal is
// sigma^2 (1 + tau^2) plus the jitter rung. A failed factorisation rebuilds K
// with the next rung of {0, 1e-10, 1e-8, 1e-6} (linalg.cpp:13-19), so no copy
// of K is kept (retries are rare), which halves the footprint and doubles the
// warps per SM.
//
// Cholesky is left-looking by columns: lane l owns rows j + l + 32c
// (c < R = ceil(k/32)) of the current column and accumulates
// a_ij - sum_p L_ip L_jp in registers with two interleaved partial sums.
#include <cfloat>

#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

__constant__ double kJitters[4] = {0.0, 1e-10, 1e-8, 1e-6};

__host__ __device__ __forceinline__ int coff(int p, int k) { return p * k - ((p * (p - 1)) >> 1); }

// The diagonal after jitter attempt `a`: the reference adds (jitter - previous)
// to the same matrix on every retry (linalg.cpp:14-18).
__device__ __forceinline__ double jittered(double v, int a) {
  for (int t = 1; t <= a; ++t) v = __dadd_rn(v, __dsub_rn(kJitters[t], kJitters[t - 1]));
  return v;
}

// In-place lower Cholesky of the packed matrix; false at the first pivot <= 0
// (Eigen LLT semantics; NaN fails too).
template <int R>
__device__ bool warp_cholesky(double* A, int k, int lane) {
  for (int j = 0; j < k; ++j) {
    const int oj = coff(j, k);
    double acc0[R], acc1[R];
#pragma unroll
    for (int c = 0; c < R; ++c) {
      const int i = j + lane + 32 * c;
      acc0[c] = i < k ? A[oj + i - j] : 0.0;
      acc1[c] = 0.0;
    }
    int p = 0;
    for (; p + 1 < j; p += 2) {
      const int op0 = coff(p, k), op1 = op0 + (k - p);  // coff(p + 1)
      const double l0 = A[op0 + j - p];
      const double l1 = A[op1 + j - p - 1];
#pragma unroll
      for (int c = 0; c < R; ++c) {
        const int i = j + lane + 32 * c;
        if (i < k) {
          acc0[c] = fma(-A[op0 + i - p], l0, acc0[c]);
          acc1[c] = fma(-A[op1 + i - p - 1], l1, acc1[c]);
        }
      }
    }
    if (p < j) {
      const int op = coff(p, k);
      const double l0 = A[op + j - p];
#pragma unroll
      for (int c = 0; c < R; ++c) {
        const int i = j + lane + 32 * c;
        if (i < k) acc0[c] = fma(-A[op + i - p], l0, acc0[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < R; ++c) acc0[c] += acc1[c];
    const double piv = __shfl_sync(0xffffffffu, acc0[0], 0);  // row j = lane 0, c = 0
    if (!(piv > 0.0)) return false;
    const double ljj = sqrt(piv);
    __syncwarp();
#pragma unroll
    for (int c = 0; c < R; ++c) {
      const int i = j + lane + 32 * c;
      if (i < k) A[oj + i - j] = (c == 0 && lane == 0) ? ljj : acc0[c] / ljj;
    }
    __syncwarp();
  }
  return true;
}

// L y = b then L^T x = y for each of the m columns of B (k x m).
__device__ void warp_llt_solve(const double* A, double* B, int k, int m, int lane) {
  for (int c = 0; c < m; ++c) {
    // forward, right-looking: y_j = b_j / L_jj; b_i -= L_ij y_j (column j contiguous)
    for (int j = 0; j < k; ++j) {
      const int oj = coff(j, k);
      const double yj = B[j * m + c] / A[oj];
      __syncwarp();
      for (int i = j + 1 + lane; i < k; i += kWarp) B[i * m + c] = fma(-A[oj + i - j], yj, B[i * m + c]);
      if (lane == 0) B[j * m + c] = yj;
      __syncwarp();
    }
    // backward: x_j = (y_j - sum_{i>j} L_ij x_i) / L_jj, a warp dot product per j
    for (int j = k - 1; j >= 0; --j) {
      const int oj = coff(j, k);
      double s = 0.0;
      for (int i = j + 1 + lane; i < k; i += kWarp) s = fma(A[oj + i - j], B[i * m + c], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      const double xj = (B[j * m + c] - s) / A[oj];
      __syncwarp();
      if (lane == 0) B[j * m + c] = xj;
      __syncwarp();
    }
  }
}

struct WarpSmem {
  double* A;
  double* xs;
  double* B;
  int32_t* sr;
};

__host__ __device__ __forceinline__ size_t per_warp_doubles(int k, int dchunk, int m) {
  return static_cast<size_t>(k) * (k + 1) / 2 + static_cast<size_t>(k) * dchunk + static_cast<size_t>(k) * m +
         (k + 1) / 2 + 1;
}

__device__ __forceinline__ WarpSmem carve(double* smem, int warp, int k, int dchunk, int m) {
  WarpSmem w;
  w.A = smem + warp * per_warp_doubles(k, dchunk, m);
  w.xs = w.A + static_cast<size_t>(k) * (k + 1) / 2;
  w.B = w.xs + static_cast<size_t>(k) * dchunk;
  w.sr = reinterpret_cast<int32_t*>(w.B + static_cast<size_t>(k) * m);
  return w;
}

// K(S_i) (cov_matrix_self, kernel.cpp:106-119) into the packed triangle with
// the diagonal at jitter rung `attempt`. Coordinates are gathered from X in
// dchunk-wide slices (the whole point when d <= dchunk).
__device__ void build_kernel_matrix(const double* __restrict__ X, int d, const int32_t* sr, int k, int dchunk,
                                    const KParams& kp, int attempt, double* A, double* xs, int lane) {
  for (int c0 = 0; c0 < d; c0 += dchunk) {
    const int dc = min(dchunk, d - c0);
    for (int e = lane; e < k * dc; e += kWarp) {
      const int t = e / dc, c = e - t * dc;
      xs[t * dc + c] = X[static_cast<int64_t>(sr[t]) * d + c0 + c];
    }
    __syncwarp();
    for (int p = 0; p < k - 1; ++p) {
      const int op = coff(p, k);
      const double* xb = xs + p * dc;
      for (int i = p + 1 + lane; i < k; i += kWarp) {
        double acc = c0 == 0 ? 0.0 : A[op + i - p];
        const double* xa = xs + i * dc;
        for (int c = 0; c < dc; ++c) {
          const double diff = __dsub_rn(xa[c], xb[c]);
          acc = __dadd_rn(acc, __dmul_rn(diff, diff));
        }
        A[op + i - p] = acc;
      }
    }
    __syncwarp();
  }
  const double dg = jittered(kp.diag, attempt);
  for (int p = 0; p < k; ++p) {
    const int op = coff(p, k);
    for (int i = p + lane; i < k; i += kWarp) A[op + i - p] = i == p ? dg : kernel_eval(sqrt(A[op + i - p]), kp);
  }
  __syncwarp();
}

template <int R>
__global__ void __launch_bounds__(256)
solve_kernel(const double* __restrict__ X, const double* __restrict__ Y, int d, int m, const int32_t* __restrict__ S,
             int64_t nrows, int64_t row_begin, int k, int dchunk, KParams kp, double* __restrict__ C,
             int32_t* __restrict__ status, unsigned long long* __restrict__ fail_min) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x % kWarp;
  const int warp = threadIdx.x / kWarp;
  const int warps = blockDim.x / kWarp;
  WarpSmem w = carve(smem, warp, k, dchunk, m);

  for (int64_t r = static_cast<int64_t>(blockIdx.x) * warps + warp; r < nrows;
       r += static_cast<int64_t>(gridDim.x) * warps) {
    for (int t = lane; t < k; t += kWarp) w.sr[t] = S[r * k + t];
    __syncwarp();
    int used = -1;
    for (int attempt = 0; attempt < 4; ++attempt) {
      build_kernel_matrix(X, d, w.sr, k, dchunk, kp, attempt, w.A, w.xs, lane);
      if (warp_cholesky<R>(w.A, k, lane)) {
        used = attempt;
        break;
      }
    }
    if (used < 0) {
      if (lane == 0) {
        if (status) status[r] = -1;
        atomicMin(fail_min, static_cast<unsigned long long>(row_begin + r));
      }
      __syncwarp();
      continue;
    }
    if (status && lane == 0) status[r] = used;
    for (int e = lane; e < k * m; e += kWarp) {
      const int t = e / m, c = e - t * m;
      w.B[e] = Y[static_cast<int64_t>(w.sr[t]) * m + c];
    }
    __syncwarp();
    warp_llt_solve(w.A, w.B, k, m, lane);
    for (int e = lane; e < k * m; e += kWarp) C[r * k * m + e] = w.B[e];
    __syncwarp();
  }
}

// solve_spd on given matrices (linalg.cpp:33-36): K batch x k x k row-major,
// lower triangle used.
template <int R>
__global__ void __launch_bounds__(256)
spd_kernel(const double* __restrict__ K, const double* __restrict__ Bin, int64_t batch, int k, int m,
           double* __restrict__ Xout, double* __restrict__ jit_out, unsigned long long* __restrict__ fail_min) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x % kWarp;
  const int warp = threadIdx.x / kWarp;
  const int warps = blockDim.x / kWarp;
  WarpSmem w = carve(smem, warp, k, 0, m);
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * warps + warp; r < batch;
       r += static_cast<int64_t>(gridDim.x) * warps) {
    const double* Kr = K + r * k * k;
    int used = -1;
    for (int attempt = 0; attempt < 4; ++attempt) {
      for (int p = 0; p < k; ++p) {
        const int op = coff(p, k);
        for (int i = p + lane; i < k; i += kWarp)
          w.A[op + i - p] = i == p ? jittered(Kr[static_cast<int64_t>(p) * k + p], attempt)
                                   : Kr[static_cast<int64_t>(i) * k + p];
      }
      __syncwarp();
      if (warp_cholesky<R>(w.A, k, lane)) {
        used = attempt;
        break;
      }
    }
    if (used < 0) {
      if (lane == 0) atomicMin(fail_min, static_cast<unsigned long long>(r));
      __syncwarp();
      continue;
    }
    if (jit_out && lane == 0) jit_out[r] = kJitters[used];
    for (int e = lane; e < k * m; e += kWarp) w.B[e] = Bin[r * k * m + e];
    __syncwarp();
    warp_llt_solve(w.A, w.B, k, m, lane);
    for (int e = lane; e < k * m; e += kWarp) Xout[r * k * m + e] = w.B[e];
    __syncwarp();
  }
}

constexpr size_t kSmemBudget = 220 * 1024;

struct LaunchShape {
  int warps;
  size_t smem;
  int64_t grid;
};

template <typename Kern>
cudaError_t shape_for(Kern kern, size_t per_warp_bytes, int64_t items, int num_sms, LaunchShape* out) {
  int warps = static_cast<int>(std::min<size_t>(8, kSmemBudget / per_warp_bytes));
  if (warps < 1) return cudaErrorInvalidValue;
  const size_t smem = per_warp_bytes * warps;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  int blocks_per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, warps * kWarp, smem);
  if (err != cudaSuccess) return err;
  if (blocks_per_sm < 1) blocks_per_sm = 1;
  const int64_t need = (items + warps - 1) / warps;
  out->grid = std::min<int64_t>(need, static_cast<int64_t>(num_sms) * blocks_per_sm);
  out->warps = warps;
  out->smem = smem;
  return cudaSuccess;
}

int dchunk_for(int k, int d) {
  int dc = 512 / (k > 0 ? k : 1);
  if (dc < 1) dc = 1;
  return dc > d ? d : dc;
}

template <int R>
cudaError_t launch_solve(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                         int64_t row_begin, int k, const KParams& kp, double* C, int32_t* status,
                         unsigned long long* fail_min, int num_sms, cudaStream_t stream) {
  const int dchunk = dchunk_for(k, d);
  LaunchShape sh;
  cudaError_t err = shape_for(solve_kernel<R>, per_warp_doubles(k, dchunk, m) * sizeof(double), nrows, num_sms, &sh);
  if (err != cudaSuccess) return err;
  solve_kernel<R><<<static_cast<unsigned>(sh.grid), sh.warps * kWarp, sh.smem, stream>>>(
      X, Y, d, m, S, nrows, row_begin, k, dchunk, kp, C, status, fail_min);
  note_launches(1);
  return cudaGetLastError();
}

template <int R>
cudaError_t launch_spd(const double* K, const double* B, int64_t batch, int k, int m, double* X, double* jit_out,
                       unsigned long long* fail_min, int num_sms, cudaStream_t stream) {
  LaunchShape sh;
  cudaError_t err = shape_for(spd_kernel<R>, per_warp_doubles(k, 0, m) * sizeof(double), batch, num_sms, &sh);
  if (err != cudaSuccess) return err;
  spd_kernel<R><<<static_cast<unsigned>(sh.grid), sh.warps * kWarp, sh.smem, stream>>>(K, B, batch, k, m, X, jit_out,
                                                                                      fail_min);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace

size_t solve_smem_per_warp(int k, int d, int m, int* ld, int* dchunk) {
  *ld = k;
  *dchunk = dchunk_for(k, d);
  return per_warp_doubles(k, *dchunk, m) * sizeof(double);
}

cudaError_t fused_solve(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                        int64_t row_begin, int k, const KParams& kp, double* C, int32_t* status,
                        unsigned long long* fail_min, int num_sms, cudaStream_t stream) {
  if (nrows <= 0) return cudaSuccess;
  const size_t bytes = per_warp_doubles(k, dchunk_for(k, d), m) * sizeof(double);
  if (k > kMaxK || bytes > kSmemBudget)
    return fused_solve_big(X, Y, d, m, S, nrows, row_begin, k, kp, C, fail_min, num_sms, stream);
  switch ((k + 31) / 32) {
    case 1: return launch_solve<1>(X, Y, d, m, S, nrows, row_begin, k, kp, C, status, fail_min, num_sms, stream);
    case 2: return launch_solve<2>(X, Y, d, m, S, nrows, row_begin, k, kp, C, status, fail_min, num_sms, stream);
    case 3: return launch_solve<3>(X, Y, d, m, S, nrows, row_begin, k, kp, C, status, fail_min, num_sms, stream);
    case 4: return launch_solve<4>(X, Y, d, m, S, nrows, row_begin, k, kp, C, status, fail_min, num_sms, stream);
    default: return launch_solve<5>(X, Y, d, m, S, nrows, row_begin, k, kp, C, status, fail_min, num_sms, stream);
  }
}

cudaError_t spd_solve_batched(const double* K, const double* B, int64_t batch, int k, int m, double* X,
                              double* jit_out, unsigned long long* fail_min, int num_sms, cudaStream_t stream) {
  if (batch <= 0) return cudaSuccess;
  const size_t bytes = per_warp_doubles(k, 0, m) * sizeof(double);
  if (k > kMaxK || bytes > kSmemBudget) return spd_solve_big(K, B, batch, k, m, X, jit_out, fail_min, num_sms, stream);
  switch ((k + 31) / 32) {
    case 1: return launch_spd<1>(K, B, batch, k, m, X, jit_out, fail_min, num_sms, stream);
    case 2: return launch_spd<2>(K, B, batch, k, m, X, jit_out, fail_min, num_sms, stream);
    case 3: return launch_spd<3>(K, B, batch, k, m, X, jit_out, fail_min, num_sms, stream);
    case 4: return launch_spd<4>(K, B, batch, k, m, X, jit_out, fail_min, num_sms, stream);
    default: return launch_spd<5>(K, B, batch, k, m, X, jit_out, fail_min, num_sms, stream);
  }
}

}  // namespace fmgp
