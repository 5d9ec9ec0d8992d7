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
//   A   the lower triangle, packed ROW-major with every row padded to an even
//       length: row i holds L[i][0..i] at ro(i) = i(i+1)/2 + ceil(i/2), so
//       rows start 16-byte aligned and two consecutive entries are one
//       128-bit load. Left-looking Cholesky, the forward solve and the
//       backward solve all walk rows.
//   dinv k: 1 / L_jj.
//   xs  k x dchunk: neighbour coordinates, dchunk dims at a time (coalesced
//       row gathers from X).
//   B   k x m right-hand sides -> solution;  s  k int32 neighbour indices.
// Squared distances are accumulated over dims in ascending order in A's
// strict lower triangle, then replaced by kernel values; the diagonal is
// sigma^2 (1 + tau^2) plus the jitter rung. A failed factorisation rebuilds K
// with the next rung of {0, 1e-10, 1e-8, 1e-6} (linalg.cpp:13-19), so no copy
// of K is kept (retries are rare).
//
// Column j of the factor: lane l owns rows i = j + l + 32c (c < R, only the
// warp-uniformly live c are executed) and accumulates
// a_ij - sum_p L_ip L_jp two p at a time from 128-bit loads (the pivot row
// L_j. is a broadcast).
#include <cfloat>
#include <cstdlib>
#include <string>

#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

__constant__ double kJitters[4] = {0.0, 1e-10, 1e-8, 1e-6};

// Start of row i in the padded row-major packed triangle.
__host__ __device__ __forceinline__ int ro(int i) { return ((i * (i + 1)) >> 1) + ((i + 1) >> 1); }

__device__ __forceinline__ double jittered(double v, int a) {
  for (int t = 1; t <= a; ++t) v = __dadd_rn(v, __dsub_rn(kJitters[t], kJitters[t - 1]));
  return v;
}

// The augmented matrix [K ; B^T]: rows 0..k-1 are the packed lower triangle
// of K (row i: i+1 entries), rows k..k+m-1 are the right-hand sides b_c^T
// (k entries each), every row padded to an even length so rows start 16-byte
// aligned. The left-looking column sweep over rows j..k+m-1 factors K and, on
// the RHS rows, performs the forward substitution y = L^-1 b in the same pass.
struct Aug {
  int k, m, rw;  // rw: padded RHS row length
  __device__ __forceinline__ int row(int i) const { return i < k ? ro(i) : ro(k) + (i - k) * rw; }
};

// Factor in place; false at the first pivot <= 0 (Eigen LLT semantics, NaN
// fails too). dinv[j] = 1 / L_jj.
template <int R>
__device__ bool warp_cholesky_aug(double* A, double* dinv, const Aug& G, int lane) {
  const int rows = G.k + G.m;
  for (int j = 0; j < G.k; ++j) {
    const int live = (rows - j + 31) >> 5;  // warp-uniform number of live row slots
    const double* Lj = A + ro(j);
    // four partial sums per row (p mod 4): ILP and a shallower summation tree
    double acc0[R], acc1[R], acc2[R], acc3[R];
    const double* Li[R];
#pragma unroll
    for (int c = 0; c < R; ++c) {
      acc0[c] = acc1[c] = acc2[c] = acc3[c] = 0.0;
      Li[c] = A;
      if (c < live) {
        const int i = min(j + lane + 32 * c, rows - 1);  // lanes past the end redo the last row
        Li[c] = A + G.row(i);
        acc0[c] = Li[c][j];
      }
    }
    int p = 0;
    for (; p + 3 < j; p += 4) {
      const double2 la = *reinterpret_cast<const double2*>(Lj + p);
      const double2 lb = *reinterpret_cast<const double2*>(Lj + p + 2);
#pragma unroll
      for (int c = 0; c < R; ++c) {
        if (c < live) {
          const double2 xa = *reinterpret_cast<const double2*>(Li[c] + p);
          const double2 xb = *reinterpret_cast<const double2*>(Li[c] + p + 2);
          acc0[c] = fma(-xa.x, la.x, acc0[c]);
          acc1[c] = fma(-xa.y, la.y, acc1[c]);
          acc2[c] = fma(-xb.x, lb.x, acc2[c]);
          acc3[c] = fma(-xb.y, lb.y, acc3[c]);
        }
      }
    }
    for (; p < j; ++p) {
      const double l = Lj[p];
#pragma unroll
      for (int c = 0; c < R; ++c)
        if (c < live) acc0[c] = fma(-Li[c][p], l, acc0[c]);
    }
#pragma unroll
    for (int c = 0; c < R; ++c) acc0[c] = (acc0[c] + acc1[c]) + (acc2[c] + acc3[c]);
    const double piv = __shfl_sync(0xffffffffu, acc0[0], 0);  // row j: lane 0, c = 0
    if (!(piv > 0.0)) return false;
    const double ljj = sqrt(piv);
    const double inv = 1.0 / ljj;
    __syncwarp();
#pragma unroll
    for (int c = 0; c < R; ++c) {
      const int i = j + lane + 32 * c;
      if (c < live && i < rows) A[G.row(i) + j] = (i == j) ? ljj : acc0[c] * inv;
    }
    if (lane == 0) dinv[j] = inv;
    __syncwarp();
  }
  return true;
}

// Backward solve L^T x = y for each RHS row (y = the factored RHS rows),
// right-looking over rows of L; x overwrites y.
__device__ void warp_back_solve(double* A, const double* dinv, const Aug& G, int lane) {
  for (int c = 0; c < G.m; ++c) {
    double* y = A + G.row(G.k + c);
    for (int j = G.k - 1; j >= 0; --j) {
      const double* Lj = A + ro(j);
      const double xj = y[j] * dinv[j];
      __syncwarp();
      for (int i = lane; i < j; i += kWarp) y[i] = fma(-Lj[i], xj, y[i]);
      if (lane == 0) y[j] = xj;
      __syncwarp();
    }
  }
}

struct WarpSmem {
  double* A;
  double* dinv;
  double* xs;
  int32_t* sr;
};

__host__ __device__ __forceinline__ size_t per_warp_doubles(int k, int dchunk, int m) {
  const size_t aug = static_cast<size_t>(ro(k)) + static_cast<size_t>(m) * ((k + 1) & ~1);
  const size_t n = aug + k + static_cast<size_t>(k) * (dchunk | 1) + (k + 1) / 2 + 2;
  return (n + 1) & ~static_cast<size_t>(1);  // even: every warp's A stays 16-byte aligned
}

__device__ __forceinline__ WarpSmem carve(double* smem, int warp, int k, int dchunk, int m) {
  WarpSmem w;
  w.A = smem + warp * per_warp_doubles(k, dchunk, m);
  w.dinv = w.A + ro(k) + static_cast<size_t>(m) * ((k + 1) & ~1);
  w.xs = w.dinv + k;
  w.sr = reinterpret_cast<int32_t*>(w.xs + static_cast<size_t>(k) * (dchunk | 1));
  return w;
}

// (i, p) of strict-lower pair number e in row-major order (p < i).
__device__ __forceinline__ void pair_of(int e, int& i, int& p) {
  i = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(e))) * 0.5f);
  while ((i * (i - 1)) / 2 > e) --i;
  while ((i * (i + 1)) / 2 <= e) ++i;
  p = e - (i * (i - 1)) / 2;
}

// [K(S_i) ; Y_{S_i}^T] (cov_matrix_self, kernel.cpp:106-119) with the diagonal
// at jitter rung `attempt`. Coordinates are gathered from X in dchunk-wide
// slices (the whole point when d <= dchunk); the k(k-1)/2 pairs are spread
// over all lanes with an incremental pair decode.
__device__ void build_aug(const double* __restrict__ X, const double* __restrict__ Y, int d, const int32_t* sr,
                          const Aug& G, int dchunk, const KParams& kp, int attempt, double* A, double* xs, int lane) {
  const int k = G.k;
  const int npairs = (k * (k - 1)) / 2;
  for (int c0 = 0; c0 < d; c0 += dchunk) {
    const int dc = min(dchunk, d - c0);
    const int ds = dc | 1;  // odd row stride: lanes reading different rows hit different banks
    for (int e = lane; e < k * dc; e += kWarp) {
      const int t = e / dc, c = e - t * dc;
      xs[t * ds + c] = X[static_cast<int64_t>(sr[t]) * d + c0 + c];
    }
    __syncwarp();
    const bool last = c0 + dc >= d;
    int i, p;
    pair_of(lane, i, p);
    int rowi = ro(i);
    for (int e = lane; e < npairs; e += kWarp) {
      const double* xa = xs + i * ds;
      const double* xb = xs + p * ds;
      double acc = c0 == 0 ? 0.0 : A[rowi + p];
      for (int c = 0; c < dc; ++c) {
        const double diff = __dsub_rn(xa[c], xb[c]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
      }
      A[rowi + p] = last ? kernel_eval_fast(sqrt(acc), kp) : acc;
      p += kWarp;  // advance to pair e + 32
      while (p >= i) {
        p -= i;
        ++i;
      }
      rowi = ro(i);
    }
    __syncwarp();
  }
  const double dg = jittered(kp.diag, attempt);
  for (int i = lane; i < k; i += kWarp) A[ro(i) + i] = dg;
  for (int e = lane; e < k * G.m; e += kWarp) {
    const int t = e / G.m, c = e - t * G.m;
    A[G.row(k + c) + t] = Y[static_cast<int64_t>(sr[t]) * G.m + c];
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
  Aug G;
  G.k = k;
  G.m = m;
  G.rw = (k + 1) & ~1;

  for (int64_t r = static_cast<int64_t>(blockIdx.x) * warps + warp; r < nrows;
       r += static_cast<int64_t>(gridDim.x) * warps) {
    for (int t = lane; t < k; t += kWarp) w.sr[t] = S[r * k + t];
    __syncwarp();
    int used = -1;
    for (int attempt = 0; attempt < 4; ++attempt) {
      build_aug(X, Y, d, w.sr, G, dchunk, kp, attempt, w.A, w.xs, lane);
      if (warp_cholesky_aug<R>(w.A, w.dinv, G, lane)) {
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
    warp_back_solve(w.A, w.dinv, G, lane);
    for (int e = lane; e < k * m; e += kWarp) {
      const int t = e / m, c = e - t * m;
      C[r * k * m + e] = w.A[G.row(k + c) + t];
    }
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
  Aug G;
  G.k = k;
  G.m = m;
  G.rw = (k + 1) & ~1;
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * warps + warp; r < batch;
       r += static_cast<int64_t>(gridDim.x) * warps) {
    const double* Kr = K + r * k * k;
    int used = -1;
    for (int attempt = 0; attempt < 4; ++attempt) {
      for (int i = 0; i < k; ++i)
        for (int p = lane; p <= i; p += kWarp)
          w.A[ro(i) + p] = i == p ? jittered(Kr[static_cast<int64_t>(i) * k + i], attempt)
                                  : Kr[static_cast<int64_t>(i) * k + p];
      for (int e = lane; e < k * m; e += kWarp) {
        const int t = e / m, c = e - t * m;
        w.A[G.row(k + c) + t] = Bin[r * k * m + e];
      }
      __syncwarp();
      if (warp_cholesky_aug<R>(w.A, w.dinv, G, lane)) {
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
    warp_back_solve(w.A, w.dinv, G, lane);
    for (int e = lane; e < k * m; e += kWarp) {
      const int t = e / m, c = e - t * m;
      Xout[r * k * m + e] = w.A[G.row(k + c) + t];
    }
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

constexpr int64_t kOrderMinRows = 1 << 16;  // below this the batch is L2-resident anyway

cudaError_t fused_solve(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                        int64_t row_begin, int k, const KParams& kp, double* C, int32_t* status,
                        unsigned long long* fail_min, int num_sms, cudaStream_t stream) {
  if (nrows <= 0) return cudaSuccess;
  // FMGP_SOLVE = reg/cta (default where the shape is compiled in) | tc | scalar, for A/B checks.
  static const int mode = [] {
    const char* e = std::getenv("FMGP_SOLVE");
    if (e == nullptr) return 0;
    const std::string v(e);
    return v == "tc" ? 1 : (v == "scalar" ? 2 : 0);
  }();
  if (mode == 0 && status == nullptr &&
      (fused_solve_dm_supported(k, d, m, kp) || fused_solve_2d_supported(k, d, m, kp) ||
       fused_solve_reg_supported(k, d, m))) {
    // Large low-d batches are solved in a cell order of their rows (FMGP_SOLVE_ORDER=0: index order):
    // warps in flight then gather overlapping neighbourhoods, so X stays in L2.
    static const bool use_order = [] {
      const char* e = std::getenv("FMGP_SOLVE_ORDER");
      return !(e != nullptr && e[0] == '0');
    }();
    int32_t* order = nullptr;
    if (use_order && d <= 3 && nrows >= kOrderMinRows) {
      cudaError_t e = cudaMallocAsync(&order, sizeof(int32_t) * nrows, stream);
      if (e != cudaSuccess) return e;
      e = spatial_row_order(X + row_begin * d, nrows, d, order, stream);
      if (e != cudaSuccess) {
        cudaFreeAsync(order, stream);
        return e;
      }
    }
    // default: the DMMA-blocked solve where its shape is compiled in; FMGP_SOLVE_2D=1 / FMGP_SOLVE_DM=0
    // select the 2-D cyclic / row-per-lane register solves (A/B and the parity tests of all three)
    const cudaError_t e =
        fused_solve_2d_supported(k, d, m, kp)
            ? fused_solve_2d(X, Y, d, S, nrows, row_begin, k, kp, C, fail_min, num_sms, stream, order)
            : (fused_solve_dm_supported(k, d, m, kp)
                   ? fused_solve_dm(X, Y, d, S, nrows, row_begin, k, kp, C, fail_min, num_sms, stream, order)
                   : fused_solve_reg(X, Y, d, m, S, nrows, row_begin, k, kp, C, fail_min, num_sms, stream, order));
    if (order != nullptr) cudaFreeAsync(order, stream);
    return e;
  }
  if (mode == 0 && status == nullptr && fused_solve_cta_supported(k, d, m))
    return fused_solve_cta(X, Y, d, m, S, nrows, row_begin, k, kp, C, fail_min, num_sms, stream);
  if (mode == 1 && status == nullptr && fused_solve_tc_supported(k, d, m))
    return fused_solve_tc(X, Y, d, m, S, nrows, row_begin, k, kp, C, fail_min, num_sms, stream);
  const size_t bytes = per_warp_doubles(k, dchunk_for(k, d), m) * sizeof(double);
  if (k + m > kMaxK || bytes > kSmemBudget)
    return fused_solve_big(X, Y, d, m, S, nrows, row_begin, k, kp, C, fail_min, num_sms, stream);
  switch ((k + m + 31) / 32) {
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
  if (k + m > kMaxK || bytes > kSmemBudget) return spd_solve_big(K, B, batch, k, m, X, jit_out, fail_min, num_sms, stream);
  switch ((k + m + 31) / 32) {
    case 1: return launch_spd<1>(K, B, batch, k, m, X, jit_out, fail_min, num_sms, stream);
    case 2: return launch_spd<2>(K, B, batch, k, m, X, jit_out, fail_min, num_sms, stream);
    case 3: return launch_spd<3>(K, B, batch, k, m, X, jit_out, fail_min, num_sms, stream);
    case 4: return launch_spd<4>(K, B, batch, k, m, X, jit_out, fail_min, num_sms, stream);
    default: return launch_spd<5>(K, B, batch, k, m, X, jit_out, fail_min, num_sms, stream);
  }
}

}  // namespace fmgp
