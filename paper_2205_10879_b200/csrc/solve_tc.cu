// K2-tc — the fused neighbourhood solve on the FP64 tensor cores (DMMA,
// mma.sync.m8n8k4.f64), one warp per neighbourhood. Same contract as the
// scalar kernel in solve.cu (gather -> cov_matrix_self -> jitter-Cholesky ->
// solve; fast_predict.cpp:98-106, kernel.cpp:106-119, linalg.cpp:10-36).
//
// Blocked left-looking Cholesky with 8x8 tiles. The matrix is padded to
// KP = 8*NB with an identity block, and the m right-hand sides are appended
// as MB = ceil(m/8) extra block rows below it (row KP + c holds b_c^T), so
// the factorisation of the augmented panel computes y = L^-1 b as well: the
// forward substitution is folded into the tile sweep.
//
// Storage ("fragment order", per warp, doubles): for block row I and column
// quad Q (columns 4Q..4Q+3) a 32-entry chunk where lane (g = lane/4,
// t = lane%4) holds element (8I + g, 4Q + t). That is exactly the DMMA A
// fragment of rows 8I.. and the B fragment of (rows 8J..)^T, so every
// operand load is one conflict-free 64-bit LDS per lane.
//   block row I < NB : quads 0 .. 2I+1 (the lower triangle incl. diagonal tile)
//   block row NB + r : quads 0 .. 2NB-1 (right-hand-side rows)
// Per block column J:
//   1. C(I, J) = K(I, J) - sum_{Q < 2J} A(I, Q) B(J, Q)  for all I >= J (DMMA),
//      written to an 8x8 row-major scratch tile;
//   2. the diagonal tile is factored (scalar, 8 steps) -> L_JJ, 1/diag;
//   3. every row below (incl. the RHS rows) solves x L_JJ^T = c (a lane per row).
// Then the backward solve L^T x = y runs over rows (right-looking).
#include <cfloat>

#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

__constant__ double kJit[4] = {0.0, 1e-10, 1e-8, 1e-6};

__device__ __forceinline__ double jittered_tc(double v, int a) {
  for (int t = 1; t <= a; ++t) v = __dadd_rn(v, __dsub_rn(kJit[t], kJit[t - 1]));
  return v;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct TcLayout {
  int k, m, nb, mb, kp;
  // chunk index of (block row I, quad Q)
  __device__ __forceinline__ int chunk(int I, int Q) const {
    return I < nb ? I * (I + 1) + Q : nb * (nb + 1) + (I - nb) * 2 * nb + Q;
  }
  // storage offset of element (row r, column c), c <= row's last column
  __device__ __forceinline__ int at(int r, int c) const { return chunk(r >> 3, c >> 2) * 32 + ((r & 7) << 2) + (c & 3); }
  __device__ __forceinline__ int nchunks() const { return nb * (nb + 1) + mb * 2 * nb; }
};

__host__ __device__ __forceinline__ size_t tc_per_warp_doubles(int k, int m, int dchunk) {
  const int nb = (k + 7) / 8, mb = (m + 7) / 8;
  const size_t store = static_cast<size_t>(nb * (nb + 1) + mb * 2 * nb) * 32;
  const size_t scratch = static_cast<size_t>(nb + mb) * 64;
  const size_t n = store + scratch + static_cast<size_t>(nb) * 8 /* dinv */ + static_cast<size_t>(k) * dchunk +
                   (k + 1) / 2 + 2;
  return (n + 1) & ~static_cast<size_t>(1);
}

// Element (i, p) of the augmented matrix for rows i < KP (kernel part).
// Writes K into fragment-order storage: strict lower = kernel values, diagonal
// = sigma^2(1+tau^2) + jitter, padding rows/cols = identity.
__device__ void tc_build(const TcLayout& L, const double* __restrict__ X, const double* __restrict__ Y, int d,
                         const int32_t* sr, int dchunk, const KParams& kp, int attempt, double* S, double* xs,
                         int lane) {
  const int k = L.k;
  // distances (pairs spread over lanes, dims in ascending order per pair)
  const int npairs = (k * (k - 1)) / 2;
  for (int c0 = 0; c0 < d; c0 += dchunk) {
    const int dc = min(dchunk, d - c0);
    for (int e = lane; e < k * dc; e += kWarp) {
      const int t = e / dc, c = e - t * dc;
      xs[t * dc + c] = X[static_cast<int64_t>(sr[t]) * d + c0 + c];
    }
    __syncwarp();
    const bool last = c0 + dc >= d;
    for (int e = lane; e < npairs; e += kWarp) {
      int i = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(e))) * 0.5f);
      while ((i * (i - 1)) / 2 > e) --i;
      while ((i * (i + 1)) / 2 <= e) ++i;
      const int p = e - (i * (i - 1)) / 2;
      const double* xa = xs + i * dc;
      const double* xb = xs + p * dc;
      const int off = L.at(i, p);
      double acc = c0 == 0 ? 0.0 : S[off];
      for (int c = 0; c < dc; ++c) {
        const double diff = __dsub_rn(xa[c], xb[c]);
        acc = __dadd_rn(acc, __dmul_rn(diff, diff));
      }
      S[off] = last ? kernel_eval_fast(sqrt(acc), kp) : acc;
    }
    __syncwarp();
  }
  const double dg = jittered_tc(kp.diag, attempt);
  for (int i = lane; i < L.kp; i += kWarp) S[L.at(i, i)] = i < k ? dg : 1.0;
  // padding rows i in [k, KP): zero below the diagonal
  for (int e = lane; e < (L.kp - k) * L.kp; e += kWarp) {
    const int i = k + e / L.kp, p = e % L.kp;
    if (p < i) S[L.at(i, p)] = 0.0;
  }
  // right-hand-side rows: row KP + c = b_c^T (zero beyond k)
  for (int e = lane; e < L.mb * 8 * L.kp; e += kWarp) {
    const int c = e / L.kp, j = e % L.kp;
    S[L.at(L.kp + c, j)] = (c < L.m && j < k) ? Y[static_cast<int64_t>(sr[j]) * L.m + c] : 0.0;
  }
  __syncwarp();
}

// Blocked left-looking factorisation of the augmented matrix. Returns false
// at the first pivot <= 0 (Eigen LLT semantics).
template <int NBM>
__device__ bool tc_factor(const TcLayout& L, double* S, double* T, double* dinv, int lane) {
  const int g = lane >> 2, t = lane & 3;
  const int nbt = L.nb + L.mb;
  for (int J = 0; J < L.nb; ++J) {
    // 1. C(I, J) for I = J .. nbt-1, accumulated over the quads left of J
    double acc[NBM + 2][2];
#pragma unroll
    for (int u = 0; u < NBM + 2; ++u) {
      const int I = J + u;
      acc[u][0] = acc[u][1] = 0.0;
      if (I < nbt) {
        // K(I, J) entries (g, 2t), (g, 2t+1): quad 2J + t/2, slots 4g + 2(t&1) (+1)
        const double2 kv =
            *reinterpret_cast<const double2*>(S + L.chunk(I, 2 * J + (t >> 1)) * 32 + 4 * g + 2 * (t & 1));
        acc[u][0] = kv.x;
        acc[u][1] = kv.y;
      }
    }
    for (int Q = 0; Q < 2 * J; ++Q) {
      const double b = -S[L.chunk(J, Q) * 32 + lane];
#pragma unroll
      for (int u = 0; u < NBM + 2; ++u) {
        const int I = J + u;
        if (I < nbt) dmma(acc[u][0], acc[u][1], S[L.chunk(I, Q) * 32 + lane], b);
      }
    }
#pragma unroll
    for (int u = 0; u < NBM + 2; ++u) {
      if (J + u < nbt) *reinterpret_cast<double2*>(T + u * 64 + 8 * g + 2 * t) = make_double2(acc[u][0], acc[u][1]);
    }
    __syncwarp();
    // 2. factor the diagonal tile T[0] (8 x 8 row-major), scalar right-looking
    for (int s = 0; s < 8; ++s) {
      const double piv = T[s * 8 + s];
      if (!(piv > 0.0)) return false;
      const double ljj = sqrt(piv);
      const double inv = 1.0 / ljj;
      __syncwarp();
      if (lane > s && lane < 8) T[lane * 8 + s] *= inv;
      if (lane == 0) {
        T[s * 8 + s] = ljj;
        dinv[8 * J + s] = inv;
      }
      __syncwarp();
      // trailing 8x8 update: pairs (r, c) with s < c <= r
      const int r = s + 1 + (lane >> 3), c = s + 1 + (lane & 7);
      if (r < 8 && c <= r) T[r * 8 + c] = fma(-T[r * 8 + s], T[c * 8 + s], T[r * 8 + c]);
      if (lane < 24) {
        const int r2 = r + 4;
        if (r2 < 8 && c <= r2) T[r2 * 8 + c] = fma(-T[r2 * 8 + s], T[c * 8 + s], T[r2 * 8 + c]);
      }
      __syncwarp();
    }
    // store L_JJ (lower part) back into fragment order
    for (int e = lane; e < 64; e += kWarp) {
      const int r = e >> 3, c = e & 7;
      if (c <= r) S[L.at(8 * J + r, 8 * J + c)] = T[e];
    }
    // 3. rows below: x L_JJ^T = c  (a lane per row)
    const int rows_below = (nbt - J - 1) * 8;
    for (int rr = lane; rr < rows_below; rr += kWarp) {
      const double* c = T + 64 + rr * 8;  // scratch tiles u >= 1 are contiguous rows
      double x[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        double v = c[s];
#pragma unroll
        for (int q = 0; q < s; ++q) v = fma(-x[q], T[s * 8 + q], v);
        x[s] = v * dinv[8 * J + s];
      }
      const int row = 8 * (J + 1) + rr;
#pragma unroll
      for (int s = 0; s < 8; ++s) S[L.at(row, 8 * J + s)] = x[s];
    }
    __syncwarp();
  }
  return true;
}

template <int NBM>
__global__ void __launch_bounds__(128)
solve_tc_kernel(const double* __restrict__ X, const double* __restrict__ Y, int d, int m,
                const int32_t* __restrict__ Sidx, int64_t nrows, int64_t row_begin, int k, int dchunk, KParams kp,
                double* __restrict__ C, unsigned long long* __restrict__ fail_min) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x % kWarp;
  const int warp = threadIdx.x / kWarp;
  const int warps = blockDim.x / kWarp;
  TcLayout L;
  L.k = k;
  L.m = m;
  L.nb = (k + 7) / 8;
  L.mb = (m + 7) / 8;
  L.kp = 8 * L.nb;
  double* S = smem + warp * tc_per_warp_doubles(k, m, dchunk);
  double* T = S + L.nchunks() * 32;
  double* dinv = T + (L.nb + L.mb) * 64;
  double* xs = dinv + L.nb * 8;
  int32_t* sr = reinterpret_cast<int32_t*>(xs + static_cast<size_t>(k) * dchunk);

  for (int64_t r = static_cast<int64_t>(blockIdx.x) * warps + warp; r < nrows;
       r += static_cast<int64_t>(gridDim.x) * warps) {
    for (int t = lane; t < k; t += kWarp) sr[t] = Sidx[r * k + t];
    __syncwarp();
    bool ok = false;
    for (int attempt = 0; attempt < 4 && !ok; ++attempt) {
      tc_build(L, X, Y, d, sr, dchunk, kp, attempt, S, xs, lane);
      ok = tc_factor<NBM>(L, S, T, dinv, lane);
      __syncwarp();
    }
    if (!ok) {
      if (lane == 0) atomicMin(fail_min, static_cast<unsigned long long>(row_begin + r));
      __syncwarp();
      continue;
    }
    // backward solve L^T x = y, right-looking over rows; y_c lives in row KP + c
    for (int c = 0; c < m; ++c) {
      const int yrow = L.kp + c;
      for (int j = k - 1; j >= 0; --j) {
        const double xj = S[L.at(yrow, j)] * dinv[j];
        __syncwarp();
        for (int i = lane; i < j; i += kWarp) {
          const int o = L.at(yrow, i);
          S[o] = fma(-S[L.at(j, i)], xj, S[o]);
        }
        if (lane == 0) S[L.at(yrow, j)] = xj;
        __syncwarp();
      }
    }
    for (int e = lane; e < k * m; e += kWarp) {
      const int t = e / m, c = e - t * m;
      C[r * k * m + e] = S[L.at(L.kp + c, t)];
    }
    __syncwarp();
  }
}

template <int NBM>
cudaError_t launch_tc(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                      int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                      int num_sms, cudaStream_t stream, int dchunk) {
  const size_t per_warp = tc_per_warp_doubles(k, m, dchunk) * sizeof(double);
  const int warps = static_cast<int>(std::min<size_t>(4, (220 * 1024) / per_warp));
  if (warps < 1) return cudaErrorInvalidValue;
  const size_t smem = per_warp * warps;
  cudaError_t err =
      cudaFuncSetAttribute(solve_tc_kernel<NBM>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  int per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_tc_kernel<NBM>, warps * kWarp, smem);
  if (err != cudaSuccess) return err;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (nrows + warps - 1) / warps;
  const int64_t grid = std::min<int64_t>(need, static_cast<int64_t>(num_sms) * per_sm);
  solve_tc_kernel<NBM><<<static_cast<unsigned>(grid), warps * kWarp, smem, stream>>>(X, Y, d, m, S, nrows, row_begin,
                                                                                   k, dchunk, kp, C, fail_min);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace

bool fused_solve_tc_supported(int k, int d, int m) {
  (void)d;
  return k >= 2 && k <= 128 && m >= 1 && m <= 16;
}

cudaError_t fused_solve_tc(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                           int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                           int num_sms, cudaStream_t stream) {
  if (nrows <= 0) return cudaSuccess;
  int dchunk = 512 / k;
  if (dchunk < 1) dchunk = 1;
  if (dchunk > d) dchunk = d;
  const int nb = (k + 7) / 8;
  if (nb <= 4) return launch_tc<4>(X, Y, d, m, S, nrows, row_begin, k, kp, C, fail_min, num_sms, stream, dchunk);
  if (nb <= 8) return launch_tc<8>(X, Y, d, m, S, nrows, row_begin, k, kp, C, fail_min, num_sms, stream, dchunk);
  return launch_tc<16>(X, Y, d, m, S, nrows, row_begin, k, kp, C, fail_min, num_sms, stream, dchunk);
}

}  // namespace fmgp
