// K2-2d — the fused neighbourhood solve for the small-d BASELINE shapes
// (d in {2, 3}, k in {30, 50}, one output column: cfg1, cfg2, cfg5), one warp
// per neighbourhood, with the augmented matrix [K(S_i) ; y^T] distributed
// over the warp in a 2-D cyclic layout and factored right-looking.
// Same contract as solve.cu / solve_reg.cu (fast_predict.cpp:98-106,
// kernel.cpp:106-119, linalg.cpp:10-36).
//
// Why (profiles/r02/ncu_solve_reg_cfg5.txt): the row-per-lane left-looking
// kernel (solve_reg.cu) keeps the FP64 pipe ~40% busy; it stalls on
// shared-memory latency (each pivot-row double it broadcasts feeds one or two
// FMAs per lane, ~2.9 k wavefronts per row) and executes every column's dot
// product on all 32 lanes although only the rows below the column are live
// (~50% of its FMA slots are idle lanes).
//
// Layout: lane = a + 4 b (a = lane & 3, b = lane >> 2). The lane owns the
// entries (i, k) with i = 4 ii + a, k = 8 kk + b of the R = k + 1 row
// augmented matrix (row k is y^T), i >= k, as registers L[ii][kk] (only the
// (ii, kk) slots that hold a lower-triangle entry for some lane exist: 49 for
// k = 50). Every lane's share of the trailing matrix shrinks at the same rate,
// so the rank-1 updates keep ~all lanes busy (1041 FMA instructions per row
// for k = 50 against ~1400 with one row per lane).
//
// Step j (unrolled, j compile-time): the owner of (j, j) supplies the pivot by
// a shuffle (Eigen LLT semantics: a pivot <= 0 fails the rung); column j's
// raw entries c_ij (stored to shared memory by their owners one step ahead)
// are read back, rows scaled by 1/c_jj, and every lane applies
// a_ik -= (c_ij / c_jj) c_kj to its slots. The slots of column j + 1 are
// updated first and stored at once, so the next step's pivot and column
// loads overlap the rest of the update. The raw columns stay in shared memory
// (class-major: column j, class a, slot ii), which is L scaled by sqrt(c_jj)
// per column: the RHS row gives z (forward substitution) and the backward
// solve x_j = (c_yj - sum_{i>j} c_ij x_i) / c_jj runs over them.
//
// Build: each lane evaluates its own slots (kernel_from_sq_build, the kernel
// kind a template parameter) from the neighbourhood's coordinates staged in
// shared memory; no pair table, no matrix staging. The jitter ladder
// (cumulative rungs 0, 1e-10, 1e-8, 1e-6 on the diagonal) rebuilds the slots.
#include <climits>
#include <cstdlib>

#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

__constant__ double kJit2[4] = {0.0, 1e-10, 1e-8, 1e-6};

__device__ __forceinline__ double jitter_2d(double v, int a) {
  for (int t = 1; t <= a; ++t) v = __dadd_rn(v, __dsub_rn(kJit2[t], kJit2[t - 1]));
  return v;
}

template <int K>
struct G2 {
  static constexpr int R = K + 1;          // augmented rows (y^T last)
  static constexpr int NI = (R + 3) / 4;   // row slots (class a)
  static constexpr int NK = (K + 7) / 8;   // column slots (class b)
  // column j is stored for slots ii >= st(j) of every class (rows i >= j + 1
  // need no more), len(j) doubles per class (even: 16-byte pairs stay aligned)
  __host__ __device__ static constexpr int st(int j) { return (j + 1) / 4; }
  __host__ __device__ static constexpr int len(int j) { return (NI - st(j) + 1) & ~1; }
  __host__ __device__ static constexpr int col_off(int j) {
    int o = 0;
    for (int q = 0; q < j; ++q) o += 4 * len(q);
    return o;
  }
  __host__ __device__ static constexpr int kk0(int j) { return (j + 1) / 8; }
  __host__ __device__ static constexpr bool has(int ii, int kk) {
    return 4 * ii + 3 >= 8 * kk && 4 * ii < R && 8 * kk < K;
  }
  static constexpr int kCols = col_off(K);
  static constexpr int kStage = 4 * K + K;  // coordinates (4 per point) + y, overlaid on the columns
  static constexpr int kArea = ((kCols > kStage ? kCols : kStage) + 1) & ~1;
  static constexpr int kPerWarp = kArea + ((K + 1) & ~1) /*1/sqrt(pivot)*/ + ((K + 3) / 4) * 2 /*S row*/;
};

template <int K, int D>
__device__ __forceinline__ void stage_nbhd(const double* __restrict__ X, const double* __restrict__ Y,
                                           const int32_t* sr, double* xs, double* ys, int lane) {
  for (int t = lane; t < K; t += kWarp) {
    const int64_t s = sr[t];
#pragma unroll
    for (int c = 0; c < D; ++c) xs[t * 4 + c] = X[s * D + c];
    ys[t] = Y[s];
  }
}

template <int K, int D>
__device__ __forceinline__ void load_pt(const double* xs, int t, double (&x)[D]) {
  const double2 v = *reinterpret_cast<const double2*>(xs + t * 4);
  x[0] = v.x;
  if constexpr (D >= 2) x[1] = v.y;
  if constexpr (D >= 3) x[2] = xs[t * 4 + 2];
}

#ifndef FMGP_S2D_MINB
#define FMGP_S2D_MINB 3
#endif
template <int K, int D, int KF>
__global__ void __launch_bounds__(128, (K > 32 ? FMGP_S2D_MINB : 4))
solve2d_kernel(const double* __restrict__ X, const double* __restrict__ Y, const int32_t* __restrict__ S,
               int64_t nrows, int64_t row_begin, KParams kp, double* __restrict__ C,
               unsigned long long* __restrict__ fail_min, const int32_t* __restrict__ order) {
  using G = G2<K>;
  constexpr int NI = G::NI, NK = G::NK;
  extern __shared__ double smem[];
  const int lane = threadIdx.x & (kWarp - 1);
  const int warp = threadIdx.x / kWarp;
  const int warps = blockDim.x / kWarp;
  double* area = smem + warp * G::kPerWarp;
  double* dinv = area + G::kArea;
  int32_t* sr = reinterpret_cast<int32_t*>(dinv + ((K + 1) & ~1));
  double* xs = area;
  double* ys = area + 4 * K;
  const int a = lane & 3, b = lane >> 2;
  const double cs = kernel_scale_build<KF>(kp);
  __shared__ double s_exp[FMGP_BUILD_TAB_N];
  stage_exp_table(s_exp);
  __syncthreads();

  // backward-solve geometry of the lane's two x entries (j0 = lane, j1 = lane + 32)
  const int j0 = lane, j1 = lane + kWarp;
  int off0 = 0, off1 = 0;
  for (int q = 0; q < j1 && q < K; ++q) {
    if (q < j0) off0 += 4 * G::len(q);
    off1 += 4 * G::len(q);
  }
  const int st0 = G::st(j0), ln0 = G::len(j0), st1 = G::st(j1), ln1 = G::len(j1);

  for (int64_t base = static_cast<int64_t>(blockIdx.x) * warps; base < nrows;
       base += static_cast<int64_t>(gridDim.x) * warps) {
    __syncthreads();  // the CTA's warps start every row together (instruction-cache locality, as solve_reg)
    const int64_t it = base + warp;
    if (it >= nrows) continue;
    const int64_t r = order != nullptr ? order[it] : it;
    for (int t = lane; t < K; t += kWarp) sr[t] = S[r * K + t];
    __syncwarp();
    bool ok = false;
    for (int attempt = 0; attempt < 4 && !ok; ++attempt) {
      stage_nbhd<K, D>(X, Y, sr, xs, ys, lane);  // (re)staged: the columns overwrite it
      __syncwarp();
      const double dg = jitter_2d(kp.diag, attempt);
      double L[NI][NK];
      // ---- build: lane's slots of [K(S_i) ; y^T]
#pragma unroll
      for (int kk = 0; kk < NK; ++kk) {
        const int k = 8 * kk + b;
        const int kc = k < K ? k : K - 1;
        double xk[D];
        load_pt<K, D>(xs, kc, xk);
        const double yk = ys[kc];
#pragma unroll
        for (int ii = 0; ii < NI; ++ii) {
          if (!G::has(ii, kk)) continue;
          const int i = 4 * ii + a;
          const int ic = i < K ? i : K - 1;
          double xi[D];
          load_pt<K, D>(xs, ic, xi);
          const double d0 = xi[0] - xk[0];
          double acc = d0 * d0;
#pragma unroll
          for (int c = 1; c < D; ++c) {
            const double dd = xi[c] - xk[c];
            acc = fma(dd, dd, acc);
          }
          double v = kernel_from_sq_build<KF>(acc, cs, kp, s_exp);
          v = i == k ? dg : v;
          v = i == K ? yk : v;
          L[ii][kk] = v;
        }
      }
      __syncwarp();  // every lane has read the staged coordinates
      // column 0 (final as built) -> shared memory, by its owners (b == 0)
      if (b == 0) {
        double* dst = area + G::col_off(0) + a * G::len(0) - G::st(0);
#pragma unroll
        for (int ii = G::st(0); ii < NI; ii += 2)
          *reinterpret_cast<double2*>(dst + ii) = make_double2(L[ii][0], ii + 1 < NI ? L[ii + 1][0] : 0.0);
      }
      __syncwarp();
      // pivot of column 0; every later pivot is taken one step ahead (right
      // after its column's slots are updated), so its shuffle + rsqrt chain
      // overlaps the rest of the current step's update
      double piv = __shfl_sync(0xffffffffu, L[0][0], 0);
      bool bad = !(piv > 0.0);
      double inv = rsqrt_pivot(piv);
      if (lane == 0) dinv[0] = inv;
#pragma unroll
      for (int j = 0; j + 1 < K; ++j) {
        const double inv2 = inv * inv;
        const int stj = G::st(j), lnj = G::len(j);
        const double* col = area + G::col_off(j) - stj;
        // row values c_ij (class a)
        double rv[NI];
        {
          const double* src = col + a * lnj;
#pragma unroll
          for (int ii = stj; ii < NI; ii += 2) {
            const double2 v = *reinterpret_cast<const double2*>(src + ii);
            rv[ii] = v.x;
            if (ii + 1 < NI) rv[ii + 1] = v.y;
          }
        }
        // column values c_kj / c_jj, k = 8 kk + b (class k & 3, slot k >> 2)
        double cv[NK];
#pragma unroll
        for (int kk = G::kk0(j); kk < NK; ++kk) {
          const int kmax = K - 1 - 8 * kk;  // absent columns read an in-range entry (never used)
          const int be = (8 * kk + 7 < K) ? b : min(b, kmax);
          cv[kk] = col[(be & 3) * lnj + 2 * kk + (be >> 2)] * inv2;
        }
        // slots of column j + 1 first: its pivot, then its owners store it for the next step
        const int kk1 = (j + 1) / 8;
#pragma unroll
        for (int ii = stj; ii < NI; ++ii)
          if (G::has(ii, kk1)) L[ii][kk1] = fma(-rv[ii], cv[kk1], L[ii][kk1]);
        const int owner = ((j + 1) & 3) | (((j + 1) & 7) << 2);
        piv = __shfl_sync(0xffffffffu, L[(j + 1) / 4][kk1], owner);
        bad |= !(piv > 0.0);
        const double inv_next = rsqrt_pivot(piv);
        if (lane == 0) dinv[j + 1] = inv_next;
        if (b == ((j + 1) & 7)) {
          const int stn = G::st(j + 1);
          double* dst = area + G::col_off(j + 1) + a * G::len(j + 1) - stn;
#pragma unroll
          for (int ii = stn; ii < NI; ii += 2)
            *reinterpret_cast<double2*>(dst + ii) = make_double2(L[ii][kk1], ii + 1 < NI ? L[ii + 1][kk1] : 0.0);
        }
        __syncwarp();
#pragma unroll
        for (int kk = G::kk0(j); kk < NK; ++kk) {
          if (kk == kk1) continue;
#pragma unroll
          for (int ii = stj; ii < NI; ++ii)
            if (G::has(ii, kk)) L[ii][kk] = fma(-rv[ii], cv[kk], L[ii][kk]);
        }
        inv = inv_next;
      }
      ok = !bad;  // uniform: the pivots are broadcast
      __syncwarp();
    }
    if (!ok) {
      if (lane == 0) atomicMin(fail_min, static_cast<unsigned long long>(row_begin + r));
      __syncwarp();
      continue;
    }
    // ---- backward solve: x_j = (c_yj - sum_{i>j} c_ij x_i) / c_jj over the stored columns
    const double* c0 = area + off0 - st0;
    const double* c1 = area + off1 - st1;
    double x0 = j0 < K ? c0[2 * ln0 + (K >> 2)] : 0.0;  // row K = y^T: class K & 3, slot K >> 2
    double x1 = j1 < K ? c1[2 * ln1 + (K >> 2)] : 0.0;
    static_assert((K & 3) == 2, "y^T row in class 2");
#pragma unroll
    for (int i = K - 1; i >= 0; --i) {
      const double s = __shfl_sync(0xffffffffu, i < kWarp ? x0 : x1, i & (kWarp - 1));
      const double iv = dinv[i];
      const double xi = s * (iv * iv);
      const int ci = (i & 3), si = (i >> 2);
      if (i < kWarp) {
        if (lane == i) x0 = xi;
        if (lane < i) x0 = fma(-c0[ci * ln0 + si], xi, x0);
      } else {
        if (lane == i - kWarp) x1 = xi;
        x0 = fma(-c0[ci * ln0 + si], xi, x0);
        if (j1 < i) x1 = fma(-c1[ci * ln1 + si], xi, x1);
      }
    }
    double* Crow = C + r * K;
    if (j0 < K) Crow[j0] = x0;
    if (j1 < K) Crow[j1] = x1;
    __syncwarp();
  }
}

template <int K, int D, int KF>
cudaError_t launch_2d(const double* X, const double* Y, const int32_t* S, int64_t nrows, int64_t row_begin,
                      const KParams& kp, double* C, unsigned long long* fail_min, int num_sms, cudaStream_t stream,
                      const int32_t* order) {
  using G = G2<K>;
  constexpr int kWarps = 4;
  const size_t smem = sizeof(double) * G::kPerWarp * kWarps;
  cudaError_t err = cudaFuncSetAttribute(solve2d_kernel<K, D, KF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  int per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve2d_kernel<K, D, KF>, kWarps * kWarp, smem);
  if (err != cudaSuccess) return err;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (nrows + kWarps - 1) / kWarps;
  const int64_t grid = std::min<int64_t>(need, static_cast<int64_t>(num_sms) * per_sm);
  solve2d_kernel<K, D, KF><<<static_cast<unsigned>(grid), kWarps * kWarp, smem, stream>>>(X, Y, S, nrows, row_begin,
                                                                                        kp, C, fail_min, order);
  note_launches(1);
  return cudaGetLastError();
}

template <int K, int D>
cudaError_t launch_2d_kind(const double* X, const double* Y, const int32_t* S, int64_t nrows, int64_t row_begin,
                           const KParams& kp, double* C, unsigned long long* fail_min, int num_sms,
                           cudaStream_t stream, const int32_t* order) {
  switch (kp.kind == 1 ? 0 : 1 + kp.nu_code) {  // kernel_code(), on the host
    case 0: return launch_2d<K, D, 0>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order);
    case 1: return launch_2d<K, D, 1>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order);
    case 2: return launch_2d<K, D, 2>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order);
    default: return launch_2d<K, D, 3>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order);
  }
}

}  // namespace

bool fused_solve_2d_supported(int k, int d, int m, const KParams& kp) {
  // FMGP_SOLVE_2D=1 selects it (A/B against the other fused solves; read per call)
  const char* e = std::getenv("FMGP_SOLVE_2D");
  const bool on = e != nullptr && e[0] == '1';
  return on && m == 1 && (d == 2 || d == 3) && (k == 50 || k == 30) && (kp.kind == 1 || kp.nu_code <= 2);
}

cudaError_t fused_solve_2d(const double* X, const double* Y, int d, const int32_t* S, int64_t nrows,
                           int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                           int num_sms, cudaStream_t stream, const int32_t* order) {
  if (nrows <= 0) return cudaSuccess;
  if (k == 50) {
    return d == 2 ? launch_2d_kind<50, 2>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order)
                  : launch_2d_kind<50, 3>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order);
  }
  return d == 2 ? launch_2d_kind<30, 2>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order)
                : launch_2d_kind<30, 3>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order);
}

}  // namespace fmgp
