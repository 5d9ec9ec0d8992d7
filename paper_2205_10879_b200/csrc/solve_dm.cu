// K2-dm — the fused neighbourhood solve with the O(k^3) part of the Cholesky
// on the FP64 tensor cores (DMMA m8n8k4), for the small-d BASELINE shapes
// (k in {30, 50}, m = 1, d in {2, 3}, closed-form kernels). Same contract as
// solve.cu / solve_reg.cu: gather -> cov_matrix_self (kernel.cpp:106-119) ->
// jitter-ladder Cholesky (linalg.cpp:10-31) -> solve (linalg.cpp:33-36) ->
// C_i (fast_predict.cpp:98-106). One warp per neighbourhood.
//
// Why: the row-per-lane register solve is bound by the shared-memory data
// pipe (profiles/r02/ncu_solve_cfg5_full.txt: ~2.9 k wavefronts per row, 1.2 k
// of them the pivot-row broadcast of the left-looking column sweep, L1 at
// 77-84%). Here the k^3/6 multiply-adds run as DMMA on register fragments,
// which need no broadcast at all; shared memory only carries the panels.
//
// Augmented matrix [K ; y^T] (R = k + 1 rows, row k = the RHS, so the
// factorisation also performs the forward substitution), blocked 8 x 8:
// row blocks I = 0 .. ceil(R/8)-1, column blocks J = 0 .. ceil(k/8)-1.
// Left-looking by block column J:
//   1. tiles (I, J), I >= J, in DMMA accumulator layout (lane (g, t) holds
//      rows 8I+g, columns 8J+2t, 8J+2t+1) start from -K(I, J): "full" tiles
//      (J < I, all eight rows real kernel rows) are evaluated right here from
//      the coordinates; the diagonal tiles and the last row block (RHS row,
//      padding) come from the packed shared-memory copy built before the
//      sweep (a pair table over those "irregular" pairs, ~22% of the k(k-1)/2);
//   2. acc(I) += sum_{Q < 2J} F(I, Q) F(J, Q)^T by DMMA, F(I, Q) = lane (g, t)
//      holding L[8I+g][4Q+t] — the A fragment of row block I and the B
//      fragment of (row block J)^T alike, kept in registers;
//   3. the panel (rows 8J .. k, eight columns) goes through the packed copy
//      to a row-per-lane layout and is factored right-looking (pivot by a
//      shuffle, 1/L_jj by a MUFU seed + two Newton steps, column values by
//      shuffles), written back (L in place of K) and loaded as the fragments
//      F(I, 2J), F(I, 2J+1) of the later block columns.
// The matrix is kept negated (-K, -y) so the DMMA can accumulate +L L^T.
// Failed pivots set a flag (Eigen LLT semantics: success iff every pivot > 0)
// and the jitter ladder reruns the row with the next rung, as solve_reg does.
// The backward solve L^T x = z keeps x in registers (x_j by a shuffle).
#include <climits>
#include <cstdlib>

#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

__constant__ double kJitDm[4] = {0.0, 1e-10, 1e-8, 1e-6};

__device__ __forceinline__ double jitter_dm(double v, int a) {
  for (int t = 1; t <= a; ++t) v = __dadd_rn(v, __dsub_rn(kJitDm[t], kJitDm[t - 1]));
  return v;
}

// packed row offsets (row i has i + 1 entries; rows start at even offsets)
__host__ __device__ constexpr int dm_ro(int i) { return ((i * (i + 1)) >> 1) + ((i + 1) >> 1); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

template <int K, int D>
struct DmShape {
  static constexpr int kR = K + 1;          // augmented rows (row K = y^T)
  static constexpr int kNBR = (kR + 7) / 8;  // row blocks
  static constexpr int kNBC = (K + 7) / 8;   // column blocks
  static constexpr int kIF = K / 8 - 1;      // last row block whose 8 rows are all kernel rows
  static_assert(K <= 63 && kIF >= 1, "two row slots per lane in the panels");
  static constexpr int kAug = ((dm_ro(K) + K + 8) + 1) & ~1;  // + slack for tile over-reads
  static constexpr int kXs = (K * D + 1) & ~1;
  static constexpr int kPerWarp = (kAug + kXs + (K + 1) / 2 + 2 + 1) & ~1;  // + sr (int32); 16-byte aligned
  // irregular pairs: strict lower (r, c), r < K, not in a full tile
  static constexpr int kNirr = 28 * (kIF + 1) + (K * (K - 1)) / 2 - (8 * (kIF + 1) * (8 * (kIF + 1) - 1)) / 2;
  static constexpr int kTabDoubles = ((kNirr + 3) / 4) * 2;
  __host__ __device__ static constexpr bool full(int I, int J) { return J < I && I <= kIF; }
};

// Irregular-pair table (shared by the CTA's warps): entry = (packed offset << 16) | (row << 8) | col.
template <int K, int D>
__device__ void fill_irr_table(uint32_t* ptab) {
  using Sh = DmShape<K, D>;
  constexpr int npairs = (K * (K - 1)) / 2;
  constexpr int r0 = 8 * (Sh::kIF + 1);
  for (int e = threadIdx.x; e < npairs; e += blockDim.x) {
    int r = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(e))) * 0.5f);
    while ((r * (r - 1)) / 2 > e) --r;
    while ((r * (r + 1)) / 2 <= e) ++r;
    const int c = e - (r * (r - 1)) / 2;
    const int rb = r >> 3;
    if (Sh::full(rb, c >> 3)) continue;
    int rank;
    if (rb <= Sh::kIF)
      rank = 28 * rb + ((r & 7) * ((r & 7) - 1)) / 2 + (c - 8 * rb);
    else
      rank = 28 * (Sh::kIF + 1) + (r * (r - 1)) / 2 - (r0 * (r0 - 1)) / 2 + c;
    ptab[rank] = (static_cast<uint32_t>(dm_ro(r) + c) << 16) | (static_cast<uint32_t>(r) << 8) |
                 static_cast<uint32_t>(c);
  }
}

template <int D, int KF>
__device__ __forceinline__ double dm_pair(const double (&u)[D], const double (&w)[D], double cs, const KParams& kn,
                                          const double* tab) {
  const double d0 = u[0] - w[0];
  double acc = d0 * d0;
#pragma unroll
  for (int c = 1; c < D; ++c) {
    const double dd = u[c] - w[c];
    acc = fma(dd, dd, acc);
  }
  return kernel_from_sq_build<KF>(acc, cs, kn, tab);
}

// 1/sqrt(x) for a pivot x > 0: MUFU seed (~2^-22) and ONE third-order step
// y (1 + e/2 + 3 e^2/8), e = 1 - x y^2 (error ~ e^3: below rounding), four
// dependent FP64 operations instead of the six of two Newton steps — the
// pivot chain is the serial part of the panel factorisation.
__device__ __forceinline__ double rsqrt_pivot3(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(x * y), y, 1.0);
  return fma(y * e, fma(e, 0.375, 0.5), y);
}

__device__ __forceinline__ int dm_row(int r, int K) { return r < K ? dm_ro(r) : dm_ro(K); }

// The blocked left-looking sweep (file header). Returns false iff some pivot
// of the kernel rows was <= 0. dv0 / dv1: 1/L_jj of columns lane / lane + 32.
template <int K, int D, int KF>
__device__ __forceinline__ bool dm_factor(double* A, const double* xs, const KParams& kn, double cs,
                                          const double* tab, int lane, double& dv0, double& dv1) {
  using Sh = DmShape<K, D>;
  constexpr int NBR = Sh::kNBR, NBC = Sh::kNBC;
  const int g = lane >> 2, t = lane & 3;
  double F[NBR][2 * NBC];
  bool bad = false;
  // -K of the full tiles of one block column, evaluated from the coordinates. The tiles of
  // block column J + 1 are evaluated inside the panel step of block column J (FMGP_DM_AHEAD):
  // independent FP64 work that runs under the panel's serial pivot chain.
  double accn[NBR][2];
  auto eval_full = [&](const int Jn) {
    double wc[2][D];
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int c = 0; c < D; ++c) wc[e][c] = xs[(8 * Jn + 2 * t + e < K ? 8 * Jn + 2 * t + e : 0) * D + c];
#pragma unroll
    for (int I = 0; I < NBR; ++I) {
      if (I >= Jn && Sh::full(I, Jn)) {
        double ur[D];
#pragma unroll
        for (int c = 0; c < D; ++c) ur[c] = xs[(8 * I + g) * D + c];
        accn[I][0] = dm_pair<D, KF>(ur, wc[0], cs, kn, tab);
        accn[I][1] = dm_pair<D, KF>(ur, wc[1], cs, kn, tab);
      }
    }
  };
#if FMGP_DM_AHEAD
  eval_full(0);
#endif
#pragma unroll
  for (int J = 0; J < NBC; ++J) {
#if FMGP_DM_SYNCJ
    __syncthreads();
#endif
    double acc[NBR][2];
    // 1. -K(I, J): full tiles from the coordinates, the rest from the packed copy
#if !FMGP_DM_AHEAD
    eval_full(J);
#endif
#pragma unroll
    for (int I = J; I < NBR; ++I) {
      if (Sh::full(I, J)) {
        acc[I][0] = accn[I][0];
        acc[I][1] = accn[I][1];
      } else {
        const int r = 8 * I + g;
        const double2 v = *reinterpret_cast<const double2*>(A + dm_row(r, K) + 8 * J + 2 * t);
        acc[I][0] = r <= K ? v.x : 0.0;
        acc[I][1] = r <= K ? v.y : 0.0;
      }
    }
    // 2. acc(I) += sum_Q F(I, Q) F(J, Q)^T
#pragma unroll
    for (int Q = 0; Q < 2 * J; ++Q)
#pragma unroll
      for (int I = J; I < NBR; ++I) dmma(acc[I], F[I][Q], F[J][Q]);
    // back to the packed copy (lower triangle of the diagonal tile, K entries of the RHS row)
#pragma unroll
    for (int I = J; I < NBR; ++I) {
      const int r = 8 * I + g, c0 = 8 * J + 2 * t;
      double* p = A + dm_row(r, K) + c0;
      if (Sh::full(I, J)) {
        *reinterpret_cast<double2*>(p) = make_double2(acc[I][0], acc[I][1]);
      } else if (r <= K) {
        const int lim = r < K ? r + 1 : K;  // columns < lim exist in row r
        if (c0 + 1 < lim) {
          *reinterpret_cast<double2*>(p) = make_double2(acc[I][0], acc[I][1]);
        } else if (c0 < lim) {
          p[0] = acc[I][0];
        }
      }
    }
    __syncwarp();
    // 3. panel: rows 8J .. K, columns 8J .. 8J + nc - 1, row-per-lane, right-looking
    constexpr int kMaxNc = 8;
    const int nc = K - 8 * J < 8 ? K - 8 * J : 8;
    const int RJ = K + 1 - 8 * J;
    const bool two = RJ > 32;
    const int ra = 8 * J + lane, rb = ra + 32;
    const int rla = lane, rlb = lane + 32;  // row index within the panel
    const double* pa = A + dm_row(ra <= K ? ra : K, K) + 8 * J;
    const double* pb = A + dm_row(rb <= K ? rb : K, K) + 8 * J;
    double xa[kMaxNc], xb[kMaxNc];
#pragma unroll
    for (int c = 0; c < kMaxNc; c += 2) {
      if (c < nc) {
        const double2 v = *reinterpret_cast<const double2*>(pa + c);
        xa[c] = v.x;
        xa[c + 1] = v.y;
        if (two) {
          const double2 q = *reinterpret_cast<const double2*>(pb + c);
          xb[c] = q.x;
          xb[c + 1] = q.y;
        }
      }
    }
#if FMGP_DM_AHEAD
    if (J + 1 < NBC) eval_full(J + 1);
#endif
    // The pivot of column c + 1 is taken from its owner lane right after column c is scaled (on that
    // lane the update of its own diagonal entry is la * la, no shuffle needed), so the next
    // shuffle -> rsqrt chain runs under the rest of column c's updates.
    double piv = -__shfl_sync(0xffffffffu, xa[0], 0);
#pragma unroll
    for (int c = 0; c < kMaxNc; ++c) {
      if (c < nc) {
        bad |= !(piv > 0.0);
        const double inv = rsqrt_pivot3(piv);
        const int col = 8 * J + c;
        if (col < 32) {
          if (lane == col) dv0 = inv;
        } else {
          if (lane == col - 32) dv1 = inv;
        }
        const double la = xa[c] * -inv;
        xa[c] = la;
        double lb = 0.0;
        if (two) {
          lb = xb[c] * -inv;
          xb[c] = lb;
        }
        if (c + 1 < nc) piv = -__shfl_sync(0xffffffffu, fma(la, la, xa[c + 1 < kMaxNc ? c + 1 : c]), c + 1);
#pragma unroll
        for (int c2 = c + 1; c2 < kMaxNc; ++c2) {
          if (c2 < nc) {
            const double lc = __shfl_sync(0xffffffffu, la, c2);
            xa[c2] = fma(la, lc, xa[c2]);
            if (two) xb[c2] = fma(lb, lc, xb[c2]);
          }
        }
      }
    }
    {
      double* wa = A + dm_row(ra <= K ? ra : K, K) + 8 * J;
      double* wb = A + dm_row(rb <= K ? rb : K, K) + 8 * J;
#pragma unroll
      for (int c = 0; c < kMaxNc; c += 2) {
        if (c < nc) {
          if (ra <= K) {
            if (c + 1 <= rla && c + 1 < nc) {
              *reinterpret_cast<double2*>(wa + c) = make_double2(xa[c], xa[c + 1]);
            } else if (c <= rla) {
              wa[c] = xa[c];
            }
          }
          if (two && rb <= K) {  // rows >= 8J + 32: every column of the panel exists
            if (c + 1 < nc)
              *reinterpret_cast<double2*>(wb + c) = make_double2(xb[c], xb[c + 1]);
            else
              wb[c] = xb[c];
          }
        }
      }
      (void)rlb;
    }
    __syncwarp();
    // 4. fragments of the new columns for the later block columns
    if (J + 1 < NBC) {
#pragma unroll
      for (int I = J + 1; I < NBR; ++I) {
        const int r = 8 * I + g;
        const double* p = A + dm_row(r <= K ? r : K, K) + 8 * J + t;
        F[I][2 * J] = r <= K ? p[0] : 0.0;
        F[I][2 * J + 1] = r <= K ? p[4] : 0.0;
      }
    }
  }
  return !bad;
}

// Backward solve L^T x = z (z = row K of the factored augmented matrix): lane
// l keeps x_l, x_{l+32}; x_j = z'_j / L_jj is formed on its owner and
// broadcast by a shuffle, then every lane updates with row j of L.
template <int K>
__device__ __forceinline__ void dm_back(const double* A, double dv0, double dv1, double* __restrict__ Crow, int lane) {
  const double* z = A + dm_ro(K);
  double y0 = lane < K ? z[lane] : 0.0;
  double y1 = lane + 32 < K ? z[lane + 32] : 0.0;
#pragma unroll
  for (int j = K - 1; j >= 0; --j) {
    const double xj = __shfl_sync(0xffffffffu, j < 32 ? y0 * dv0 : y1 * dv1, j & 31);
    const double* Lj = A + dm_ro(j);
    if (j < 32) {
      if (lane == j) y0 = xj;
      if (lane < j) y0 = fma(-Lj[lane < j ? lane : 0], xj, y0);
    } else {
      if (lane == j - 32) y1 = xj;
      y0 = fma(-Lj[lane], xj, y0);
      if (lane + 32 < j) y1 = fma(-Lj[lane + 32 < j ? lane + 32 : 0], xj, y1);
    }
  }
  if (lane < K) Crow[lane] = y0;
  if (lane + 32 < K) Crow[lane + 32] = y1;
}

#ifndef FMGP_DM_WARPS  // warps per CTA; with the per-row barrier below the CTA runs its rows in lockstep
#define FMGP_DM_WARPS 16
#endif
#ifndef FMGP_DM_PP
#define FMGP_DM_PP 3
#endif
#ifndef FMGP_DM_LOCKSTEP
#define FMGP_DM_LOCKSTEP 1
#endif
#ifndef FMGP_DM_AHEAD  // 1: the next block column's full tiles are evaluated under the current panel (A/B: no gain)
#define FMGP_DM_AHEAD 0
#endif
#ifndef FMGP_DM_SYNCJ  // 1: the CTA's warps also meet at every block column of the factorisation
#define FMGP_DM_SYNCJ 0
#endif
constexpr int kDmWarps = FMGP_DM_WARPS;
#ifndef FMGP_DM_MINB
#define FMGP_DM_MINB 1
#endif

template <int K, int D, int KF>
__global__ void __launch_bounds__(kDmWarps * kWarp, FMGP_DM_MINB)
solve_dm_kernel(const double* __restrict__ X, const double* __restrict__ Y, const int32_t* __restrict__ S,
                int64_t nrows, int64_t row_begin, KParams kp, double* __restrict__ C,
                unsigned long long* __restrict__ fail_min, const int32_t* __restrict__ order) {
  using Sh = DmShape<K, D>;
  extern __shared__ double smem[];
  __shared__ double s_exp[FMGP_BUILD_TAB_N];
  const int lane = threadIdx.x % kWarp;
  const int warp = threadIdx.x / kWarp;
  const int warps = blockDim.x / kWarp;
  uint32_t* ptab = reinterpret_cast<uint32_t*>(smem);
  stage_exp_table(s_exp);
  fill_irr_table<K, D>(ptab);
  __syncthreads();
  double* A = smem + Sh::kTabDoubles + warp * Sh::kPerWarp;
  double* xs = A + Sh::kAug;
  int32_t* sr = reinterpret_cast<int32_t*>(xs + Sh::kXs);
  KParams kn = kp;  // the matrix is built negated
  kn.s2 = -kp.s2;
  kn.diag = -kp.diag;
  const double cs = kernel_scale_build<KF>(kp);
  // Software pipeline over the warp's rows: the gathers of row i + 1 (S row -> X rows, Y) are
  // issued into registers while row i is solved — the S indices at the top of row i, the
  // coordinates just before its backward solve, where few registers are live — so the
  // dependent order -> S -> X chain (three DRAM/L2 round trips) is off the critical path.
  constexpr int NX = (K * D + kWarp - 1) / kWarp;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * warps;
  const int64_t it0 = static_cast<int64_t>(blockIdx.x) * warps + warp;
  auto row_of = [&](int64_t it) -> int64_t {
    if (it >= nrows) return -1;
    return order != nullptr ? order[it] : it;
  };
  double xn[NX], yn0 = 0.0, yn1 = 0.0;
  auto gather_xy = [&]() {  // from the indices staged in sr
#pragma unroll
    for (int i = 0; i < NX; ++i) {
      const int e = lane + i * kWarp;
      const int q = e / D, c = e - q * D;
      xn[i] = e < K * D ? X[static_cast<int64_t>(sr[q]) * D + c] : 0.0;
    }
    yn0 = lane < K ? Y[sr[lane < K ? lane : 0]] : 0.0;
    yn1 = lane + 32 < K ? Y[sr[lane + 32 < K ? lane + 32 : 0]] : 0.0;
  };
  // FMGP_DM_PREFETCH: 1 = the full register prefetch described above; 2 = only the next row's S entries are
  // kept in registers (3: plus an L1 prefetch of its coordinate rows); 0 = every row gathers at its own start
#ifndef FMGP_DM_PREFETCH
#define FMGP_DM_PREFETCH 2
#endif
  int64_t r = row_of(it0), rn = row_of(it0 + stride);
#if FMGP_DM_PREFETCH >= 2
  int32_t s0p = 0, s1p = 0;
  if (r >= 0) {
    if (lane < K) s0p = S[r * K + lane];
    if (lane + 32 < K) s1p = S[r * K + lane + 32];
  }
#endif
  if (FMGP_DM_PREFETCH == 1 && r >= 0) {
    for (int q = lane; q < K; q += kWarp) sr[q] = S[r * K + q];
    __syncwarp();
    gather_xy();
  }
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * warps; base < nrows; base += stride) {
#if FMGP_DM_LOCKSTEP
    __syncthreads();  // the CTA's warps start each row together (instruction-cache locality)
#endif
    const int64_t it = base + warp;
#if FMGP_DM_SYNCJ
    const bool active = it < nrows;  // a warp without a row still meets the CTA's barriers
#else
    if (it >= nrows) continue;
    constexpr bool active = true;
#endif
#if FMGP_DM_PREFETCH == 1
    const int64_t rnn = row_of(it + 2 * stride);
    int32_t s0n = 0, s1n = 0;
    if (rn >= 0) {
      if (lane < K) s0n = S[rn * K + lane];
      if (lane + 32 < K) s1n = S[rn * K + lane + 32];
    }
#elif FMGP_DM_PREFETCH >= 2
    if (lane < K) sr[lane] = s0p;
    if (lane + 32 < K) sr[lane + 32] = s1p;
    __syncwarp();
    gather_xy();
    rn = row_of(it + stride);
    if (rn >= 0) {  // in flight through the whole solve of this row
      if (lane < K) s0p = S[rn * K + lane];
      if (lane + 32 < K) s1p = S[rn * K + lane + 32];
    }
#else
    r = row_of(it);
    for (int q = lane; q < K; q += kWarp) sr[q] = S[r * K + q];
    __syncwarp();
    gather_xy();
#endif
#pragma unroll
    for (int i = 0; i < NX; ++i)
      if (lane + i * kWarp < K * D) xs[lane + i * kWarp] = xn[i];
    const double yl0 = yn0, yl1 = yn1;
    __syncwarp();
    bool ok = false;
    double dv0 = 0.0, dv1 = 0.0;
#pragma unroll 1
    for (int attempt = 0; attempt < 4; ++attempt) {
      const bool need = active && !ok;
#if FMGP_DM_SYNCJ
      if (!__syncthreads_or(need ? 1 : 0)) break;
      if (!need) {  // keep the barrier count of dm_factor
        for (int J = 0; J < Sh::kNBC; ++J) __syncthreads();
        continue;
      }
#else
      if (!need) break;
#endif
      // build: irregular pairs, diagonal, RHS
      {
        constexpr int NI = Sh::kNirr;
        constexpr int STEPS = (NI + kWarp - 1) / kWarp;
        constexpr int PP = FMGP_DM_PP;  // pairs in flight per lane (independent sqrt/exp chains)
#pragma unroll
        for (int s0 = 0; s0 < STEPS; s0 += PP) {
          uint32_t tw[PP];
          double u[PP][D], w[PP][D];
#pragma unroll
          for (int i = 0; i < PP; ++i) {
            const int e = lane + (s0 + i) * kWarp;
            tw[i] = ptab[e < NI ? e : lane];
            const double* xa = xs + ((tw[i] >> 8) & 0xffu) * D;
            const double* xb = xs + (tw[i] & 0xffu) * D;
#pragma unroll
            for (int c = 0; c < D; ++c) {
              u[i][c] = xa[c];
              w[i][c] = xb[c];
            }
          }
#pragma unroll
          for (int i = 0; i < PP; ++i) {
            if (s0 + i < STEPS) {
              const double v = dm_pair<D, KF>(u[i], w[i], cs, kn, s_exp);
              if (lane + (s0 + i) * kWarp < NI) A[tw[i] >> 16] = v;
            }
          }
        }
        const double dg = -jitter_dm(kp.diag, attempt);
        if (lane < K) A[dm_ro(lane) + lane] = dg;
        if (lane + 32 < K) A[dm_ro(lane + 32) + lane + 32] = dg;
        if (lane < K) A[dm_ro(K) + lane] = -yl0;
        if (lane + 32 < K) A[dm_ro(K) + lane + 32] = -yl1;
      }
      __syncwarp();
      ok = dm_factor<K, D, KF>(A, xs, kn, cs, s_exp, lane, dv0, dv1);
      __syncwarp();
    }
#if FMGP_DM_PREFETCH == 3
    if (rn >= 0) {  // the next row's coordinate rows and responses towards L2 / L1 before the backward solve
      if (lane < K) {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(X + static_cast<int64_t>(s0p) * D));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(Y + s0p));
      }
      if (lane + 32 < K) {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(X + static_cast<int64_t>(s1p) * D));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(Y + s1p));
      }
    }
#endif
#if FMGP_DM_PREFETCH == 1
    // the next row's coordinates and responses: in flight during the backward solve
    if (rn >= 0) {
      if (lane < K) sr[lane] = s0n;
      if (lane + 32 < K) sr[lane + 32] = s1n;
      __syncwarp();
      gather_xy();
    }
#endif
    if (!active) {
    } else if (!ok) {
      if (lane == 0) atomicMin(fail_min, static_cast<unsigned long long>(row_begin + r));
      __syncwarp();
    } else {
      dm_back<K>(A, dv0, dv1, C + r * K, lane);
      __syncwarp();
    }
#if FMGP_DM_PREFETCH == 1
    r = rn;
    rn = rnn;
#elif FMGP_DM_PREFETCH >= 2
    r = rn;
#endif
  }
}

template <int K, int D, int KF>
cudaError_t launch_dm(const double* X, const double* Y, const int32_t* S, int64_t nrows, int64_t row_begin,
                      const KParams& kp, double* C, unsigned long long* fail_min, int num_sms, cudaStream_t stream,
                      const int32_t* order) {
  using Sh = DmShape<K, D>;
  const size_t smem = sizeof(double) * (Sh::kTabDoubles + Sh::kPerWarp * kDmWarps);
  cudaError_t err = cudaFuncSetAttribute(solve_dm_kernel<K, D, KF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  int per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_dm_kernel<K, D, KF>, kDmWarps * kWarp, smem);
  if (err != cudaSuccess) return err;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (nrows + kDmWarps - 1) / kDmWarps;
  const int64_t grid = std::min<int64_t>(need, static_cast<int64_t>(num_sms) * per_sm);
  solve_dm_kernel<K, D, KF><<<static_cast<unsigned>(grid), kDmWarps * kWarp, smem, stream>>>(
      X, Y, S, nrows, row_begin, kp, C, fail_min, order);
  note_launches(1);
  return cudaGetLastError();
}

template <int K, int D>
cudaError_t launch_dm_kind(const double* X, const double* Y, const int32_t* S, int64_t nrows, int64_t row_begin,
                           const KParams& kp, double* C, unsigned long long* fail_min, int num_sms,
                           cudaStream_t stream, const int32_t* order) {
  switch (kp.kind == 1 ? 0 : 1 + kp.nu_code) {  // kernel_code(), on the host
    case 0: return launch_dm<K, D, 0>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order);
    case 1: return launch_dm<K, D, 1>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order);
    case 2: return launch_dm<K, D, 2>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order);
    default: return launch_dm<K, D, 3>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order);
  }
}

}  // namespace

bool fused_solve_dm_supported(int k, int d, int m, const KParams& kp) {
  const char* e = std::getenv("FMGP_SOLVE_DM");  // read per call: A/B in one process; 0 = register solve
  const bool on = !(e != nullptr && e[0] == '0');
  return on && m == 1 && (d == 2 || d == 3) && (k == 50 || k == 30) && (kp.kind == 1 || kp.nu_code <= 2);
}

cudaError_t fused_solve_dm(const double* X, const double* Y, int d, const int32_t* S, int64_t nrows,
                           int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                           int num_sms, cudaStream_t stream, const int32_t* order) {
  if (nrows <= 0) return cudaSuccess;
  if (k == 50) {
    return d == 2 ? launch_dm_kind<50, 2>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order)
                  : launch_dm_kind<50, 3>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order);
  }
  return d == 2 ? launch_dm_kind<30, 2>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order)
                : launch_dm_kind<30, 3>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order);
}

}  // namespace fmgp
