// K2-reg — the fused neighbourhood solve with register-resident rows, for
// compile-time neighbourhood sizes (the BASELINE shapes k in {30, 50}).
// Same contract as solve.cu (fast_predict.cpp:98-106, kernel.cpp:106-119,
// linalg.cpp:10-36), one warp per neighbourhood.
//
// Why: the shared-memory left-looking kernel is bound by the LSU pipe (one
// per-lane 64-bit load per FMA). Here each lane owns rows of the augmented
// matrix [K ; Y^T] in registers (static indexing: K and M are template
// parameters and the column loop is fully unrolled). Column j needs only the
// pivot row L_j., which its owner writes to shared memory as it is produced
// and every lane reads as a 128-bit broadcast. The RHS rows (K .. K+M-1) ride
// along, so the column sweep also performs the forward substitution; the
// backward solve then runs over the shared-memory copy of L.
//
// Row ownership (R = K + M rows): lane l owns row P + l (slot B) where
// P = max(R - 32, 0), and for l < P also row l (slot A). Slot A rows finish
// by column P - 1, so columns >= P run on one slot, and slot-B entries >= P
// are only loaded (still the original values) when column P starts: the
// live register set is at most max(2P, K) doubles per lane.
//
// Build (small d): the strict lower triangle is spread over the lanes by a
// CTA-shared pair table; the entries use the branch-free build arithmetic of
// fmgp_common.cuh (kernel_from_sq_build). The factorisation is branch-free:
// a failed pivot is recorded in a flag and the jitter ladder retried after
// the sweep (Eigen LLT semantics: success iff every pivot > 0).
#include <climits>
#include <cstdlib>

#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

__constant__ double kJitR[4] = {0.0, 1e-10, 1e-8, 1e-6};

// The Gram build replaces the direct difference loop from this dimension on
// (FMGP_SOLVE_GRAM=0 turns it off for A/B checks).
constexpr int kGramMinD = 32;

__host__ __device__ constexpr int ro_r(int i) { return ((i * (i + 1)) >> 1) + ((i + 1) >> 1); }

__device__ __forceinline__ double jitter_r(double v, int a) {
  for (int t = 1; t <= a; ++t) v = __dadd_rn(v, __dsub_rn(kJitR[t], kJitR[t - 1]));
  return v;
}

template <int K, int M>
struct RegShape {
  static constexpr int kRows = K + M;
  static constexpr int kRw = (K + 1) & ~1;             // padded RHS row length
  static constexpr int kAug = ro_r(K) + M * kRw;       // augmented packed size (doubles)
  static constexpr bool kTwo = kRows > 32;            // two row slots on some lanes?
  static_assert(kRows <= 64, "at most two row slots per lane");
  // slot A: rows 0 .. kP-1 on lanes 0 .. kP-1; slot B: row kP + lane
  static constexpr int kP = kTwo ? kRows - 32 : 0;
  static constexpr int kDch = 16;                      // coordinate slice width staged per pass
  static constexpr int kXsStride = kDch + 2;           // = 2 mod 4 doubles: conflict-light 128-bit row loads
  // xs holds K x D coordinates for the small-d build (D > 0), K x kXsStride slices otherwise
  // Gram build (d >= kGramMinD, K <= 32): 32 rows x kGramS doubles of one
  // 16-dimension chunk plus the 32 Gram diagonal entries
  static constexpr int kGramS = 20;  // row stride = 4 mod 16 doubles: conflict-free fragment loads
  static constexpr int kGramXs = 32 * kGramS + 32;
  __host__ __device__ static constexpr int xs_doubles(int D) {
    return D > 0 ? ((K * D + 1) & ~1) : (K <= 32 && kGramXs > kXsStride * K ? kGramXs : kXsStride * K);
  }
  __host__ __device__ static constexpr int per_warp(int D) {
    return ((kAug + ((K + 1) & ~1) /*dinv*/ + xs_doubles(D) + (K + 1) / 2 + 2) + 1) & ~1;
  }
  static constexpr int kTabDoubles = ((K * (K - 1) / 2 + 3) / 4) * 2;  // pair table (uint32), 16 B granules
  __host__ __device__ static constexpr int row_off(int i) { return i < K ? ro_r(i) : ro_r(K) + (i - K) * kRw; }
};

// Build [K(S_i) ; Y^T] in the packed shared-memory layout (pairs spread over
// lanes, incremental decode), diagonal at jitter rung `attempt`.
// Pair table shared by the CTA's warps: entry e of the strict lower triangle
// (row-major order) = (packed offset << 16) | (row << 8) | col.
template <int K>
__device__ void fill_pair_table(uint32_t* ptab) {
  constexpr int npairs = (K * (K - 1)) / 2;
  for (int e = threadIdx.x; e < npairs; e += blockDim.x) {
    int i = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(e))) * 0.5f);
    while ((i * (i - 1)) / 2 > e) --i;
    while ((i * (i + 1)) / 2 <= e) ++i;
    const int p = e - (i * (i - 1)) / 2;
    ptab[e] = (static_cast<uint32_t>(ro_r(i) + p) << 16) | (static_cast<uint32_t>(i) << 8) | static_cast<uint32_t>(p);
  }
}

template <int D>
__device__ __forceinline__ void load_pair(const double* xs, uint32_t t, double (&u)[D], double (&w)[D]) {
  const double* xa = xs + ((t >> 8) & 0xffu) * D;
  const double* xb = xs + (t & 0xffu) * D;
  if constexpr (D == 2) {
    const double2 a2 = *reinterpret_cast<const double2*>(xa);
    const double2 b2 = *reinterpret_cast<const double2*>(xb);
    u[0] = a2.x; u[1] = a2.y; w[0] = b2.x; w[1] = b2.y;
  } else {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      u[c] = xa[c];
      w[c] = xb[c];
    }
  }
}

// PP pairs per lane per step (e, e + NL, ..., independent: their sqrt/exp
// chains interleave); the next step's table words and coordinates are loaded
// at the top of the step, so the shared-memory chain table -> coordinates
// has a whole step of arithmetic to complete behind.
#ifndef FMGP_BUILD_PP
#define FMGP_BUILD_PP 4
#endif
#ifndef FMGP_BUILD_PP3
#define FMGP_BUILD_PP3 2
#endif
template <int K, int D, int KF, int NL = kWarp>
__device__ __forceinline__ void pair_loop(const double* xs, const uint32_t* ptab, const KParams& kp, double* A,
                                          int lane, const double* tab) {
  constexpr int PP = D <= 2 ? FMGP_BUILD_PP : FMGP_BUILD_PP3;  // fewer in flight for d = 3 (registers)
  constexpr int npairs = (K * (K - 1)) / 2;
  static_assert(npairs >= PP * NL, "first step loads PP entries per lane");
  const double c = kernel_scale_build<KF>(kp);
  // Two register sets (a, b) in ping-pong: a step evaluates one set while the
  // other is loaded for the next step, with no register copies between steps.
  uint32_t ta[PP], tb[PP];
  double ua[PP][D], wa[PP][D], ub[PP][D], wb[PP][D];
  auto load = [&](int e, uint32_t (&t)[PP], double (&u)[PP][D], double (&w)[PP][D]) {
#pragma unroll
    for (int i = 0; i < PP; ++i) {
      const int f = e + i * NL;
      t[i] = ptab[f < npairs ? f : lane];
      load_pair<D>(xs, t[i], u[i], w[i]);
    }
  };
  auto eval = [&](int e, const uint32_t (&t)[PP], const double (&u)[PP][D], const double (&w)[PP][D]) {
    double v[PP];
#pragma unroll
    for (int i = 0; i < PP; ++i) {
      const double d0 = u[i][0] - w[i][0];
      double acc = d0 * d0;
#pragma unroll
      for (int cc = 1; cc < D; ++cc) {
        const double dd = u[i][cc] - w[i][cc];
        acc = fma(dd, dd, acc);
      }
      v[i] = kernel_from_sq_build<KF>(acc, c, kp, tab);
    }
#pragma unroll
    for (int i = 0; i < PP; ++i)
      if (e + i * NL < npairs) A[t[i] >> 16] = v[i];
  };
  load(lane, ta, ua, wa);
#pragma unroll 1
  for (int e = lane; e < npairs; e += 2 * PP * NL) {
    load(e + PP * NL, tb, ub, wb);
    eval(e, ta, ua, wa);
    if (e + PP * NL >= npairs) break;
    load(e + 2 * PP * NL, ta, ua, wa);
    eval(e + PP * NL, tb, ub, wb);
  }
}

// Small-d build (d = D known at compile time): all K coordinates staged once,
// one pair per lane per step from the pair table, no index decode.
template <int K, int M, int D>
__device__ void build_small(const double* __restrict__ X, const double* __restrict__ Y, const int32_t* sr,
                            const KParams& kp, int attempt, double* A, double* xs, const uint32_t* ptab, int lane,
                            const double* tab) {
  using Sh = RegShape<K, M>;
  for (int e = lane; e < K * D; e += kWarp) {
    const int t = e / D, c = e - t * D;
    xs[e] = X[static_cast<int64_t>(sr[t]) * D + c];
  }
  __syncwarp();
  switch (kernel_code(kp)) {  // uniform: one pair loop per kernel kind, no per-pair dispatch
    case 0: pair_loop<K, D, 0>(xs, ptab, kp, A, lane, tab); break;
    case 1: pair_loop<K, D, 1>(xs, ptab, kp, A, lane, tab); break;
    case 2: pair_loop<K, D, 2>(xs, ptab, kp, A, lane, tab); break;
    case 3: pair_loop<K, D, 3>(xs, ptab, kp, A, lane, tab); break;
    default: pair_loop<K, D, 4>(xs, ptab, kp, A, lane, tab); break;
  }
  const double dg = jitter_r(kp.diag, attempt);
  for (int i = lane; i < K; i += kWarp) A[ro_r(i) + i] = dg;
  for (int e = lane; e < K * M; e += kWarp) {
    const int t = e / M, c = e - t * M;
    A[Sh::row_off(K + c) + t] = Y[static_cast<int64_t>(sr[t]) * M + c];
  }
  __syncwarp();
}

template <int K, int M>
__device__ void build_reg(const double* __restrict__ X, const double* __restrict__ Y, int d, const int32_t* sr,
                          const KParams& kp, int attempt, double* A, double* xs, int lane) {
  using Sh = RegShape<K, M>;
  constexpr int npairs = (K * (K - 1)) / 2;
  const int dchunk = d < Sh::kDch ? d : Sh::kDch;
  for (int c0 = 0; c0 < d; c0 += dchunk) {
    const int dc = min(dchunk, d - c0);
    for (int e = lane; e < K * dc; e += kWarp) {
      const int t = e / dc, c = e - t * dc;
      xs[t * Sh::kXsStride + c] = X[static_cast<int64_t>(sr[t]) * d + c0 + c];
    }
    __syncwarp();
    const bool last = c0 + dc >= d;
    // two independent pairs per iteration (e and e + 32) for ILP through sqrt/exp
    int ia, pa, ib, pb;
    {
      const int e0 = lane, e1 = lane + 32;
      ia = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(e0))) * 0.5f);
      while ((ia * (ia - 1)) / 2 > e0) --ia;
      while ((ia * (ia + 1)) / 2 <= e0) ++ia;
      pa = e0 - (ia * (ia - 1)) / 2;
      ib = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(e1))) * 0.5f);
      while ((ib * (ib - 1)) / 2 > e1) --ib;
      while ((ib * (ib + 1)) / 2 <= e1) ++ib;
      pb = e1 - (ib * (ib - 1)) / 2;
    }
    for (int e = lane; e < npairs; e += 2 * kWarp) {
      const bool hb = e + kWarp < npairs;
      const double* xa = xs + ia * Sh::kXsStride;
      const double* xa2 = xs + pa * Sh::kXsStride;
      const double* xb = xs + (hb ? ib : ia) * Sh::kXsStride;
      const double* xb2 = xs + (hb ? pb : pa) * Sh::kXsStride;
      const int offa = ro_r(ia) + pa;
      const int offb = ro_r(hb ? ib : ia) + (hb ? pb : pa);
      double acca = c0 == 0 ? 0.0 : A[offa];
      double accb = c0 == 0 ? 0.0 : A[offb];
      int c = 0;
#pragma unroll 4
      for (; c + 1 < dc; c += 2) {  // t-ordered, fused multiply-add (matrix entries within ~1 ulp)
        const double2 ua = *reinterpret_cast<const double2*>(xa + c);
        const double2 wa = *reinterpret_cast<const double2*>(xa2 + c);
        const double2 ub = *reinterpret_cast<const double2*>(xb + c);
        const double2 wb = *reinterpret_cast<const double2*>(xb2 + c);
        const double da0 = ua.x - wa.x, da1 = ua.y - wa.y, db0 = ub.x - wb.x, db1 = ub.y - wb.y;
        acca = fma(da0, da0, acca);
        accb = fma(db0, db0, accb);
        acca = fma(da1, da1, acca);
        accb = fma(db1, db1, accb);
      }
      if (c < dc) {
        const double da = xa[c] - xa2[c], db = xb[c] - xb2[c];
        acca = fma(da, da, acca);
        accb = fma(db, db, accb);
      }
      if (last) {
        const double va = kernel_eval_fast(sqrt(acca), kp);
        const double vb = kernel_eval_fast(sqrt(accb), kp);
        A[offa] = va;
        if (hb) A[offb] = vb;
      } else {
        A[offa] = acca;
        if (hb) A[offb] = accb;
      }
      pa += 2 * kWarp;
      while (pa >= ia) {
        pa -= ia;
        ++ia;
      }
      pb += 2 * kWarp;
      while (pb >= ib) {
        pb -= ib;
        ++ib;
      }
    }
    __syncwarp();
  }
  const double dg = jitter_r(kp.diag, attempt);
  for (int i = lane; i < K; i += kWarp) A[ro_r(i) + i] = dg;
  for (int e = lane; e < K * M; e += kWarp) {
    const int t = e / M, c = e - t * M;
    A[Sh::row_off(K + c) + t] = Y[static_cast<int64_t>(sr[t]) * M + c];
  }
  __syncwarp();
}

// Large-d build (D = 0, K <= 32) on the FP64 tensor cores: the Gram matrix
// G = X_N X_N^T of the neighbourhood's coordinates (rows padded to 32) is
// accumulated with DMMA m8n8k4 over 16-dimension chunks staged in shared
// memory (lane (g, t) holds X[8I + g][c + t], which is both the A fragment of
// row block I and the B fragment of column block I, so one 64-bit load per
// block and k-step feeds the 10 lower-triangle tiles), then
// d^2 = G_ii + G_jj - 2 G_ij (clamped at 0) feeds the kernel. Cost per pair
// ~2d/16 DMMA-thread ops instead of 2d scalar ops with two shared loads; the
// distance differs from the reference's sum of squared differences by
// rounding relative to the neighbourhood's squared extent (coordinates are
// centred on the query point first), far inside the coefficient tolerance.
// A pair with d^2 <= 1e-12 (G_ii + G_jj) is recomputed exactly
// from X (sum of squared differences), so exact duplicates keep the nugget
// (kernel.cpp:106-119) bit for bit. The next chunk's coordinates are loaded
// from global memory while the current chunk's MMAs run.
__device__ __forceinline__ void dmma_884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int K, int M>
__device__ void build_gram(const double* __restrict__ X, const double* __restrict__ Y, int d, const int32_t* sr,
                           const KParams& kp, int attempt, double* A, double* xs, int lane) {
  using Sh = RegShape<K, M>;
  static_assert(K <= 32, "one 32-row Gram block");
  constexpr int S = Sh::kGramS;
  double* gd = xs + 32 * S;
  const int g = lane >> 2, t = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int I = 0; I < 4; ++I)
#pragma unroll
    for (int J = 0; J < 4; ++J) acc[I][J][0] = acc[I][J][1] = 0.0;
  // gather slots: element e = lane + 32 u of a 32 x 16 chunk is (row e >> 4, dim e & 15).
  // Coordinates are taken relative to the neighbourhood's first point (its
  // query row, S[i][0] = i): the Gram form d^2 = G_ii + G_jj - 2 G_ij then
  // loses digits relative to the neighbourhood's extent, not to |x|^2 (data
  // far from the origin keeps the coefficient tolerance).
  const double* x0 = X + static_cast<int64_t>(sr[0]) * d;
  double pre[16];
  auto gather = [&](int c0) {
    const int dim = lane & 15;
    const double ref = c0 + dim < d ? x0[c0 + dim] : 0.0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int row = (lane >> 4) + 2 * u;
      const bool ok = row < K && c0 + dim < d;
      pre[u] = ok ? X[static_cast<int64_t>(sr[row < K ? row : 0]) * d + c0 + dim] - ref : 0.0;
    }
  };
  gather(0);
  for (int c0 = 0; c0 < d; c0 += 16) {
#pragma unroll
    for (int u = 0; u < 16; ++u) xs[((lane >> 4) + 2 * u) * S + (lane & 15)] = pre[u];
    __syncwarp();
    if (c0 + 16 < d) gather(c0 + 16);
#pragma unroll
    for (int kq = 0; kq < 16; kq += 4) {
      double f[4];
#pragma unroll
      for (int I = 0; I < 4; ++I) f[I] = xs[(8 * I + g) * S + kq + t];
#pragma unroll
      for (int I = 0; I < 4; ++I)
#pragma unroll
        for (int J = 0; J <= I; ++J) dmma_884(acc[I][J], f[I], f[J]);
    }
    __syncwarp();
  }
  // Gram diagonal -> shared memory
#pragma unroll
  for (int I = 0; I < 4; ++I) {
    if (g == 2 * t) gd[8 * I + g] = acc[I][I][0];
    if (g == 2 * t + 1) gd[8 * I + g] = acc[I][I][1];
  }
  __syncwarp();
#pragma unroll
  for (int I = 0; I < 4; ++I) {
#pragma unroll
    for (int J = 0; J <= I; ++J) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = 8 * I + g, c = 8 * J + 2 * t + e;
        if (r < K && c < r) {
          const double gr = gd[r], gc = gd[c];
          double d2 = fmax(gr + gc - 2.0 * acc[I][J][e], 0.0);
          if (d2 <= 1e-12 * (gr + gc)) {  // near or exact duplicate: the exact key decides
            const double* xa = X + static_cast<int64_t>(sr[r]) * d;
            const double* xb = X + static_cast<int64_t>(sr[c]) * d;
            double ex = 0.0;
            for (int q = 0; q < d; ++q) {
              const double df = xa[q] - xb[q];
              ex = fma(df, df, ex);
            }
            d2 = ex;
          }
          A[ro_r(r) + c] = kernel_eval_fast(sqrt(d2), kp);
        }
      }
    }
  }
  const double dg = jitter_r(kp.diag, attempt);
  for (int i = lane; i < K; i += kWarp) A[ro_r(i) + i] = dg;
  for (int e = lane; e < K * M; e += kWarp) {
    const int tt = e / M, cc = e - tt * M;
    A[Sh::row_off(K + cc) + tt] = Y[static_cast<int64_t>(sr[tt]) * M + cc];
  }
  __syncwarp();
}

// Register-resident left-looking factorisation of the augmented matrix
// (ownership in the file header): column j of the lane's rows accumulates
// a_rj - sum_{p<j} a_rp L_jp from its registers and the pivot row L_j.
// broadcast from shared memory (128-bit). The owner of row j supplies the
// pivot by a shuffle; every lane scales by the same 1/L_jj (the owner's own
// entry becomes piv * (1/sqrt(piv)) = L_jj). Rows below the column are
// inactive for it: their lanes compute and discard (stores are predicated).
// Returns false iff some pivot was <= 0 (Eigen LLT semantics).
template <int K, int M>
__device__ bool factor_reg(double* A, double* dinv, int lane) {
  using Sh = RegShape<K, M>;
  constexpr int kP = Sh::kP;
  constexpr int kB0 = kP > 0 ? kP : K;  // slot-B entries loaded before the sweep
  const int rB = kP + lane;
  const bool hasB = rB < Sh::kRows;
  const bool hasA = lane < kP;
  double* RB = A + Sh::row_off(hasB ? rB : 0);
  double* RA = A + Sh::row_off(hasA ? lane : 0);
  double b[K];
  double a[kP > 0 ? kP : 1];
  // Entries beyond a row's length read the next packed row (in bounds, never
  // used: a row r only ever reads its entries < j <= r).
#pragma unroll
  for (int p = 0; p + 1 < kB0; p += 2) {
    const double2 v = *reinterpret_cast<const double2*>(RB + p);
    b[p] = v.x;
    b[p + 1] = v.y;
  }
  if constexpr (kB0 & 1) b[kB0 - 1] = RB[kB0 - 1];
  if constexpr (kP > 0) {
#pragma unroll
    for (int p = 0; p + 1 < kP; p += 2) {
      const double2 v = *reinterpret_cast<const double2*>(RA + p);
      a[p] = v.x;
      a[p + 1] = v.y;
    }
    if constexpr (kP & 1) a[kP - 1] = RA[kP - 1];
  }
  bool bad = false;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if constexpr (kP > 0) {
      if (j == kP) {  // slot A is finished: bring in the rest of slot B (still original values)
        constexpr int p0 = (kP + 1) & ~1;  // 128-bit loads from the first even entry
        if constexpr (kP & 1) b[kP] = RB[kP];
#pragma unroll
        for (int p = p0; p + 1 < K; p += 2) {
          const double2 v = *reinterpret_cast<const double2*>(RB + p);
          b[p] = v.x;
          b[p + 1] = v.y;
        }
        if constexpr ((K - p0) & 1) b[K - 1] = RB[K - 1];
      }
    }
    const bool twoA = kP > 0 && j < kP;
    const double* Lj = A + ro_r(j);  // pivot row j (entries < j are final)
    // four independent accumulators per slot (DFMA latency chains of j/4)
    double b0 = b[j], b1 = 0.0, b2 = 0.0, b3 = 0.0;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (twoA) a0 = a[j < kP ? j : 0];
#pragma unroll
    for (int p = 0; p + 3 < j; p += 4) {
      const double2 l = *reinterpret_cast<const double2*>(Lj + p);
      const double2 m = *reinterpret_cast<const double2*>(Lj + p + 2);
      b0 = fma(-b[p], l.x, b0);
      b1 = fma(-b[p + 1], l.y, b1);
      b2 = fma(-b[p + 2], m.x, b2);
      b3 = fma(-b[p + 3], m.y, b3);
      if (twoA) {
        a0 = fma(-a[p < kP ? p : 0], l.x, a0);
        a1 = fma(-a[p + 1 < kP ? p + 1 : 0], l.y, a1);
        a2 = fma(-a[p + 2 < kP ? p + 2 : 0], m.x, a2);
        a3 = fma(-a[p + 3 < kP ? p + 3 : 0], m.y, a3);
      }
    }
    {  // up to three leftover columns (j is a compile-time constant here)
      const int p0 = j & ~3;
      if ((j & 3) >= 2) {
        const double2 l = *reinterpret_cast<const double2*>(Lj + p0);
        b0 = fma(-b[p0], l.x, b0);
        b1 = fma(-b[p0 + 1], l.y, b1);
        if (twoA) {
          a0 = fma(-a[p0 < kP ? p0 : 0], l.x, a0);
          a1 = fma(-a[p0 + 1 < kP ? p0 + 1 : 0], l.y, a1);
        }
      }
      if ((j & 1) == 1) {
        const int q = j - 1;
        const double l = Lj[q];
        b2 = fma(-b[q], l, b2);
        if (twoA) a2 = fma(-a[q < kP ? q : 0], l, a2);
      }
    }
    const double sB = (b0 + b1) + (b2 + b3);
    const double sA = (a0 + a1) + (a2 + a3);
    const double piv = __shfl_sync(0xffffffffu, twoA ? sA : sB, twoA ? j : j - kP);
    bad |= !(piv > 0.0);
    const double inv = rsqrt_pivot(piv);
    const double vB = sB * inv;
    b[j] = vB;
    if (hasB && rB >= j) RB[j] = vB;
    if (twoA) {
      const double vA = sA * inv;
      a[j < kP ? j : 0] = vA;
      if (hasA && lane >= j) RA[j] = vA;
    }
    if (lane == 0) dinv[j] = inv;
    __syncwarp();
  }
  return !bad;
}

// Backward solve L^T x = z, z = the forward-substituted RHS rows. Lane l keeps
// x_l and x_{l+32} in registers; column j (descending) broadcasts x_j by a
// shuffle and every lane updates its entries with row j of L (a contiguous
// shared-memory row, conflict-free). Writes C directly (coalesced for M = 1).
template <int K, int M>
__device__ void back_solve_reg(const double* A, const double* dinv, double* __restrict__ Crow, int lane) {
  using Sh = RegShape<K, M>;
  static_assert(K <= 64, "two register slots per lane");
#pragma unroll 1
  for (int c = 0; c < M; ++c) {
    const double* z = A + Sh::row_off(K + c);
    double y0 = lane < K ? z[lane] : 0.0;
    double y1 = lane + 32 < K ? z[lane + 32] : 0.0;
#pragma unroll
    for (int j = K - 1; j >= 0; --j) {
      const double yj = __shfl_sync(0xffffffffu, j < 32 ? y0 : y1, j & 31);
      const double xj = yj * dinv[j];
      const double* Lj = A + ro_r(j);
      if (j < 32) {
        if (lane == j) y0 = xj;
        if (lane < j) y0 = fma(-Lj[lane], xj, y0);
      } else {
        if (lane == j - 32) y1 = xj;
        if (lane < 32) y0 = fma(-Lj[lane], xj, y0);
        if (lane + 32 < j) y1 = fma(-Lj[lane + 32], xj, y1);
      }
    }
    if (lane < K) Crow[lane * M + c] = y0;
    if (lane + 32 < K) Crow[(lane + 32) * M + c] = y1;
  }
}

// ---------------------------------------------------------------- K2-pair
// (A/B variant, FMGP_SOLVE_PAIR=1; profiles/r01/ab_pair_solve.txt.)
// Two neighbourhoods per warp, one per half-warp (lanes 0-15 / 16-31), for
// the small-d shapes. Why: the register sweep above is bound by the
// shared-memory data pipe, and its largest consumer is the pivot-row
// broadcast (every lane reads L_j. for its one or two rows; a broadcast
// 128-bit load costs two wavefronts per 16 bytes). With 16 lanes per
// neighbourhood each lane owns up to four rows, so one broadcast feeds up to
// four FMAs per lane, and a single load instruction serves both halves
// (each half-warp is one wavefront anyway): half the pivot traffic, half the
// per-column pivot/rsqrt/shuffle overhead and fewer idle FMA lanes per
// neighbourhood, at the cost of half as many warps (the shared memory per
// neighbourhood, not registers, caps the neighbourhoods in flight).
//
// Ownership within a half (hl = lane & 15, R = k + m rows, NS = ceil(R/16)
// slots): slot s holds row base(s) + hl, base(s) = R - 16 (NS - s) (rows < 0
// absent). Slot s finishes at column base(s) + 15, so its entries are loaded
// in stages: at column end(t-1) every slot s >= t loads its (still original)
// entries end(t-1) .. end(t)-1, end(s) = min(base(s) + 16, k).
template <int K, int M>
struct PairShape {
  static constexpr int kRows = K + M;
  static constexpr int kNS = (kRows + 15) / 16;
  static_assert(kNS <= 4, "at most four row slots per lane");
  __host__ __device__ static constexpr int base(int s) { return kRows - 16 * (kNS - s); }
  __host__ __device__ static constexpr int end(int s) { return base(s) + 16 < K ? base(s) + 16 : K; }
  __host__ __device__ static constexpr int start(int t) { return t == 0 ? 0 : end(t - 1); }
  __host__ __device__ static constexpr int owner_slot(int j) { return (j - base(0)) / 16; }
};

template <int K, int M>
__device__ bool factor_pair(double* A, double* dinv, int lane) {
  using Ps = PairShape<K, M>;
  using Sh = RegShape<K, M>;
  constexpr int NS = Ps::kNS;
  const int hl = lane & 15;
  const int hbase = lane & 16;
  double x[NS][K];
  double* Rs[NS];
  int rs[NS];
  bool vs[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    rs[s] = Ps::base(s) + hl;
    vs[s] = rs[s] >= 0 && rs[s] < Sh::kRows;
    Rs[s] = A + Sh::row_off(vs[s] ? rs[s] : 0);
  }
  bool bad = false;
#pragma unroll
  for (int j = 0; j < K; ++j) {
#pragma unroll
    for (int t = 0; t < NS; ++t) {
      if (j == Ps::start(t) && Ps::start(t) < Ps::end(t)) {
        // stage t: slots >= t load entries start(t) .. end(t)-1 (original values; entries
        // beyond a row's length read the next packed row and are never used)
#pragma unroll
        for (int s = t; s < NS; ++s) {
          int p = Ps::start(t);
          if (p & 1) {
            x[s][p] = Rs[s][p];
            ++p;
          }
#pragma unroll
          for (; p + 1 < Ps::end(t); p += 2) {
            const double2 v = *reinterpret_cast<const double2*>(Rs[s] + p);
            x[s][p] = v.x;
            x[s][p + 1] = v.y;
          }
          if (p < Ps::end(t)) x[s][p] = Rs[s][p];
        }
      }
    }
    const double* Lj = A + ro_r(j);  // pivot row j (entries < j are final)
    double acc[NS][4];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const bool act = Ps::base(s) + 15 >= j;
      acc[s][0] = act ? x[s][act ? j : 0] : 0.0;
      acc[s][1] = acc[s][2] = acc[s][3] = 0.0;
    }
#pragma unroll
    for (int p = 0; p + 3 < j; p += 4) {
      const double2 l = *reinterpret_cast<const double2*>(Lj + p);
      const double2 m = *reinterpret_cast<const double2*>(Lj + p + 2);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        if (Ps::base(s) + 15 >= j) {
          acc[s][0] = fma(-x[s][p], l.x, acc[s][0]);
          acc[s][1] = fma(-x[s][p + 1], l.y, acc[s][1]);
          acc[s][2] = fma(-x[s][p + 2], m.x, acc[s][2]);
          acc[s][3] = fma(-x[s][p + 3], m.y, acc[s][3]);
        }
      }
    }
    {
      const int p0 = j & ~3;
      if ((j & 3) >= 2) {
        const double2 l = *reinterpret_cast<const double2*>(Lj + p0);
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          if (Ps::base(s) + 15 >= j) {
            acc[s][0] = fma(-x[s][p0], l.x, acc[s][0]);
            acc[s][1] = fma(-x[s][p0 + 1], l.y, acc[s][1]);
          }
        }
      }
      if ((j & 1) == 1) {
        const int q = j - 1;
        const double l = Lj[q];
#pragma unroll
        for (int s = 0; s < NS; ++s)
          if (Ps::base(s) + 15 >= j) acc[s][2] = fma(-x[s][q], l, acc[s][2]);
      }
    }
    double sum[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) sum[s] = (acc[s][0] + acc[s][1]) + (acc[s][2] + acc[s][3]);
    const int so = Ps::owner_slot(j);
    const double piv = __shfl_sync(0xffffffffu, sum[so], hbase | (j - Ps::base(so)));
    bad |= !(piv > 0.0);
    const double inv = rsqrt_pivot(piv);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (Ps::base(s) + 15 >= j) {
        const double v = sum[s] * inv;
        x[s][j] = v;
        if (vs[s] && rs[s] >= j) Rs[s][j] = v;
      }
    }
    if (hl == 0) dinv[j] = inv;
    __syncwarp();
  }
  return !bad;
}

// Backward solve L^T x = z per half: lane hl keeps x_p for p = hl, hl+16,
// hl+32, ... in registers; x_j is broadcast within the half by a shuffle and
// row j of L is read contiguously (16 lanes x 8 bytes per half).
template <int K, int M>
__device__ void back_solve_pair(const double* A, const double* dinv, double* __restrict__ Crow, bool store, int lane) {
  using Sh = RegShape<K, M>;
  constexpr int NY = (K + 15) / 16;
  const int hl = lane & 15;
  const int hbase = lane & 16;
#pragma unroll 1
  for (int c = 0; c < M; ++c) {
    const double* z = A + Sh::row_off(K + c);
    double y[NY];
#pragma unroll
    for (int t = 0; t < NY; ++t) y[t] = 16 * t + hl < K ? z[16 * t + hl < K ? 16 * t + hl : 0] : 0.0;
#pragma unroll
    for (int j = K - 1; j >= 0; --j) {
      const double yj = __shfl_sync(0xffffffffu, y[j / 16], hbase | (j & 15));
      const double xj = yj * dinv[j];
      const double* Lj = A + ro_r(j);
#pragma unroll
      for (int t = 0; t < NY; ++t) {
        if (16 * t > j) continue;
        const int p = 16 * t + hl;
        if (16 * t + 15 < j) {
          y[t] = fma(-Lj[p], xj, y[t]);
        } else {
          if (p < j) y[t] = fma(-Lj[p < j ? p : 0], xj, y[t]);
          if (p == j) y[t] = xj;
        }
      }
    }
    if (store) {
#pragma unroll
      for (int t = 0; t < NY; ++t)
        if (16 * t + hl < K) Crow[(16 * t + hl) * M + c] = y[t];
    }
  }
}

// Small-d build of one half's neighbourhood with its 16 lanes.
template <int K, int M, int D>
__device__ void build_small_half(const double* __restrict__ X, const double* __restrict__ Y, const int32_t* sr,
                                 const KParams& kp, int rung, double* A, double* xs, const uint32_t* ptab, int hl) {
  using Sh = RegShape<K, M>;
  for (int e = hl; e < K * D; e += 16) {
    const int t = e / D, c = e - t * D;
    xs[e] = X[static_cast<int64_t>(sr[t]) * D + c];
  }
  __syncwarp();
  switch (kernel_code(kp)) {
    case 0: pair_loop<K, D, 0, 16>(xs, ptab, kp, A, hl, kExp2NegTab); break;
    case 1: pair_loop<K, D, 1, 16>(xs, ptab, kp, A, hl, kExp2NegTab); break;
    case 2: pair_loop<K, D, 2, 16>(xs, ptab, kp, A, hl, kExp2NegTab); break;
    case 3: pair_loop<K, D, 3, 16>(xs, ptab, kp, A, hl, kExp2NegTab); break;
    default: pair_loop<K, D, 4, 16>(xs, ptab, kp, A, hl, kExp2NegTab); break;
  }
  const double dg = jitter_r(kp.diag, rung);
  for (int i = hl; i < K; i += 16) A[ro_r(i) + i] = dg;
  for (int e = hl; e < K * M; e += 16) {
    const int t = e / M, c = e - t * M;
    A[Sh::row_off(K + c) + t] = Y[static_cast<int64_t>(sr[t]) * M + c];
  }
  __syncwarp();
}

constexpr int kPairWarps = 4;

template <int K, int M, int D>
__global__ void __launch_bounds__(kPairWarps * kWarp, 2)
solve_pair_kernel(const double* __restrict__ X, const double* __restrict__ Y, const int32_t* __restrict__ S,
                  int64_t nrows, int64_t row_begin, KParams kp, double* __restrict__ C,
                  unsigned long long* __restrict__ fail_min) {
  using Sh = RegShape<K, M>;
  extern __shared__ double smem[];
  const int lane = threadIdx.x % kWarp;
  const int warp = threadIdx.x / kWarp;
  const int warps = blockDim.x / kWarp;
  const int h = lane >> 4, hl = lane & 15;
  uint32_t* ptab = reinterpret_cast<uint32_t*>(smem);
  fill_pair_table<K>(ptab);
  __syncthreads();
  double* A = smem + Sh::kTabDoubles + (2 * warp + h) * Sh::per_warp(D);
  double* dinv = A + Sh::kAug;
  double* xs = dinv + ((K + 1) & ~1);
  int32_t* sr = reinterpret_cast<int32_t*>(xs + Sh::xs_doubles(D));
  for (int64_t pr = static_cast<int64_t>(blockIdx.x) * warps + warp; 2 * pr < nrows;
       pr += static_cast<int64_t>(gridDim.x) * warps) {
    const int64_t r = 2 * pr + h;
    const bool has = r < nrows;
    const int64_t rr = has ? r : 2 * pr;  // a missing second row repeats the first (never stored)
    for (int t = hl; t < K; t += 16) sr[t] = S[rr * K + t];
    __syncwarp();
    int rung = 0;
    bool ok = false;
    for (int it = 0; it < 4; ++it) {
      build_small_half<K, M, D>(X, Y, sr, kp, rung, A, xs, ptab, hl);
      ok = factor_pair<K, M>(A, dinv, lane);
      __syncwarp();
      // a half that failed moves to the next jitter rung; a half that succeeded
      // repeats its rung (same arithmetic, same result) while the other retries
      const bool retry = !ok && rung < 3;
      if (!__any_sync(0xffffffffu, retry)) break;
      if (retry) ++rung;
    }
    if (!ok && has && hl == 0) atomicMin(fail_min, static_cast<unsigned long long>(row_begin + r));
    back_solve_pair<K, M>(A, dinv, C + r * K * M, ok && has, lane);
    __syncwarp();
  }
}

template <int K, int M, int D>
cudaError_t launch_pair(const double* X, const double* Y, const int32_t* S, int64_t nrows, int64_t row_begin,
                        const KParams& kp, double* C, unsigned long long* fail_min, int num_sms, cudaStream_t stream) {
  using Sh = RegShape<K, M>;
  const size_t smem = sizeof(double) * (Sh::kTabDoubles + 2 * Sh::per_warp(D) * kPairWarps);
  cudaError_t err = cudaFuncSetAttribute(solve_pair_kernel<K, M, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  int per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_pair_kernel<K, M, D>, kPairWarps * kWarp, smem);
  if (err != cudaSuccess) return err;
  if (per_sm < 1) per_sm = 1;
  const int64_t pairs = (nrows + 1) / 2;
  const int64_t need = (pairs + kPairWarps - 1) / kPairWarps;
  const int64_t grid = std::min<int64_t>(need, static_cast<int64_t>(num_sms) * per_sm);
  solve_pair_kernel<K, M, D><<<static_cast<unsigned>(grid), kPairWarps * kWarp, smem, stream>>>(
      X, Y, S, nrows, row_begin, kp, C, fail_min);
  note_launches(1);
  return cudaGetLastError();
}

// CTA shape: 4 warps (one pair table per 4 neighbourhoods in flight), 4 CTAs
// per SM: <= 128 registers per thread, 16 warps per SM.
#ifndef FMGP_REG_WARPS
#define FMGP_REG_WARPS 4
#endif
template <int K, int M>
struct RegLaunch {
  static constexpr int kWarps = FMGP_REG_WARPS;
  static constexpr int kMinBlocks = 16 / kWarps;  // 16 warps/SM at <= 128 registers
};
// FMGP_REG_LOCKSTEP (default 1): the CTA's warps start every row together (a
// CTA barrier per row), so they run the same region of the ~8 k-instruction
// unrolled kernel at the same time. Without it the warps drift apart and, in
// some row orders, miss in the 32 KB instruction cache (cfg5 through
// fmgp_precompute_device: 128.7 -> 111.7 ms with it; the group path
// 110.8 -> 112.2 ms; cfg2 13.45 -> 13.23 ms; profiles/r02/ab_cta_shape.txt).
#ifndef FMGP_REG_LOCKSTEP
#define FMGP_REG_LOCKSTEP 1
#endif

template <int K, int M, int D>
__global__ void __launch_bounds__(RegLaunch<K, M>::kWarps * kWarp, RegLaunch<K, M>::kMinBlocks)
solve_reg_kernel(const double* __restrict__ X, const double* __restrict__ Y, int d, const int32_t* __restrict__ S,
                 int64_t nrows, int64_t row_begin, KParams kp, double* __restrict__ C,
                 unsigned long long* __restrict__ fail_min, int gram_min_d, const int32_t* __restrict__ order) {
  using Sh = RegShape<K, M>;
  extern __shared__ double smem[];
  const int lane = threadIdx.x % kWarp;
  const int warp = threadIdx.x / kWarp;
  const int warps = blockDim.x / kWarp;
  uint32_t* ptab = reinterpret_cast<uint32_t*>(smem);
  __shared__ double s_exp[FMGP_BUILD_TAB_N];
  stage_exp_table(s_exp);
  if constexpr (D > 0) fill_pair_table<K>(ptab);
  __syncthreads();
  double* A = smem + (D > 0 ? Sh::kTabDoubles : 0) + warp * Sh::per_warp(D);
  double* dinv = A + Sh::kAug;
  double* xs = dinv + ((K + 1) & ~1);
  int32_t* sr = reinterpret_cast<int32_t*>(xs + Sh::xs_doubles(D));
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * warps; base < nrows;
       base += static_cast<int64_t>(gridDim.x) * warps) {
    if constexpr (FMGP_REG_LOCKSTEP) __syncthreads();
    const int64_t it = base + warp;
    if (it >= nrows) continue;
    const int64_t r = order != nullptr ? order[it] : it;
    for (int t = lane; t < K; t += kWarp) sr[t] = S[r * K + t];
    __syncwarp();
    bool ok = false;
    for (int attempt = 0; attempt < 4 && !ok; ++attempt) {
      if constexpr (D > 0)
        build_small<K, M, D>(X, Y, sr, kp, attempt, A, xs, ptab, lane, s_exp);
      else
      {
        if constexpr (K <= 32) {
          if (d >= gram_min_d) {
            build_gram<K, M>(X, Y, d, sr, kp, attempt, A, xs, lane);
          } else {
            build_reg<K, M>(X, Y, d, sr, kp, attempt, A, xs, lane);
          }
        } else {
          build_reg<K, M>(X, Y, d, sr, kp, attempt, A, xs, lane);
        }
      }
      ok = factor_reg<K, M>(A, dinv, lane);
      __syncwarp();
    }
    if (!ok) {
      if (lane == 0) atomicMin(fail_min, static_cast<unsigned long long>(row_begin + r));
      __syncwarp();
      continue;
    }
    back_solve_reg<K, M>(A, dinv, C + r * K * M, lane);
    __syncwarp();
  }
}

template <int K, int M, int D>
cudaError_t launch_reg(const double* X, const double* Y, int d, const int32_t* S, int64_t nrows, int64_t row_begin,
                       const KParams& kp, double* C, unsigned long long* fail_min, int num_sms, cudaStream_t stream,
                       const int32_t* order) {
  using Sh = RegShape<K, M>;
  constexpr int kWarps = RegLaunch<K, M>::kWarps;
  const size_t smem = sizeof(double) * ((D > 0 ? Sh::kTabDoubles : 0) + Sh::per_warp(D) * kWarps);
  cudaError_t err = cudaFuncSetAttribute(solve_reg_kernel<K, M, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
  if (err != cudaSuccess) return err;
  int per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_reg_kernel<K, M, D>, kWarps * kWarp, smem);
  if (err != cudaSuccess) return err;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (nrows + kWarps - 1) / kWarps;
  const int64_t grid = std::min<int64_t>(need, static_cast<int64_t>(num_sms) * per_sm);
  static const int gram_min_d = [] {
    const char* e = std::getenv("FMGP_SOLVE_GRAM");
    return (e != nullptr && e[0] == '0') ? INT_MAX : kGramMinD;
  }();
  solve_reg_kernel<K, M, D><<<static_cast<unsigned>(grid), kWarps * kWarp, smem, stream>>>(
      X, Y, d, S, nrows, row_begin, kp, C, fail_min, gram_min_d, order);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace

bool fused_solve_reg_supported(int k, int d, int m) {
  (void)d;
  return (k == 50 && m == 1) || (k == 30 && m == 1) || (k == 30 && m == 10);
}

cudaError_t fused_solve_reg(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                            int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                            int num_sms, cudaStream_t stream, const int32_t* order) {
  if (nrows <= 0) return cudaSuccess;
#define FMGP_REG_CASE(KK, MM, DD) \
  return launch_reg<KK, MM, DD>(X, Y, d, S, nrows, row_begin, kp, C, fail_min, num_sms, stream, order)
  // FMGP_SOLVE_PAIR=1 selects two neighbourhoods per warp for small d (A/B:
  // fewer instructions and shared wavefronts per row, but only 8 warps/SM fit
  // and it is latency-bound: cfg2 solve 14.2 ms vs 13.9 ms for the default)
  static const bool pair = [] {
    const char* e = std::getenv("FMGP_SOLVE_PAIR");
    return e != nullptr && e[0] == '1';
  }();
  if (pair && m == 1 && (d == 2 || d == 3) && (k == 50 || k == 30)) {
    if (k == 50) return d == 2 ? launch_pair<50, 1, 2>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream)
                               : launch_pair<50, 1, 3>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream);
    return d == 2 ? launch_pair<30, 1, 2>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream)
                  : launch_pair<30, 1, 3>(X, Y, S, nrows, row_begin, kp, C, fail_min, num_sms, stream);
  }
  if (k == 50 && m == 1) {
    if (d == 2) FMGP_REG_CASE(50, 1, 2);
    if (d == 3) FMGP_REG_CASE(50, 1, 3);
    FMGP_REG_CASE(50, 1, 0);
  }
  if (k == 30 && m == 1) {
    if (d == 2) FMGP_REG_CASE(30, 1, 2);
    if (d == 3) FMGP_REG_CASE(30, 1, 3);
    FMGP_REG_CASE(30, 1, 0);
  }
  if (k == 30 && m == 10) FMGP_REG_CASE(30, 10, 0);
#undef FMGP_REG_CASE
  return cudaErrorInvalidValue;
}

}  // namespace fmgp
