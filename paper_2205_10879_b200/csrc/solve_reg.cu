// K2-reg — the fused neighbourhood solve with register-resident rows, for
// compile-time neighbourhood sizes (the BASELINE shapes k in {30, 50}).
// Same contract as solve.cu (fast_predict.cpp:98-106, kernel.cpp:106-119,
// linalg.cpp:10-36), one warp per neighbourhood.
//
// Why: the shared-memory left-looking kernel is bound by the LSU pipe (one
// per-lane 64-bit load per FMA). Here lane l owns rows l and l+32 of the
// augmented matrix [K ; Y^T] for the whole factorisation, in registers
// (static indexing: K and M are template parameters and both loops are fully
// unrolled). Column j needs only the pivot row L_j., which its owner writes to
// shared memory as it is produced and every lane reads as a 128-bit
// broadcast. The RHS rows (K .. K+M-1) ride along, so the column sweep also
// performs the forward substitution; the backward solve then runs over the
// shared-memory copy of L.
#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

__constant__ double kJitR[4] = {0.0, 1e-10, 1e-8, 1e-6};

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
  static constexpr bool kTwo = kRows > 32;  // two row slots per lane?
  // Rows are paired head-to-tail: lane l owns row l (slot 0) and row kRows-1-l
  // (slot 1), so slot 0 (the short rows) is finished after column kN0 - 1 and
  // both slots stay busy until then; one slot: lane l owns row l.
  static constexpr int kN0 = kTwo ? (kRows + 1) / 2 : K;  // slot-0 rows 0 .. kN0-1 (their entries < kN0)
  static constexpr int kDch = 16;                      // coordinate slice width staged per pass
  static constexpr int kXsStride = kDch + 2;           // = 2 mod 4 doubles: conflict-light 128-bit row loads
  static constexpr int kCol = (K + 2) & ~1;            // colbuf (even: 16-byte aligned pairs)
  // xs holds K x D coordinates for the small-d build (D > 0), K x kXsStride slices otherwise
  __host__ __device__ static constexpr int xs_doubles(int D) { return D > 0 ? ((K * D + 1) & ~1) : kXsStride * K; }
  __host__ __device__ static constexpr int per_warp(int D) {
    return ((kAug + ((K + 1) & ~1) /*dinv*/ + kCol + xs_doubles(D) + (K + 1) / 2 + 2) + 1) & ~1;
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

template <int K, int D, int KF>
__device__ __forceinline__ void pair_loop(const double* xs, const uint32_t* ptab, const KParams& kp, double* A,
                                          int lane) {
  constexpr int npairs = (K * (K - 1)) / 2;
#pragma unroll 2
  for (int e = lane; e < npairs; e += kWarp) {
    const uint32_t t = ptab[e];
    const double* xa = xs + ((t >> 8) & 0xffu) * D;
    const double* xb = xs + (t & 0xffu) * D;
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double dd = __dsub_rn(xa[c], xb[c]);
      acc = __dadd_rn(acc, __dmul_rn(dd, dd));
    }
    A[t >> 16] = kernel_from_sq<KF>(acc, kp);
  }
}

// Small-d build (d = D known at compile time): all K coordinates staged once,
// one pair per lane per step from the pair table, no index decode.
template <int K, int M, int D>
__device__ void build_small(const double* __restrict__ X, const double* __restrict__ Y, const int32_t* sr,
                            const KParams& kp, int attempt, double* A, double* xs, const uint32_t* ptab, int lane) {
  using Sh = RegShape<K, M>;
  for (int e = lane; e < K * D; e += kWarp) {
    const int t = e / D, c = e - t * D;
    xs[e] = X[static_cast<int64_t>(sr[t]) * D + c];
  }
  __syncwarp();
  switch (kernel_code(kp)) {  // uniform: one pair loop per kernel kind, no per-pair dispatch
    case 0: pair_loop<K, D, 0>(xs, ptab, kp, A, lane); break;
    case 1: pair_loop<K, D, 1>(xs, ptab, kp, A, lane); break;
    case 2: pair_loop<K, D, 2>(xs, ptab, kp, A, lane); break;
    case 3: pair_loop<K, D, 3>(xs, ptab, kp, A, lane); break;
    default: pair_loop<K, D, 4>(xs, ptab, kp, A, lane); break;
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

// Register-resident left-looking factorisation of the augmented matrix:
// column j of the lane's rows accumulates a_rj - sum_{p<j} a_rp L_jp from its
// registers and the pivot row L_j. broadcast from shared memory (128-bit).
// Returns false at the first pivot <= 0 (Eigen LLT semantics).
template <int K, int M>
__device__ bool factor_reg(double* A, double* dinv, double* colbuf, int lane) {
  (void)colbuf;
  using Sh = RegShape<K, M>;
  constexpr int kRows = Sh::kRows;
  const int r0 = lane, r1 = kRows - 1 - lane;
  const bool has0 = Sh::kTwo ? r0 < Sh::kN0 : r0 < kRows;
  const bool has1 = Sh::kTwo && lane < kRows - Sh::kN0;
  double a0[Sh::kN0];
  double a1[Sh::kTwo ? K : 1];
  // Slot-1 entries p >= kN0 are loaded only when column kN0 starts (they are
  // still the original values in shared memory then): their registers reuse
  // the dead slot-0 rows, which keeps the peak register count down.
  const double* R1 = A + Sh::row_off(has1 ? r1 : 0);
  {
    const double* R0 = A + Sh::row_off(has0 ? r0 : 0);
#pragma unroll
    for (int p = 0; p < Sh::kN0; ++p) a0[p] = (has0 && (p <= r0 || r0 >= K)) ? R0[p] : 0.0;
    if constexpr (Sh::kTwo) {
#pragma unroll
      for (int p = 0; p < Sh::kN0; ++p) a1[p] = (has1 && (p <= r1 || r1 >= K)) ? R1[p] : 0.0;
    }
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if constexpr (Sh::kTwo) {
      if (j == Sh::kN0) {
#pragma unroll
        for (int p = Sh::kN0; p < K; ++p) a1[p] = (has1 && (p <= r1 || r1 >= K)) ? R1[p] : 0.0;
      }
    }
    const double* Lj = A + ro_r(j);  // pivot row j (entries < j are final)
    // four independent accumulators per row slot (DFMA latency chains of j/4)
    double s0a = 0.0, s0b = 0.0, s0c = 0.0, s0d = 0.0, s1a = 0.0, s1b = 0.0, s1c = 0.0, s1d = 0.0;
    if (j < Sh::kN0) s0a = a0[j < Sh::kN0 ? j : 0];
    if constexpr (Sh::kTwo) s1a = a1[j];
#pragma unroll
    for (int p = 0; p + 3 < j; p += 4) {
      const double2 l = *reinterpret_cast<const double2*>(Lj + p);
      const double2 m = *reinterpret_cast<const double2*>(Lj + p + 2);
      if (j < Sh::kN0) {
        s0a = fma(-a0[p], l.x, s0a);
        s0b = fma(-a0[p + 1], l.y, s0b);
        s0c = fma(-a0[p + 2], m.x, s0c);
        s0d = fma(-a0[p + 3], m.y, s0d);
      }
      if constexpr (Sh::kTwo) {
        s1a = fma(-a1[p], l.x, s1a);
        s1b = fma(-a1[p + 1], l.y, s1b);
        s1c = fma(-a1[p + 2], m.x, s1c);
        s1d = fma(-a1[p + 3], m.y, s1d);
      }
    }
    {  // up to three leftover columns (j is a compile-time constant here)
      const int p0 = j & ~3;
      if ((j & 3) >= 1) {
        const double l = Lj[p0];
        if (j < Sh::kN0) s0a = fma(-a0[p0 < Sh::kN0 ? p0 : 0], l, s0a);
        if constexpr (Sh::kTwo) s1a = fma(-a1[p0], l, s1a);
      }
      if ((j & 3) >= 2) {
        const double l = Lj[p0 + 1];
        if (j < Sh::kN0) s0b = fma(-a0[(p0 + 1) < Sh::kN0 ? p0 + 1 : 0], l, s0b);
        if constexpr (Sh::kTwo) s1b = fma(-a1[p0 + 1], l, s1b);
      }
      if ((j & 3) >= 3) {
        const double l = Lj[p0 + 2];
        if (j < Sh::kN0) s0c = fma(-a0[(p0 + 2) < Sh::kN0 ? p0 + 2 : 0], l, s0c);
        if constexpr (Sh::kTwo) s1c = fma(-a1[p0 + 2], l, s1c);
      }
    }
    const double s0 = (s0a + s0b) + (s0c + s0d), s1 = (s1a + s1b) + (s1c + s1d);
    const double mine = j < Sh::kN0 ? s0 : s1;
    const double piv = __shfl_sync(0xffffffffu, mine, j < Sh::kN0 ? j : kRows - 1 - j);
    if (!(piv > 0.0)) return false;
    const double inv = rsqrt(piv);  // 1/L_jj and L_jj = piv/L_jj from one reciprocal square root
    const double ljj = piv * inv;
    if (j < Sh::kN0) {
      if (has0 && r0 >= j) {
        const double v = r0 == j ? ljj : s0 * inv;
        a0[j < Sh::kN0 ? j : 0] = v;
        A[Sh::row_off(r0) + j] = v;
      }
    }
    if constexpr (Sh::kTwo) {
      if (has1 && r1 >= j) {
        const double v = r1 == j ? ljj : s1 * inv;
        a1[j] = v;
        A[Sh::row_off(r1) + j] = v;
      }
    }
    if (lane == 0) dinv[j] = inv;
    __syncwarp();
  }
  return true;
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

template <int K, int M, int D>
__global__ void __launch_bounds__(64, K <= 32 ? 8 : 6)
solve_reg_kernel(const double* __restrict__ X, const double* __restrict__ Y, int d, const int32_t* __restrict__ S,
                 int64_t nrows, int64_t row_begin, KParams kp, double* __restrict__ C,
                 unsigned long long* __restrict__ fail_min) {
  using Sh = RegShape<K, M>;
  extern __shared__ double smem[];
  const int lane = threadIdx.x % kWarp;
  const int warp = threadIdx.x / kWarp;
  const int warps = blockDim.x / kWarp;
  uint32_t* ptab = reinterpret_cast<uint32_t*>(smem);
  if constexpr (D > 0) {
    fill_pair_table<K>(ptab);
    __syncthreads();
  }
  double* A = smem + (D > 0 ? Sh::kTabDoubles : 0) + warp * Sh::per_warp(D);
  double* dinv = A + Sh::kAug;
  double* colbuf = dinv + ((K + 1) & ~1);
  double* xs = colbuf + Sh::kCol;
  int32_t* sr = reinterpret_cast<int32_t*>(xs + Sh::xs_doubles(D));
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * warps + warp; r < nrows;
       r += static_cast<int64_t>(gridDim.x) * warps) {
    for (int t = lane; t < K; t += kWarp) sr[t] = S[r * K + t];
    __syncwarp();
    bool ok = false;
    for (int attempt = 0; attempt < 4 && !ok; ++attempt) {
      if constexpr (D > 0)
        build_small<K, M, D>(X, Y, sr, kp, attempt, A, xs, ptab, lane);
      else
        build_reg<K, M>(X, Y, d, sr, kp, attempt, A, xs, lane);
      ok = factor_reg<K, M>(A, dinv, colbuf, lane);
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
                       const KParams& kp, double* C, unsigned long long* fail_min, int num_sms, cudaStream_t stream) {
  using Sh = RegShape<K, M>;
  constexpr int kWarps = 2;
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
  solve_reg_kernel<K, M, D><<<static_cast<unsigned>(grid), kWarps * kWarp, smem, stream>>>(X, Y, d, S, nrows, row_begin,
                                                                                        kp, C, fail_min);
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
                            int num_sms, cudaStream_t stream) {
  if (nrows <= 0) return cudaSuccess;
#define FMGP_REG_CASE(KK, MM, DD) \
  return launch_reg<KK, MM, DD>(X, Y, d, S, nrows, row_begin, kp, C, fail_min, num_sms, stream)
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
