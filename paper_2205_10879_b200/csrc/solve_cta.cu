// K2-cta — the fused neighbourhood solve for large compile-time k (cfg4:
// k = 100), one thread block per neighbourhood. Same contract as solve.cu
// (fast_predict.cpp:98-106 gather, kernel.cpp:106-119 nugget-regularised
// matrix, linalg.cpp:10-36 jitter-ladder LLT + solve).
//
// Why: the warp-per-neighbourhood kernels keep a whole k x k triangle per
// warp; at k = 100 that is ~46 KB of shared memory per warp (4 warps per SM,
// latency-bound). Here the CTA's R = K + M threads own one row each of the
// augmented matrix [K ; Y^T] in registers:
//  * build: all K neighbour coordinates are staged once in shared memory
//    (padded rows); for d >= 16 the squared distances come from a Gram matrix
//    on the FP64 tensor cores (cta_gram: DMMA m8n8k4 over the 8 x 8 tiles of
//    the lower triangle, coordinates centred at the neighbourhood's own point,
//    exact recompute of near-duplicates), otherwise the strict lower triangle
//    is spread over the CTA through a pair table; entries land in a packed
//    row-major triangle;
//  * factor: left-looking column sweep. For column j every row r > j forms
//    s_r = a_rj - sum_{p<j} a_rp L_jp from its registers and the pivot row
//    L_j. (a shared-memory 128-bit broadcast); the rows also keep a running
//    diagonal d_r = a_rr - sum_p L_rp^2, so the owner of row j+1 has its pivot
//    as soon as it has L_{j+1,j}: one barrier per column. The RHS rows ride
//    along (forward substitution);
//  * backward solve: warp 0, x in registers, x_j broadcast by shuffle.
#include <cstdlib>

#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

__constant__ double kJitC[4] = {0.0, 1e-10, 1e-8, 1e-6};

__host__ __device__ constexpr int ro_c(int i) { return ((i * (i + 1)) >> 1) + ((i + 1) >> 1); }  // 16 B aligned rows

template <int K, int M>
struct CtaShape {
  static constexpr int kRows = K + M;
  static constexpr int kThreads = ((kRows + 31) / 32) * 32;
  static constexpr int kTri = ro_c(K);                        // packed triangle (doubles)
  static constexpr int kPairs = K * (K - 1) / 2;
  static constexpr int kXsD = 48;                             // coordinate slice staged per pass
  static constexpr int kXsStride = kXsD + 2;  // = 2 mod 4 doubles: 128-bit loads of 8 lanes on distinct bank groups
  // Gram build (d >= 16): rows of kXsD + 4 doubles (= 4 mod 16: the DMMA fragment load of lane (g, t),
  // row 8 I + g, column 4 c + t, touches every 8-byte bank pair exactly twice: two wavefronts for 32 doubles)
  static constexpr int kGsStride = kXsD + 4;
  static constexpr int kXs = ((K * kGsStride + 1) / 2) * 2;
  static constexpr int kNB = (K + 7) / 8;  // 8-row blocks of the Gram matrix
  // doubles: tri | xs | invd[K] | zbuf[M*K] | nrm[K] | misc[2]; then uint32 pairs, int32 sr
  static constexpr int kDoubles = kTri + kXs + ((K + 1) & ~1) + ((M * K + 1) & ~1) + ((K + 1) & ~1) + 2;
  static constexpr size_t kBytes = sizeof(double) * kDoubles + sizeof(uint32_t) * kPairs + sizeof(int32_t) * K;
};

__device__ __forceinline__ double jitter_c(double v, int a) {
  for (int t = 1; t <= a; ++t) v = __dadd_rn(v, __dsub_rn(kJitC[t], kJitC[t - 1]));
  return v;
}

// Pairs of the strict lower triangle over this CTA, distances accumulated over
// coordinate slices in t order; the last slice turns them into kernel values.
template <int K, int M, int KF>
__device__ __forceinline__ void cta_pairs(const double* xs, const uint32_t* ptab, const KParams& kp, double* tri,
                                          int c0, int dc, int tid) {
  using Sh = CtaShape<K, M>;
  for (int e = tid; e < Sh::kPairs; e += Sh::kThreads) {
    const uint32_t pt = ptab[e];
    const double* xa = xs + ((pt >> 8) & 0xffu) * Sh::kXsStride;
    const double* xb = xs + (pt & 0xffu) * Sh::kXsStride;
    double acc = c0 == 0 ? 0.0 : tri[pt >> 16];
    int c = 0;
#pragma unroll 4
    for (; c + 1 < dc; c += 2) {  // t-ordered, fused multiply-add (matrix entries within ~1 ulp)
      const double2 u = *reinterpret_cast<const double2*>(xa + c);
      const double2 w = *reinterpret_cast<const double2*>(xb + c);
      const double e0 = u.x - w.x, e1 = u.y - w.y;
      acc = fma(e0, e0, acc);
      acc = fma(e1, e1, acc);
    }
    if (c < dc) {
      const double e0 = xa[c] - xb[c];
      acc = fma(e0, e0, acc);
    }
    if constexpr (KF < 0) tri[pt >> 16] = acc;
    else tri[pt >> 16] = kernel_from_sq<KF>(acc, kp);
  }
}

// 1/sqrt(x) for a pivot x > 0: MUFU seed (~2^-22) and one third-order step (as solve_dm.cu's rsqrt_pivot3:
// four dependent FP64 operations; the pivot chain is the serial part of the panel)
__device__ __forceinline__ double rsqrt_pivot3_c(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(x * y), y, 1.0);
  return fma(y * e, fma(e, 0.375, 0.5), y);
}

__device__ __forceinline__ void dmma_c(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// Gram build of one coordinate slice (d >= 16; cfg4: d = 40, one slice): the squared distances of
// the neighbourhood come from G = Xc Xc^T on the FP64 tensor cores, Xc = the staged coordinates
// centred at the neighbourhood's own point (row 0), so |x|^2 is of the order of the distances and
// d^2 = |a|^2 + |b|^2 - 2 a.b keeps its digits. The 8 x 8 tiles of the lower triangle are dealt
// over the CTA's warps; lane (g, t) holds Xc[8 I + g][4 c + t], which is the A fragment of row
// block I and the B fragment of row block J alike. Partial sums of G (and of the norms) go through
// the packed triangle between slices; the last slice turns them into kernel values. A pair with
// d^2 <= 1e-12 (|a|^2 + |b|^2) is recomputed as the exact sum of squared differences, so exact
// duplicates keep the nugget bit for bit (kernel.cpp:58-60, :81-83). The direct difference loop
// this replaces took ~25 k of the kernel's ~75 k warp instructions per neighbourhood at cfg4.
template <int K, int M, int KF, bool LEAN>
__device__ __forceinline__ void cta_gram(const double* gs, const double* nrm, const KParams& kp, double* tri, int c0,
                                         int dc4, int tid, bool last, int gst, const double* __restrict__ X,
                                         const int32_t* sr, int d) {
  using Sh = CtaShape<K, M>;
  constexpr int NB = Sh::kNB;
  constexpr int NT = NB * (NB + 1) / 2;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  // tile e = I (I + 1) / 2 + J, J <= I; a warp's tiles are NW apart, so (I, J) advance incrementally.
  // kG tiles per step: kG independent DMMA chains, then their 2 kG entries per lane go through the
  // kernel evaluation together (independent sqrt / exp chains).
  constexpr int NW = Sh::kThreads / 32;
  constexpr int kG = 3;
  int I = 0, J = warp;
  for (int e0 = warp; e0 < NT; e0 += kG * NW) {
    const double* pa[kG];
    const double* pb[kG];
    int ra[kG], col[kG];
    double acc[kG][2];
#pragma unroll
    for (int i = 0; i < kG; ++i) {
      while (J > I) {
        J -= I + 1;
        ++I;
      }
      const bool tv = e0 + i * NW < NT;  // past the last tile: row block 0 again, nothing stored
      const int Ii = tv ? I : 0, Ji = tv ? J : 0;
      const int rb = 8 * Ji + g;
      ra[i] = tv ? 8 * Ii + g : K;
      col[i] = 8 * Ji + 2 * t;
      // rows past K read row 0: what they produce (rows >= K of the tile, columns >= K > ra) is never stored
      pa[i] = gs + (ra[i] < K ? ra[i] : 0) * gst + t;
      pb[i] = gs + (rb < K ? rb : 0) * gst + t;
      acc[i][0] = 0.0;
      acc[i][1] = 0.0;
      J += NW;
    }
#pragma unroll 2
    for (int c = 0; c < dc4; c += 4) {
#pragma unroll
      for (int i = 0; i < kG; ++i) dmma_c(acc[i], pa[i][c], pb[i][c]);
    }
    // accumulator layout: row 8 I + g, columns 8 J + 2 t, + 1; strict lower triangle only (the diagonal is
    // set with the jitter rung)
    double* out[kG][2];
    bool st[kG][2];
    double val[kG][2];
#pragma unroll
    for (int i = 0; i < kG; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cc = col[i] + h;
        st[i][h] = ra[i] < K && cc < ra[i];
        out[i][h] = tri + (st[i][h] ? ro_c(ra[i]) + cc : 0);
        double gsum = acc[i][h];
        if (c0 != 0 && st[i][h]) gsum += *out[i][h];
        val[i][h] = gsum;
      }
    if (last) {
#pragma unroll
      for (int i = 0; i < kG; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cc = col[i] + h;
          const double na = nrm[st[i][h] ? ra[i] : 0], nb = nrm[st[i][h] ? cc : 0];
          double d2 = fma(-2.0, val[i][h], na + nb);
          if (st[i][h] && !(d2 > 1e-12 * (na + nb))) {  // (near-)duplicate: exact differences (the full-footprint
            d2 = 0.0;  // layout holds every dimension when d <= kXsD; for wider rows the earlier slices are gone: clamp)
            if constexpr (LEAN) {  // lean layout: narrow slices, so the differences come from global memory
              const double* xa = X + static_cast<int64_t>(sr[ra[i]]) * d;
              const double* xb = X + static_cast<int64_t>(sr[cc]) * d;
              for (int c = 0; c < d; ++c) {
                const double df = xa[c] - xb[c];
                d2 = fma(df, df, d2);
              }
            } else if (c0 == 0) {
              const double* xa = gs + ra[i] * gst;
              const double* xb = gs + cc * gst;
              for (int c = 0; c < dc4; ++c) {
                const double df = xa[c] - xb[c];
                d2 = fma(df, df, d2);
              }
            }
          }
          val[i][h] = kernel_from_sq<KF>(st[i][h] ? d2 : 1.0, kp);
        }
    }
#pragma unroll
    for (int i = 0; i < kG; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (st[i][h]) *out[i][h] = val[i][h];
  }
}

// Blocked factorisation in shared memory (M == 1; FMGP_CTA_BLOCKED=0 selects the row-per-thread
// sweep below): the augmented matrix [K ; y^T] (row K = the RHS, kept in zbuf, so the
// factorisation also does the forward substitution) is blocked 8 x 8 and factored left-looking
// by block column J, in place in the packed triangle:
//   1. update: tile (I, J) -= sum_{Q < 2J} F(I, Q) F(J, Q)^T on the FP64 tensor cores (DMMA
//      m8n8k4), tiles dealt over the CTA's warps; F(I, Q) = lane (g, t) holding
//      L[8I+g][4Q+t], read from the triangle; the (negated) fragments of row block J stay in
//      registers for all of a warp's tiles;
//   2. panel: thread i takes row 8J + i (down to the RHS row). Every thread factors the 8 x 8
//      diagonal block itself, in registers (36 broadcast loads, no shuffles, no barrier between
//      the pivots), then solves its own row against it and writes its 8 entries back.
// Two barriers per block column (26 instead of the 100 of the column sweep), and the k^3/6
// multiply-adds leave the scalar FP64 path with its shared-memory broadcasts.
template <int K>
__device__ __forceinline__ double* cta_row(double* tri, double* zrow, int r) { return r < K ? tri + ro_c(r) : zrow; }

template <int K, int M>
__device__ __forceinline__ void cta_factor_blocked(double* tri, double* zrow, double* invd, double* misc, int tid) {
  using Sh = CtaShape<K, M>;
  constexpr int NBC = (K + 7) / 8;      // column blocks
  constexpr int NBR = (K + 1 + 7) / 8;  // row blocks (rows 0 .. K; row K = RHS)
  constexpr int NW = Sh::kThreads / 32;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
#pragma unroll 1
  for (int J = 0; J < NBC; ++J) {
    const int c0 = 8 * J;
    if (J > 0) {
      // 1. update of block column J
      // The warp's tiles I = J + warp + NW i (at most kTW of them) are updated together: per k-step one
      // B fragment and kTW independent DMMA chains. Rows past the matrix read row 0 (rows > K of a
      // tile and columns >= K of the block column are never stored), so no operand needs zeroing.
      constexpr int kTW = (NBR - 1 + NW - 1) / NW;
      const int rb = c0 + g;  // the tile's column index this lane's B fragment belongs to
      const double* pb = tri + ro_c(rb < K ? rb : 0) + t;
      const int cc = c0 + 2 * t;
      double acc[kTW][2];
      double* prow[kTW];
      bool st0[kTW], st1[kTW];
#pragma unroll
      for (int i = 0; i < kTW; ++i) {
        const int I = J + warp + NW * i;
        const int ra = 8 * I + g;
        const bool rok = I < NBR && ra <= K;
        prow[i] = cta_row<K>(tri, zrow, rok ? ra : 0);
        const int lim = ra < K ? ra + 1 : K;  // columns < lim exist in row ra
        st0[i] = rok && cc < lim;
        st1[i] = rok && cc + 1 < lim;
        acc[i][0] = st0[i] ? prow[i][cc] : 0.0;
        acc[i][1] = st1[i] ? prow[i][cc + 1] : 0.0;
      }
      static_assert(kTW <= 3, "tile-count dispatch below");
      const int ntw = (NBR - J - warp + NW - 1) / NW;  // this warp's tiles (warp-uniform)
      if (ntw >= 3) {
#pragma unroll 2
        for (int Q = 0; Q < 2 * J; ++Q) {
          const double b = -pb[4 * Q];
#pragma unroll
          for (int i = 0; i < kTW; ++i) dmma_c(acc[i], prow[i][4 * Q + t], b);
        }
      } else if (ntw == 2) {
#pragma unroll 2
        for (int Q = 0; Q < 2 * J; ++Q) {
          const double b = -pb[4 * Q];
#pragma unroll
          for (int i = 0; i < (kTW < 2 ? kTW : 2); ++i) dmma_c(acc[i], prow[i][4 * Q + t], b);
        }
      } else if (ntw == 1) {
#pragma unroll 4
        for (int Q = 0; Q < 2 * J; ++Q) dmma_c(acc[0], prow[0][4 * Q + t], -pb[4 * Q]);
      }
#pragma unroll
      for (int i = 0; i < kTW; ++i) {
        if (st0[i]) prow[i][cc] = acc[i][0];
        if (st1[i]) prow[i][cc + 1] = acc[i][1];
      }
      __syncthreads();
    }
    // 2. panel: every thread factors the diagonal block, then solves its own row (a warp whose 32 rows are
    // all past the RHS row has nothing to solve and skips the block too)
    const int nc = K - c0 < 8 ? K - c0 : 8;
    const int r = c0 + tid;
    double x[8];
    if (c0 + 32 * warp <= K) {
    double dblk[8][8];
    double inv[8];
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int c = 0; c <= i; ++c) dblk[i][c] = i < nc ? tri[ro_c(i < nc ? c0 + i : c0) + c0 + c] : (i == c ? 1.0 : 0.0);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double piv = dblk[c][c];
      bad = bad || !(piv > 0.0);
      inv[c] = rsqrt_pivot3_c(piv);
      dblk[c][c] = piv * inv[c];
#pragma unroll
      for (int i = c + 1; i < 8; ++i) dblk[i][c] *= inv[c];
#pragma unroll
      for (int i = c + 1; i < 8; ++i)
#pragma unroll
        for (int c2 = c + 1; c2 <= i; ++c2) dblk[i][c2] = fma(-dblk[i][c], dblk[c2][c], dblk[i][c2]);
    }
    if (r <= K) {
      double* prow = cta_row<K>(tri, zrow, r);
      if (tid < 8) {  // a row of the diagonal block: its factor row (tid < nc here: r <= K and r < c0 + 8)
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i == tid)
#pragma unroll
            for (int c = 0; c <= i; ++c) x[c] = dblk[i][c];
        // written back after the barrier below: the other warps may still be reading the unfactored block
      }
      if (tid >= 8 || r == K) {  // a row below the block (or the RHS row inside the last block's span)
#pragma unroll
        for (int c = 0; c < 8; ++c) x[c] = c < nc ? prow[c0 + c] : 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {  // right-looking: two dependent operations per column
          x[c] *= inv[c];
#pragma unroll
          for (int c2 = c + 1; c2 < 8; ++c2) x[c2] = fma(-x[c], dblk[c2][c], x[c2]);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < nc) prow[c0 + c] = x[c];
      }
    }
    if (tid == 0) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < nc) invd[c0 + c] = inv[c];
      if (bad) misc[0] = 1.0;
    }
    }  // warps with rows
    __syncthreads();
    // The factor rows of the diagonal block go in place only now: every thread loaded the unfactored block
    // at the top of the panel without a barrier of its own, and no later block column reads these rows
    // (left-looking: block column J' > J touches rows >= 8 J' only) until the backward solve.
    if (tid < 8 && r < K) {
      double* prow = tri + ro_c(r);
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c <= tid) prow[c0 + c] = x[c];
    }
  }
}

#ifndef FMGP_CTA_LEAN_MINB  // CTAs per SM the lean kernel's registers are bounded for
#define FMGP_CTA_LEAN_MINB 4
#endif

// LEAN (M == 1, Gram build + blocked factorisation, 16 <= d <= kXsD — cfg4): the same arithmetic with
// a smaller footprint, so that more than two neighbourhoods are resident per SM (the kernel is bound
// by the latency of its barriers and pivot chains, not by a pipe): no pair table, the coordinates
// staged in narrow slices of `xsd` dimensions (rows of `gst` doubles; partial Gram sums go through the
// triangle), and the row-per-thread sweep (100 doubles of registers per thread) compiled out.
template <int K, int M, bool LEAN>
__global__ void __launch_bounds__(CtaShape<K, M>::kThreads, LEAN ? FMGP_CTA_LEAN_MINB : 1)
solve_cta_kernel(const double* __restrict__ X, const double* __restrict__ Y, int d, const int32_t* __restrict__ S,
                 int64_t nrows, int64_t row_begin, KParams kp, double* __restrict__ C,
                 unsigned long long* __restrict__ fail_min, int use_gram, int xsd, int gst_arg) {
  using Sh = CtaShape<K, M>;
  extern __shared__ double smem[];
  const int W = LEAN ? xsd : Sh::kXsD;             // dimensions staged per slice
  const int gst = LEAN ? gst_arg : Sh::kGsStride;  // doubles per staged row (Gram build)
  double* tri = smem;
  double* xs = tri + Sh::kTri;
  double* invd = xs + (LEAN ? ((K * gst + 1) & ~1) : Sh::kXs);
  double* zbuf = invd + ((K + 1) & ~1);
  double* nrm = zbuf + ((M * K + 1) & ~1);  // Gram build: |x - x_0|^2 per neighbour
  double* misc = nrm + ((K + 1) & ~1);      // [0] = failure flag
  uint32_t* ptab = reinterpret_cast<uint32_t*>(misc + 2);
  int32_t* sr = reinterpret_cast<int32_t*>(ptab + (LEAN ? 0 : Sh::kPairs));
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

  for (int e = tid; !LEAN && e < Sh::kPairs; e += Sh::kThreads) {
    int i = static_cast<int>((1.0f + sqrtf(1.0f + 8.0f * static_cast<float>(e))) * 0.5f);
    while ((i * (i - 1)) / 2 > e) --i;
    while ((i * (i + 1)) / 2 <= e) ++i;
    const int p = e - (i * (i - 1)) / 2;
    ptab[e] = (static_cast<uint32_t>(ro_c(i) + p) << 16) | (static_cast<uint32_t>(i) << 8) | static_cast<uint32_t>(p);
  }

  // LEAN: thread t < K carries entry t of the NEXT neighbourhood's index row in a register (loaded one
  // neighbourhood ahead), so the row is in shared memory without a DRAM round trip, and that
  // neighbourhood's coordinate rows are prefetched into L2 once the current build is done.
  int32_t s_next = -1;
  if (LEAN && tid < K && static_cast<int64_t>(blockIdx.x) < nrows) s_next = S[static_cast<int64_t>(blockIdx.x) * K + tid];
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    __syncthreads();  // previous neighbourhood fully consumed
    bool prefetch_due = false;
    if constexpr (LEAN) {
      if (tid < K) {
        sr[tid] = s_next;
        prefetch_due = r + gridDim.x < nrows;
        if (prefetch_due) s_next = S[(r + gridDim.x) * K + tid];
      }
    } else {
      for (int t = tid; t < K; t += Sh::kThreads) sr[t] = S[r * K + t];
    }
    __syncthreads();
    double y_mine = 0.0;  // this thread's response, in flight during the build
    if (LEAN && tid < K) y_mine = Y[static_cast<int64_t>(sr[tid]) * M];
    bool ok = false;
    for (int attempt = 0; attempt < 4 && !ok; ++attempt) {
      // ---- build K(S_r) into the packed triangle (sequential-in-t distance)
      // one slice only (d <= kXsD): the exact recompute of near-duplicates needs every dimension staged
      const bool gram = LEAN || ((use_gram & 1) && d >= 16 && d <= Sh::kXsD);
      for (int c0 = 0; gram && c0 < d; c0 += W) {
        const int dc = min(W, d - c0), dc4 = (dc + 3) & ~3;
        const double* x0 = X + static_cast<int64_t>(sr[0]) * d + c0;  // centre: the neighbourhood's own point
        {  // 8, 16 or 32 threads per neighbour row (dc4 <= 48: at most two columns per thread)
          const int sh = dc4 <= 8 ? 3 : (dc4 <= 16 ? 4 : 5);
          const int cl = tid & ((1 << sh) - 1);
          const int rpp = Sh::kThreads >> sh;  // rows per pass of the CTA
          const int ca = cl, cb = cl + (1 << sh);
          const double x0a = ca < dc ? x0[ca] : 0.0, x0b = cb < dc ? x0[cb] : 0.0;
          constexpr int RB = LEAN ? 13 : 2;  // rows in flight per thread: the gather is a chain of L2 / DRAM round trips otherwise
          for (int tb = tid >> sh; tb < K; tb += RB * rpp) {
            double va[RB], vb[RB];
#pragma unroll
            for (int i = 0; i < RB; ++i) {
              const int t = tb + i * rpp;
              const double* xr = X + static_cast<int64_t>(sr[t < K ? t : 0]) * d + c0;
              va[i] = ca < dc ? xr[ca] : 0.0;
              vb[i] = cb < dc ? xr[cb] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < RB; ++i) {
              const int t = tb + i * rpp;
              if (t < K) {
                if (ca < dc4) xs[t * gst + ca] = va[i] - x0a;
                if (cb < dc4) xs[t * gst + cb] = vb[i] - x0b;
              }
            }
          }
        }
        __syncthreads();
        if (tid < K) {
          double nn = c0 == 0 ? 0.0 : nrm[tid];
          const double* xr = xs + tid * gst;
          for (int c = 0; c < dc4; ++c) nn = fma(xr[c], xr[c], nn);
          nrm[tid] = nn;
        }
        __syncthreads();
        const bool last = c0 + dc >= d;
        switch (last ? kernel_code(kp) : 0) {  // uniform; the kind only matters in the last slice
          case 0: cta_gram<K, M, 0, LEAN>(xs, nrm, kp, tri, c0, dc4, tid, last, gst, X, sr, d); break;
          case 1: cta_gram<K, M, 1, LEAN>(xs, nrm, kp, tri, c0, dc4, tid, last, gst, X, sr, d); break;
          case 2: cta_gram<K, M, 2, LEAN>(xs, nrm, kp, tri, c0, dc4, tid, last, gst, X, sr, d); break;
          case 3: cta_gram<K, M, 3, LEAN>(xs, nrm, kp, tri, c0, dc4, tid, last, gst, X, sr, d); break;
          default: cta_gram<K, M, 4, LEAN>(xs, nrm, kp, tri, c0, dc4, tid, last, gst, X, sr, d); break;
        }
        __syncthreads();
      }
      for (int c0 = 0; !LEAN && !gram && c0 < d; c0 += Sh::kXsD) {
        const int dc = min(Sh::kXsD, d - c0);
        for (int e = tid; e < K * dc; e += Sh::kThreads) {
          const int t = e / dc, c = e - t * dc;
          xs[t * Sh::kXsStride + c] = X[static_cast<int64_t>(sr[t]) * d + c0 + c];
        }
        __syncthreads();
        const int kf = c0 + dc >= d ? kernel_code(kp) : -1;  // -1: partial sums only
        switch (kf) {  // uniform: one pair loop per kernel kind
          case -1: cta_pairs<K, M, -1>(xs, ptab, kp, tri, c0, dc, tid); break;
          case 0: cta_pairs<K, M, 0>(xs, ptab, kp, tri, c0, dc, tid); break;
          case 1: cta_pairs<K, M, 1>(xs, ptab, kp, tri, c0, dc, tid); break;
          case 2: cta_pairs<K, M, 2>(xs, ptab, kp, tri, c0, dc, tid); break;
          case 3: cta_pairs<K, M, 3>(xs, ptab, kp, tri, c0, dc, tid); break;
          default: cta_pairs<K, M, 4>(xs, ptab, kp, tri, c0, dc, tid); break;
        }
        __syncthreads();
      }
      const double dg = jitter_c(kp.diag, attempt);
      if (LEAN && prefetch_due) {  // (X is far larger than L2 at cfg4: the staging gather would wait on DRAM)
        const char* px = reinterpret_cast<const char*>(X + static_cast<int64_t>(s_next) * d);
        for (int o = 0; o < d * 8; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(px + o));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(Y + static_cast<int64_t>(s_next) * M));
        prefetch_due = false;
      }
      if (LEAN || (M == 1 && (use_gram & 2))) {
        // ---- blocked DMMA factorisation in shared memory (cta_factor_blocked)
        if (tid < K) {
          tri[ro_c(tid) + tid] = dg;
          zbuf[tid] = LEAN ? y_mine : Y[static_cast<int64_t>(sr[tid]) * M];
        }
        if (tid == 0) misc[0] = 0.0;
        __syncthreads();
        cta_factor_blocked<K, M>(tri, zbuf, invd, misc, tid);
        ok = misc[0] == 0.0;
        __syncthreads();
        continue;
      }
      if constexpr (!LEAN) {
      // ---- load the owned row into registers
      double a[K];
      double dacc = 0.0;
      if (tid < K) {
        const double* row = tri + ro_c(tid);
#pragma unroll
        for (int p = 0; p < K; ++p) a[p] = p < tid ? row[p] : (p == tid ? dg : 0.0);
        dacc = dg;
      } else if (tid < Sh::kRows) {
        const int c = tid - K;
#pragma unroll
        for (int p = 0; p < K; ++p) a[p] = Y[static_cast<int64_t>(sr[p]) * M + c];
      } else {
#pragma unroll
        for (int p = 0; p < K; ++p) a[p] = 0.0;
      }
      if (tid == 0) {
        misc[0] = 0.0;
        if (!(dg > 0.0)) {
          misc[0] = 1.0;
        } else {
          invd[0] = rsqrt(dg);
          const double l00 = dg * invd[0];
          tri[0] = l00;
          a[0] = l00;
        }
      }
      __syncthreads();  // row reads of the triangle done; pivot 0 published
      if (misc[0] != 0.0) continue;
      // ---- left-looking sweep, one barrier per column (a failed pivot only sets
      // the flag: the rest of the sweep runs on garbage and is discarded)
#pragma unroll
      for (int j = 0; j < K; ++j) {
        if (32 * warp + 31 > j) {  // warp has rows > j (uniform branch)
          const double* Lj = tri + ro_c(j);
          double s0 = a[j], s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int p = 0; p + 3 < j; p += 4) {
            const double2 l0 = *reinterpret_cast<const double2*>(Lj + p);
            const double2 l1 = *reinterpret_cast<const double2*>(Lj + p + 2);
            s0 = fma(-a[p], l0.x, s0);
            s1 = fma(-a[p + 1], l0.y, s1);
            s2 = fma(-a[p + 2], l1.x, s2);
            s3 = fma(-a[p + 3], l1.y, s3);
          }
#pragma unroll
          for (int p = j & ~3; p < j; ++p) s0 = fma(-a[p], Lj[p], s0);
          const double s = (s0 + s1) + (s2 + s3);
          if (tid > j && tid < Sh::kRows) {
            const double l = s * invd[j];
            a[j] = l;
            if (tid < K) {
              tri[ro_c(tid) + j] = l;
              dacc = fma(-l, l, dacc);
              if (j + 1 < K && tid == j + 1) {  // next pivot is complete
                if (!(dacc > 0.0)) {
                  misc[0] = 1.0;
                } else {
                  const double inv = rsqrt(dacc);
                  const double ljj = dacc * inv;
                  invd[j + 1] = inv;
                  tri[ro_c(tid) + tid] = ljj;
                  a[j + 1] = ljj;
                }
              }
            }
          }
        }
        __syncthreads();
      }
      ok = misc[0] == 0.0;
      if (ok && tid >= K && tid < Sh::kRows) {
        const int c = tid - K;
#pragma unroll
        for (int p = 0; p < K; ++p) zbuf[c * K + p] = a[p];
      }
      __syncthreads();
      }  // !LEAN
    }
    if (!ok) {
      if (tid == 0) atomicMin(fail_min, static_cast<unsigned long long>(row_begin + r));
      continue;
    }
    // ---- backward solve L^T x = z (warp 0; x_j broadcast by shuffle)
    if (warp == 0) {
      constexpr int kS = (K + 31) / 32;
      for (int c = 0; c < M; ++c) {
        double y[kS];
#pragma unroll
        for (int s = 0; s < kS; ++s) y[s] = s * 32 + lane < K ? zbuf[c * K + s * 32 + lane] : 0.0;
#pragma unroll
        for (int j = K - 1; j >= 0; --j) {
          const double xj = __shfl_sync(0xffffffffu, y[j >> 5], j & 31) * invd[j];
          const double* Lj = tri + ro_c(j);
          if (lane == (j & 31)) y[j >> 5] = xj;
#pragma unroll
          for (int s = 0; s <= (j >> 5); ++s) {
            if (s * 32 + lane < j) y[s] = fma(-Lj[s * 32 + lane], xj, y[s]);
          }
        }
        double* Crow = C + r * K * M;
#pragma unroll
        for (int s = 0; s < kS; ++s)
          if (s * 32 + lane < K) Crow[(s * 32 + lane) * M + c] = y[s];
      }
    }
  }
}

template <int K, int M>
cudaError_t launch_cta(const double* X, const double* Y, int d, const int32_t* S, int64_t nrows, int64_t row_begin,
                       const KParams& kp, double* C, unsigned long long* fail_min, int num_sms, cudaStream_t stream) {
  using Sh = CtaShape<K, M>;
  // FMGP_SOLVE_GRAM=0: the direct difference build for every d (A/B, as in the register solve)
  const char* ge = std::getenv("FMGP_SOLVE_GRAM");
  const char* be = std::getenv("FMGP_CTA_BLOCKED");  // 0: row-per-thread column sweep instead of the blocked DMMA factor
  const int use_gram = (!(ge != nullptr && ge[0] == '0') ? 1 : 0) | (!(be != nullptr && be[0] == '0') ? 2 : 0);
  if constexpr (M == 1) {
    // FMGP_CTA_SLICE: dimensions staged per slice in the lean kernel (multiple of 4; 0 = the full-footprint kernel)
    const char* se = std::getenv("FMGP_CTA_SLICE");
    int xsd = se != nullptr ? std::atoi(se) : 24;
    if (use_gram == 3 && d >= 16 && d <= Sh::kXsD && xsd > 0) {
      xsd = std::min(Sh::kXsD, (xsd + 3) & ~3);
      int gst = xsd + 4;  // = 4 or 12 mod 16 doubles: the fragment loads of a warp take two wavefronts
      if (gst % 16 == 0 || gst % 16 == 8) gst += 4;
      const size_t bytes = sizeof(double) * (Sh::kTri + ((K * gst + 1) & ~1) + 3 * ((K + 1) & ~1) + 2) +
                           sizeof(int32_t) * K;
      cudaError_t err = cudaFuncSetAttribute(solve_cta_kernel<K, M, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(bytes));
      if (err != cudaSuccess) return err;
      int per_sm = 0;
      err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_cta_kernel<K, M, true>, Sh::kThreads, bytes);
      if (err != cudaSuccess) return err;
      if (per_sm < 1) per_sm = 1;
      const int64_t grid = std::min<int64_t>(nrows, static_cast<int64_t>(num_sms) * per_sm);
      solve_cta_kernel<K, M, true><<<static_cast<unsigned>(grid), Sh::kThreads, bytes, stream>>>(
          X, Y, d, S, nrows, row_begin, kp, C, fail_min, use_gram, xsd, gst);
      note_launches(1);
      return cudaGetLastError();
    }
  }
  cudaError_t err = cudaFuncSetAttribute(solve_cta_kernel<K, M, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Sh::kBytes));
  if (err != cudaSuccess) return err;
  int per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_cta_kernel<K, M, false>, Sh::kThreads, Sh::kBytes);
  if (err != cudaSuccess) return err;
  if (per_sm < 1) per_sm = 1;
  const int64_t grid = std::min<int64_t>(nrows, static_cast<int64_t>(num_sms) * per_sm);
  solve_cta_kernel<K, M, false><<<static_cast<unsigned>(grid), Sh::kThreads, Sh::kBytes, stream>>>(
      X, Y, d, S, nrows, row_begin, kp, C, fail_min, use_gram, 0, 0);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace

bool fused_solve_cta_supported(int k, int d, int m) {
  (void)d;
  return k == 100 && m == 1;
}

cudaError_t fused_solve_cta(const double* X, const double* Y, int d, int m, const int32_t* S, int64_t nrows,
                            int64_t row_begin, int k, const KParams& kp, double* C, unsigned long long* fail_min,
                            int num_sms, cudaStream_t stream) {
  if (nrows <= 0) return cudaSuccess;
  if (k == 100 && m == 1) return launch_cta<100, 1>(X, Y, d, S, nrows, row_begin, kp, C, fail_min, num_sms, stream);
  return cudaErrorInvalidValue;
}

}  // namespace fmgp
