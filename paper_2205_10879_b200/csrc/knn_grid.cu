// K1-grid — exact k-nearest neighbours for low dimension (d <= 3) through a
// uniform cell grid, bit-exact with the reference's Exact NeighborIndex
// (proj/core/src/nn_index.cpp:254-287, :351-366).
//
// The reference scans all n points per query (O(n^2 d) for precompute). For
// d <= 3 the same answer is found by examining only the points in the cells
// around the query: cells are visited as a block of radius 1 and then in
// rings of growing Chebyshev radius, and the search stops once every point
// outside the visited block is provably farther than the current k-th
// neighbour. "Provably" uses the computed key itself: the stop test compares
// the k-th key against (lower bound - margin)^2 with a margin far above any
// rounding in the cell assignment, so the neighbour set and order are the
// reference's, not an approximation.
//
// Layout in HBM (built per call, O(n)):
//   cell id   key(x) = ((c_z * G_y) + c_y) * G_x + c_x, c_t = floor((x_t - lo_t) / h) clamped
//   cstart    n_cells + 1 offsets (counting sort by key)
//   pts       n x d f64, points in cell order;  pid  n int32 original indices
// Rows of cells along x are contiguous, so a block of radius r is (2r+1)^(d-1)
// contiguous ranges.
//
// Query side: one warp per query. Candidates are evaluated 32 at a time
// (one per lane, coalesced loads from `pts`); a ballot skips batches with no
// candidate below the current k-th key; otherwise the batch is bitonic-sorted
// across lanes and merged into the warp's sorted top-KP list, which lives in
// registers (E = KP/32 entries per lane, lane-strided). Order is the
// reference's (dist_sq, index) pair order.
#include <cfloat>
#include <climits>
#include <cstdlib>
#include <string>

#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

struct GridParams {
  double lo[3];
  double h, inv_h;
  double margin;  // slack of every cell-bound test: 1e-7 h + the rounding of lo + c h (~eps |coordinates|)
  int G[3];
  int d;
  int64_t ncells;
};

// ---------------------------------------------------------------- build

__device__ __forceinline__ unsigned long long ord_key(double v) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ull) ? (k & ~0x8000000000000000ull) : ~k;
  return __longlong_as_double(static_cast<long long>(b));
}

__global__ void bbox_kernel(const double* __restrict__ X, int64_t n, int d, unsigned long long* __restrict__ mm) {
  // per-thread min/max -> warp shuffles -> CTA (shared memory) -> one atomic pair
  // per dimension per CTA (per-warp atomics on six words serialise in L2)
  __shared__ unsigned long long slo[3][32], shi[3][32];
  unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    for (int t = 0; t < d; ++t) {
      unsigned long long k = ord_key(X[i * d + t]);
      lo[t] = k < lo[t] ? k : lo[t];
      hi[t] = k > hi[t] ? k : hi[t];
    }
  }
  const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int t = 0; t < d; ++t) {
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long a = __shfl_xor_sync(0xffffffffu, lo[t], o);
      unsigned long long b = __shfl_xor_sync(0xffffffffu, hi[t], o);
      lo[t] = a < lo[t] ? a : lo[t];
      hi[t] = b > hi[t] ? b : hi[t];
    }
    if ((threadIdx.x & 31) == 0) {
      slo[t][wid] = lo[t];
      shi[t][wid] = hi[t];
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    for (int t = 0; t < d; ++t) {
      unsigned long long a = threadIdx.x < nw ? slo[t][threadIdx.x] : ~0ull;
      unsigned long long b = threadIdx.x < nw ? shi[t][threadIdx.x] : 0ull;
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long a2 = __shfl_xor_sync(0xffffffffu, a, o);
        const unsigned long long b2 = __shfl_xor_sync(0xffffffffu, b, o);
        a = a2 < a ? a2 : a;
        b = b2 > b ? b2 : b;
      }
      if (threadIdx.x == 0) {
        atomicMin(&mm[2 * t], a);
        atomicMax(&mm[2 * t + 1], b);
      }
    }
  }
}

// Cubic cells with ~`per_cell` points on average over the bounding box;
// degenerate (zero-extent) dimensions get one cell. Capped at max_cells.
__global__ void grid_params_kernel(const unsigned long long* __restrict__ mm, int64_t n, int d, double per_cell,
                                   int64_t max_cells, GridParams* __restrict__ gp) {
  double lo[3], ext[3];
  double vol = 1.0;
  int live = 0;
  for (int t = 0; t < d; ++t) {
    lo[t] = ord_val(mm[2 * t]);
    ext[t] = ord_val(mm[2 * t + 1]) - lo[t];
    if (ext[t] > 0.0) {
      vol *= ext[t];
      ++live;
    }
  }
  double cells = fmax(1.0, static_cast<double>(n) / per_cell);
  double h = live > 0 ? pow(vol / cells, 1.0 / live) : 1.0;
  int G[3] = {1, 1, 1};
  for (int iter = 0; iter < 64; ++iter) {
    double total = 1.0;
    for (int t = 0; t < d; ++t) {
      double g = ext[t] > 0.0 ? ceil(ext[t] / h) : 1.0;
      g = fmin(fmax(g, 1.0), 1048576.0);
      G[t] = static_cast<int>(g);
      total *= g;
    }
    if (total <= static_cast<double>(max_cells)) break;
    h *= 1.25;
  }
  GridParams p;
  p.d = d;
  p.h = h;
  p.inv_h = 1.0 / h;
  p.ncells = 1;
  double span = 0.0;
  for (int t = 0; t < 3; ++t) {
    p.lo[t] = t < d ? lo[t] : 0.0;
    p.G[t] = t < d ? G[t] : 1;
    p.ncells *= p.G[t];
    if (t < d) span = fmax(span, fabs(lo[t]) + G[t] * h);
  }
  // the cell boundaries lo + c h and the cell assignment round at ~eps of the
  // coordinates' magnitude; far from the origin (|lo| / h > ~1e9) that exceeds
  // 1e-7 h, so the margin carries it too
  p.margin = 1e-7 * h + 8.0 * 2.220446049250313e-16 * span;
  *gp = p;
}

__device__ __forceinline__ int cell_coord(double x, double lo, double inv_h, int G) {
  double f = floor(__dmul_rn(__dsub_rn(x, lo), inv_h));
  // !(f >= 0) also takes NaN to cell 0 (a NaN coordinate reaches here on the device-pointer
  // entry points; the query kernels give such a point no neighbour)
  int c = !(f >= 0.0) ? 0 : (f >= static_cast<double>(G) ? G - 1 : static_cast<int>(f));
  return c;
}

template <int D>
__device__ __forceinline__ int64_t cell_key(const double* x, const GridParams& g, int c[3]) {
#pragma unroll
  for (int t = 0; t < 3; ++t) c[t] = t < D ? cell_coord(x[t], g.lo[t], g.inv_h, g.G[t]) : 0;
  return (static_cast<int64_t>(c[2]) * g.G[1] + c[1]) * g.G[0] + c[0];
}

template <int D>
__global__ void count_kernel(const double* __restrict__ X, int64_t n, const GridParams* __restrict__ gpp,
                             int32_t* __restrict__ counts, int32_t* __restrict__ key, int32_t* __restrict__ slot) {
  const GridParams g = *gpp;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double x[3];
#pragma unroll
    for (int t = 0; t < D; ++t) x[t] = X[i * D + t];
    int c[3];
    int64_t kk = cell_key<D>(x, g, c);
    key[i] = static_cast<int32_t>(kk);
    slot[i] = atomicAdd(&counts[kk], 1);
  }
}

// Exclusive scan of counts[0..m) into start[0..m] (start[m] = total): per-block
// scan, then a scan of block sums, then the add-back.
constexpr int kScanBlock = 1024;
constexpr int kScanItems = 4;  // per thread

__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* warp_sums, int32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int32_t w = lane < (blockDim.x >> 5) ? warp_sums[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    warp_sums[lane] = w;
  }
  __syncthreads();
  int32_t before = wid > 0 ? warp_sums[wid - 1] : 0;
  if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
  return before + x - v;
}

__global__ void scan_local_kernel(const int32_t* __restrict__ in, int64_t m, int32_t* __restrict__ out,
                                  int32_t* __restrict__ block_sums) {
  __shared__ int32_t ws[32];
  __shared__ int32_t tot;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanBlock * kScanItems;
  int32_t v[kScanItems];
  int32_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    int64_t i = base + static_cast<int64_t>(threadIdx.x) * kScanItems + j;
    v[j] = i < m ? in[i] : 0;
    s += v[j];
  }
  int32_t pre = block_excl_scan(s, ws, threadIdx.x == 0 ? &tot : nullptr);
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    int64_t i = base + static_cast<int64_t>(threadIdx.x) * kScanItems + j;
    if (i < m) out[i] = pre;
    pre += v[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

__global__ void scan_sums_kernel(int32_t* __restrict__ sums, int64_t nb, int32_t* __restrict__ total_out) {
  __shared__ int32_t ws[32];
  __shared__ int32_t carry;
  __shared__ int32_t tot;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < nb; b0 += blockDim.x) {
    int64_t i = b0 + threadIdx.x;
    int32_t v = i < nb ? sums[i] : 0;
    int32_t pre = block_excl_scan(v, ws, threadIdx.x == 0 ? &tot : nullptr);
    __syncthreads();
    if (i < nb) sums[i] = carry + pre;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total_out = carry;
}

__global__ void scan_add_kernel(int32_t* __restrict__ out, int64_t m, const int32_t* __restrict__ sums) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanBlock * kScanItems;
  const int32_t add = sums[blockIdx.x];
  for (int j = 0; j < kScanItems; ++j) {
    int64_t i = base + static_cast<int64_t>(threadIdx.x) * kScanItems + j;
    if (i < m) out[i] += add;
  }
}

template <int D>
__global__ void scatter_kernel(const double* __restrict__ X, int64_t n, const int32_t* __restrict__ key,
                               const int32_t* __restrict__ slot, const int32_t* __restrict__ start,
                               double* __restrict__ pts, int32_t* __restrict__ pid, int32_t* __restrict__ pos_of) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t p = static_cast<int64_t>(start[key[i]]) + slot[i];
#pragma unroll
    for (int t = 0; t < D; ++t) pts[p * D + t] = X[i * D + t];
    pid[p] = static_cast<int32_t>(i);
    if (pos_of) pos_of[i] = static_cast<int32_t>(p);
  }
}

// ---------------------------------------------------------------- warp top-k

struct Cand {
  double d;
  int32_t i;
};

__device__ __forceinline__ bool cless(const Cand& a, const Cand& b) { return pair_less(a.d, a.i, b.d, b.i); }

__device__ __forceinline__ Cand shfl_xor_c(const Cand& c, int m) {
  return Cand{__shfl_xor_sync(0xffffffffu, c.d, m), __shfl_xor_sync(0xffffffffu, c.i, m)};
}
__device__ __forceinline__ Cand shfl_c(const Cand& c, int src) {
  return Cand{__shfl_sync(0xffffffffu, c.d, src), __shfl_sync(0xffffffffu, c.i, src)};
}

// One compare-exchange stage across lanes: lanes whose `stride` bit is clear
// keep the min when `up`, else the max.
__device__ __forceinline__ Cand cx_stage(Cand v, int stride, bool up, int lane) {
  Cand o = shfl_xor_c(v, stride);
  const bool lower = (lane & stride) == 0;
  const bool take_min = (lower == up);
  const bool o_less = cless(o, v);
  return (take_min == o_less) ? o : v;
}

__device__ __forceinline__ Cand bitonic_sort32(Cand v, int lane) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) v = cx_stage(v, stride, (lane & size) == 0, lane);
  }
  return v;
}

// Sort a bitonic 32-sequence ascending.
__device__ __forceinline__ Cand bitonic_clean32(Cand v, int lane) {
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) v = cx_stage(v, stride, true, lane);
  return v;
}

// Merge two ascending 32-sequences: a <- 32 smallest (ascending), b <- 32 largest (ascending).
__device__ __forceinline__ void merge32(Cand& a, Cand& b, int lane) {
  Cand br = shfl_c(b, 31 - lane);
  Cand lo = cless(br, a) ? br : a;
  Cand hi = cless(br, a) ? a : br;
  a = bitonic_clean32(lo, lane);
  b = bitonic_clean32(hi, lane);
}

// Keep the KP = 32*E smallest of (L u batch); L ascending over (e, lane).
template <int E>
__device__ __forceinline__ void merge_batch_chain(Cand (&L)[E], Cand c, int lane) {
  c = bitonic_sort32(c, lane);
  Cand cr = shfl_c(c, 31 - lane);
  Cand x = cless(cr, L[E - 1]) ? cr : L[E - 1];
  x = bitonic_clean32(x, lane);
  // Insert the sorted segment x into the sorted chain L[0..E-2] from the top:
  // merge(L[E-2], x) -> (L[E-2], L[E-1]), then merge(L[E-3], L[E-2]) -> ...
#pragma unroll
  for (int e = E - 1; e >= 1; --e) {
    Cand a = L[e - 1];
    Cand b = (e == E - 1) ? x : L[e];
    merge32(a, b, lane);
    L[e - 1] = a;
    L[e] = b;
  }
  if (E == 1) L[0] = x;
}

// ---------------------------------------------------------------- query

// Squared lower bound on the distance from q to any point outside the block
// of radius r (infinite when the block covers the grid), shrunk by a margin
// (1e-7 h) that dominates every rounding in the cell assignment (~eps * G * h)
// and in the key itself (~5 eps relative).
template <int D>
__device__ __forceinline__ double outside_lb_sq(const GridParams& g, const double* q, const int c[3], int r) {
  double lb = INFINITY;
#pragma unroll
  for (int t = 0; t < D; ++t) {
    if (c[t] - r > 0) lb = fmin(lb, q[t] - (g.lo[t] + (c[t] - r) * g.h));
    if (c[t] + r < g.G[t] - 1) lb = fmin(lb, (g.lo[t] + (c[t] + r + 1) * g.h) - q[t]);
  }
  if (lb == INFINITY) return INFINITY;
  lb -= g.margin;
  if (!(lb > 0.0)) return 0.0;
  return lb * lb * (1.0 - 1e-12);
}

constexpr int kQueryThreads = 256;
#ifndef FMGP_LANEDOT_UNROLL
#define FMGP_LANEDOT_UNROLL 4
#endif
constexpr int kLaneDotUnroll = FMGP_LANEDOT_UNROLL;  // neighbour pairs per unrolled step of the lane-per-point dot
constexpr int kSlots = 64;  // ranges per chunk: 2 per lane (one cell-row per lane)
#ifndef FMGP_INSERT_MAX
#define FMGP_INSERT_MAX 4
#endif
constexpr int kInsertMax = FMGP_INSERT_MAX;  // batches with at most this many admissions are inserted one by one
#ifndef FMGP_GQ_SELECT  // 1: threshold selection of the first chunk (A/B: slower, see profiles/r02/ab_gq_select.txt)
#define FMGP_GQ_SELECT 0
#endif

// Static cell visiting order for the warp kernel: every offset o of Chebyshev
// radius <= R sorted by its static lower bound sb(o) = sum_t max(|o_t| - 1, 0)^2
// (in h^2: no point of cell c + o is closer than h sqrt(sb) to any point of
// cell c), the sb = 0 block (3^D cells) first. Packed (o_x + 128) |
// (o_y + 128) << 8 | (o_z + 128) << 16 | sb << 24. Generated at compile time.
template <int D>
struct OrdR {
  static constexpr int R = D == 3 ? 3 : 4;
  static constexpr int N = D == 3 ? 343 : (D == 2 ? 81 : 9);
};
template <int D>
struct OrdTable {
  int32_t e[OrdR<D>::N];
};
template <int D>
constexpr OrdTable<D> make_ord() {
  constexpr int R = OrdR<D>::R, N = OrdR<D>::N, W = 2 * R + 1;
  OrdTable<D> t{};
  int sb[N] = {}, l1[N] = {};
  for (int i = 0; i < N; ++i) {
    int o[3] = {0, 0, 0};
    int v = i;
    for (int a = 0; a < D; ++a) {
      o[a] = v % W - R;
      v /= W;
    }
    int s2 = 0, n1 = 0;
    for (int a = 0; a < D; ++a) {
      const int m = (o[a] < 0 ? -o[a] : o[a]) - 1;
      s2 += m > 0 ? m * m : 0;
      n1 += o[a] < 0 ? -o[a] : o[a];
    }
    t.e[i] = (o[0] + 128) | ((o[1] + 128) << 8) | ((o[2] + 128) << 16) | (s2 << 24);
    sb[i] = s2;
    l1[i] = n1;
  }
  for (int i = 1; i < N; ++i) {  // insertion sort by (sb, |o|_1), stable
    const int e = t.e[i], s0 = sb[i], n0 = l1[i];
    int j = i - 1;
    while (j >= 0 && (sb[j] > s0 || (sb[j] == s0 && l1[j] > n0))) {
      t.e[j + 1] = t.e[j];
      sb[j + 1] = sb[j];
      l1[j + 1] = l1[j];
      --j;
    }
    t.e[j + 1] = e;
    sb[j + 1] = s0;
    l1[j + 1] = n0;
  }
  return t;
}
__constant__ OrdTable<2> kOrd2 = make_ord<2>();
__constant__ OrdTable<3> kOrd3 = make_ord<3>();
template <int D>
__device__ __forceinline__ int32_t ord_entry(int i) {
  if constexpr (D == 3) return kOrd3.e[i];
  else return kOrd2.e[i];
}

// One warp per query. Query w is: sorted position qpos[w] (self mode,
// exclusion by original index), or sorted position w when qpos == nullptr
// and Q == nullptr, or external coordinates Q[w] (no exclusion). Output row
// index: original index - row_offset (self modes) or qout[w] / w.
//
// Walk (d = 2, 3): the cells of Chebyshev radius <= R in the static order
// above, one chunk of up to 32 cells at a time (the 3^D block first); a cell
// whose exact box distance to q (each axis gap shrunk by the 1e-7 h margin)
// exceeds the current kk-th key is skipped, and the walk stops before a chunk
// whose static bound h sqrt(min(sb, R^2)) - slack - 1e-7 h (slack = distance
// of q outside its own cell's box, 0 for points of the set) already exceeds
// the kk-th key (cells beyond radius R have sb >= R^2). If the list runs out
// the Chebyshev-ring walk continues from radius R + 1 with the
// outside-the-block stop test. With cells of ~kk/6 (2-D) or ~kk/16 (3-D)
// points this examines ~2x (2-D) to ~3x (3-D) fewer candidates than a radius-1
// block of ~kk/2 points per cell, and returns the same rows.
#ifndef FMGP_GQ_MINB
#define FMGP_GQ_MINB 4
#endif
#ifndef FMGP_GP_MINB
#define FMGP_GP_MINB 3
#endif
template <int D, int E>
__global__ void __launch_bounds__(kQueryThreads, FMGP_GQ_MINB)
grid_query_kernel(const GridParams* __restrict__ gpp, const double* __restrict__ pts, const int32_t* __restrict__ pid,
                  const int32_t* __restrict__ cstart, int64_t nq, const int32_t* __restrict__ qpos,
                  const double* __restrict__ Q, const int32_t* __restrict__ qout, const int32_t* __restrict__ excl_arr,
                  int kk, int with_self, int64_t row_offset, int32_t* __restrict__ out, double* __restrict__ out_d) {
  __shared__ int32_t s_beg[kQueryThreads / 32][kSlots];
  __shared__ int32_t s_pre[kQueryThreads / 32][kSlots + 1];
  __shared__ double s_ck[E == 2 ? kQueryThreads / 32 : 1][64];  // first-chunk selection: the 64 kept candidates
  __shared__ int32_t s_ci[E == 2 ? kQueryThreads / 32 : 1][64];
  const GridParams g = *gpp;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int32_t* rb = s_beg[wib];
  int32_t* rp = s_pre[wib];
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = warp0; w < nq; w += nwarps) {
    double q[D];
    int32_t self = -1;
    int64_t orow;
    if (Q == nullptr) {
      const int64_t p = qpos != nullptr ? qpos[w] : w;
#pragma unroll
      for (int t = 0; t < D; ++t) q[t] = pts[p * D + t];
      self = pid[p];
      orow = static_cast<int64_t>(self) - row_offset;
    } else {
#pragma unroll
      for (int t = 0; t < D; ++t) q[t] = Q[w * D + t];
      orow = qout != nullptr ? qout[w] : w;
      if (excl_arr != nullptr) self = excl_arr[orow];
    }
    {
      // a non-finite query ranks no point (the host entry points reject it with FMGP_EINVAL):
      // the row is INT_MAX / inf, no walk
      bool qfin = true;
#pragma unroll
      for (int t = 0; t < D; ++t) qfin = qfin && (__double2hiint(q[t]) & 0x7ff00000) != 0x7ff00000;
      if (!qfin) {
        const int width = kk + (with_self ? 1 : 0);
        if (with_self && lane == 0) out[orow * width] = self;
        for (int t = lane; t < kk; t += 32) {
          out[orow * width + (with_self ? 1 : 0) + t] = INT_MAX;
          if (out_d) out_d[orow * kk + t] = INFINITY;
        }
        continue;
      }
    }
    int c[3];
    cell_key<D>(q, g, c);

    Cand L[E];
#pragma unroll
    for (int e = 0; e < E; ++e) L[e] = Cand{INFINITY, INT_MAX};
    Cand thr{INFINITY, INT_MAX};
    const int tl = (kk - 1) & 31, te = (kk - 1) >> 5;
    bool fresh = true;  // list still empty (nothing merged yet)

    // Scan up to 64 ranges (two per lane) of cell-ordered points: candidates
    // 32 at a time, ballot skip, bitonic sort + merge into the top-KP list.
    auto scan_ranges = [&](int32_t b0, int32_t l0, int32_t b1, int32_t l1) {
      int32_t incl = l0 + l1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int32_t excl = incl - (l0 + l1);
      rb[2 * lane] = b0;
      rb[2 * lane + 1] = b1;
      rp[2 * lane] = excl;
      rp[2 * lane + 1] = excl + l0;
      const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
      if (lane == 31) rp[kSlots] = total;
      __syncwarp();
      auto fetch = [&](int32_t want) -> Cand {
        Cand cd{INFINITY, INT_MAX};
        if (want < total) {
          int j = 0;  // largest slot j with rp[j] <= want (skips empty slots)
#pragma unroll
          for (int step = kSlots / 2; step > 0; step >>= 1)
            if (rp[j + step] <= want) j += step;
          const int64_t p = static_cast<int64_t>(rb[j]) + (want - rp[j]);
          const int32_t id = pid[p];
          double x[D];
#pragma unroll
          for (int t = 0; t < D; ++t) x[t] = pts[p * D + t];
          const double sd = dist_sq_fixed<D>(q, x);
          if (id != self) cd = Cand{sd, id};
        }
        return cd;
      };
      int32_t base = 0;
      bool selected = false;
#if FMGP_GQ_SELECT
      if constexpr (E == 2) {
        if (fresh && total > 64 && total <= 128) {
          // The list is empty and the first chunk (the 3^D block) holds 65..128 candidates,
          // of which 64 can stay: instead of sorting all of them (a 64-network plus one
          // 30-stage sort + merge per further batch), find a key value with exactly 64
          // candidates at or below it by bisection (one redux per round), compact those 64
          // through shared memory and sort only them. Exact: the 64 kept are the 64
          // smallest keys; when no such value exists (a tie across the 64th / 65th key)
          // or fewer than 64 candidates are valid, the sort path below runs instead.
          Cand c4[4];
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4) c4[s4] = fetch(s4 * 32 + lane);
          double mn = INFINITY, mx = 0.0;
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4) {
            mn = fmin(mn, c4[s4].d);
            mx = c4[s4].d < INFINITY ? fmax(mx, c4[s4].d) : mx;
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
          }
          auto count_le = [&](double v) {
            int cl = 0;
#pragma unroll
            for (int s4 = 0; s4 < 4; ++s4) cl += c4[s4].d <= v ? 1 : 0;
            return __reduce_add_sync(0xffffffffu, cl);
          };
          double cut = mx;
          int cnt = count_le(mx);  // the valid candidates (self and padding are inf)
          if (cnt > 64) {
            double lo = mn, hi = mx;  // count(<= lo) >= 1, count(<= hi) > 64
            for (int round = 0; round < 24; ++round) {
              const double mid = lo + 0.5 * (hi - lo);
              if (!(mid > lo && mid < hi)) break;  // adjacent doubles: a tie across the boundary
              cnt = count_le(mid);
              cut = mid;
              if (cnt == 64) break;
              if (cnt < 64) lo = mid;
              else hi = mid;
            }
          }
          if (cnt == 64) {
            double* ck = s_ck[wib];
            int32_t* ci = s_ci[wib];
            int pos0 = 0;
#pragma unroll
            for (int s4 = 0; s4 < 4; ++s4) {
              const bool keep = c4[s4].d <= cut;
              const unsigned bal = __ballot_sync(0xffffffffu, keep);
              if (keep) {
                const int pp = pos0 + __popc(bal & ((1u << lane) - 1u));
                ck[pp] = c4[s4].d;
                ci[pp] = c4[s4].i;
              }
              pos0 += __popc(bal);
            }
            __syncwarp();
            Cand a = bitonic_sort32(Cand{ck[lane], ci[lane]}, lane);
            Cand b2 = bitonic_sort32(Cand{ck[32 + lane], ci[32 + lane]}, lane);
            merge32(a, b2, lane);
            L[0] = a;
            L[1] = b2;
            thr = shfl_c(te == 0 ? L[0] : L[1], tl);
            base = total;
            selected = true;
            __syncwarp();
          }
        }
      }
#endif
      if (!selected && fresh && total >= 64) {
        // the list is empty: sort the first 64 candidates as one bitonic network
        // (two 32-sorts + one merge: 41 compare-exchange stages instead of the
        // 60 of two batch merges) and take them as the list
        Cand a = bitonic_sort32(fetch(lane), lane);
        Cand b2 = bitonic_sort32(fetch(32 + lane), lane);
        merge32(a, b2, lane);
#pragma unroll
        for (int e = 0; e < E; ++e) L[e] = e == 0 ? a : (e == 1 ? b2 : Cand{INFINITY, INT_MAX});
        Cand t{0, 0};
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (e == te) t = L[e];
        thr = shfl_c(t, tl);
        base = 64;
      }
      fresh = false;
      for (; base < total; base += 32) {
        Cand cd = fetch(base + lane);
        const bool pass = cless(cd, thr);
        const unsigned bal = __ballot_sync(0xffffffffu, pass);
        if (bal == 0) continue;
        if (__popc(bal) <= kInsertMax) {
          // few candidates: insert each into the sorted list (rank by ballots,
          // shift the tail up one slot) instead of a 30-stage sort + merge
          unsigned mleft = bal;
          while (mleft != 0) {
            const int src = __ffs(mleft) - 1;
            mleft &= mleft - 1;
            const Cand c = shfl_c(cd, src);
            if (!cless(c, thr)) continue;  // the threshold fell since the ballot
            int rank = 0;
#pragma unroll
            for (int e = 0; e < E; ++e) rank += __popc(__ballot_sync(0xffffffffu, cless(L[e], c)));
#pragma unroll
            for (int e = E - 1; e >= 0; --e) {  // descending: L[e-1] is still the old segment
              Cand up = Cand{__shfl_up_sync(0xffffffffu, L[e].d, 1), __shfl_up_sync(0xffffffffu, L[e].i, 1)};
              if (e > 0) {
                const Cand last = shfl_c(L[e > 0 ? e - 1 : 0], 31);
                if (lane == 0) up = last;
              }
              const int g = 32 * e + lane;
              if (g == rank) L[e] = c;
              else if (g > rank) L[e] = up;
            }
            Cand t{0, 0};
#pragma unroll
            for (int e = 0; e < E; ++e)
              if (e == te) t = L[e];
            thr = shfl_c(t, tl);
          }
          continue;
        }
        if (!pass) cd = Cand{INFINITY, INT_MAX};
        merge_batch_chain<E>(L, cd, lane);
        Cand t{0, 0};
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (e == te) t = L[e];
        thr = shfl_c(t, tl);
      }
      __syncwarp();
    };

    int r0 = 1;  // first Chebyshev ring of the fallback walk
    bool done = false;
    if constexpr (D >= 2) {
      constexpr int R = OrdR<D>::R, N = OrdR<D>::N, N0 = D == 3 ? 27 : 9;
      double slack2 = 0.0, lo_c[D];
#pragma unroll
      for (int t = 0; t < D; ++t) {
        lo_c[t] = g.lo[t] + c[t] * g.h;
        const double gap = fmax(fmax(lo_c[t] - q[t], q[t] - (lo_c[t] + g.h)), 0.0);
        slack2 += gap * gap;
      }
      const double slack = sqrt(slack2), margin = g.margin;
      for (int base = 0; base < N;) {
        const int len = base == 0 ? N0 : min(32, N - base);
        if (base > 0) {
          const int sbv = min(static_cast<int>(static_cast<uint32_t>(ord_entry<D>(base)) >> 24), R * R);
          const double lb = g.h * sqrt(static_cast<double>(sbv)) - slack - margin;
          if (lb > 0.0 && thr.d < lb * lb * (1.0 - 1e-12)) {
            done = true;
            break;
          }
        }
        int32_t b0 = 0, l0 = 0;
        if (lane < len) {
          const int32_t e = ord_entry<D>(base + lane);
          int cc[3] = {c[0] + ((e & 0xff) - 128), c[1] + (((e >> 8) & 0xff) - 128), D == 3 ? c[2] + (((e >> 16) & 0xff) - 128) : 0};
          bool in = true;
          double lb2 = 0.0;
#pragma unroll
          for (int t = 0; t < D; ++t) {
            in = in && cc[t] >= 0 && cc[t] < g.G[t];
            const double lo = g.lo[t] + cc[t] * g.h;
            const double gap = fmax(fmax(lo - q[t], q[t] - (lo + g.h)) - margin, 0.0);
            lb2 += gap * gap;
          }
          if (in && !(lb2 * (1.0 - 1e-12) > thr.d)) {
            const int64_t key = D == 3 ? (static_cast<int64_t>(cc[2]) * g.G[1] + cc[1]) * g.G[0] + cc[0]
                                       : static_cast<int64_t>(cc[1]) * g.G[0] + cc[0];
            b0 = cstart[key];
            l0 = cstart[key + 1] - b0;
          }
        }
        scan_ranges(b0, l0, 0, 0);
        base += len;
      }
      if (!done) {
        const double lb2 = outside_lb_sq<D>(g, q, c, R);
        done = lb2 == INFINITY || thr.d < lb2;
      }
      r0 = R + 1;
    }

    for (int r = r0; !done; ++r) {
      const bool block = (r == 1);
      const int z0 = D >= 3 ? max(0, c[2] - r) : 0, z1 = D >= 3 ? min(g.G[2] - 1, c[2] + r) : 0;
      const int y0 = D >= 2 ? max(0, c[1] - r) : 0, y1 = D >= 2 ? min(g.G[1] - 1, c[1] + r) : 0;
      const int xl = c[0] - r, xr = c[0] + r;
      const int x0 = max(0, xl), x1 = min(g.G[0] - 1, xr);
      const int ny = y1 - y0 + 1;
      const int nrows = (z1 - z0 + 1) * ny;
      for (int rbase = 0; rbase < nrows; rbase += 32) {
        // each lane turns one cell-row of the ring into <= 2 contiguous ranges
        const int ridx = rbase + lane;
        int32_t b0 = 0, l0 = 0, b1 = 0, l1 = 0;
        if (ridx < nrows) {
          const int z = z0 + ridx / ny, y = y0 + ridx % ny;
          const bool edge = block || (D >= 3 && (z == c[2] - r || z == c[2] + r)) ||
                            (D >= 2 && (y == c[1] - r || y == c[1] + r));
          const int64_t rowkey = (static_cast<int64_t>(z) * g.G[1] + y) * g.G[0];
          if (edge) {
            b0 = cstart[rowkey + x0];
            l0 = cstart[rowkey + x1 + 1] - b0;
          } else {
            if (xl >= 0) {
              b0 = cstart[rowkey + xl];
              l0 = cstart[rowkey + xl + 1] - b0;
            }
            if (xr < g.G[0]) {
              b1 = cstart[rowkey + xr];
              l1 = cstart[rowkey + xr + 1] - b1;
            }
          }
        }
        scan_ranges(b0, l0, b1, l1);
      }
      const double lb2 = outside_lb_sq<D>(g, q, c, r);
      if (lb2 == INFINITY) break;  // the block covers every cell
      if (thr.d < lb2) break;      // nothing outside can enter the top-kk
    }
    // write the row: [self,] top kk in order
    const int width = kk + (with_self ? 1 : 0);
    int32_t* row = out + orow * width;
    if (with_self && lane == 0) row[0] = self;
    const int o = with_self ? 1 : 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int t = e * 32 + lane;
      if (t < kk) {
        row[o + t] = L[e].i;
        if (out_d) out_d[orow * kk + t] = L[e].d;
      }
    }
  }
}

// Thread-per-query variant (A/B only, FMGP_KNN_GRID=thread; walks the
// Chebyshev rings from radius 1, measured no faster than the warp kernel:
// the per-thread heap sifts diverge across the warp and the heaps' shared
// memory leaves little L1 for the candidate loads): each thread
// owns one query, walks the same block/rings with its own loop and keeps its
// top-kk in a max-heap on (key, index) in shared memory (slot-major, so the
// heap accesses of a warp are bank-conflict-free), root cached in registers.
// With ~4-5 k candidates per query at cfg2 the warp kernel spends most of its
// instructions in 32-wide bitonic sorts and merges; here a rejected
// candidate costs one compare and an admitted one a heap sift (<= log2 kk
// levels), and consecutive threads hold queries of the same or neighbouring
// cells (cell order), so their candidate loads are mostly the same address.
// Same walk, stop test and (key, index) order as grid_query_kernel: the
// rows are identical.
constexpr int kThreadMaxK = 64;
constexpr int kThreadQueryThreads = 64;

template <int D>
__global__ void __launch_bounds__(kThreadQueryThreads)
grid_query_thread_kernel(const GridParams* __restrict__ gpp, const double* __restrict__ pts,
                         const int32_t* __restrict__ pid, const int32_t* __restrict__ cstart, int64_t nq,
                         const int32_t* __restrict__ qpos, const double* __restrict__ Q,
                         const int32_t* __restrict__ qout, const int32_t* __restrict__ excl_arr, int kk,
                         int with_self, int64_t row_offset, int32_t* __restrict__ out, double* __restrict__ out_d) {
  extern __shared__ double hsm[];
  const int T = blockDim.x;
  double* hd = hsm + threadIdx.x;                                                  // hd[s * T]
  int32_t* hi = reinterpret_cast<int32_t*>(hsm + static_cast<size_t>(kk) * T) + threadIdx.x;  // hi[s * T]
  const GridParams g = *gpp;
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * T + threadIdx.x; w < nq;
       w += static_cast<int64_t>(gridDim.x) * T) {
    double q[D];
    int32_t self = -1;
    int64_t orow;
    if (Q == nullptr) {
      const int64_t p = qpos != nullptr ? qpos[w] : w;
#pragma unroll
      for (int t = 0; t < D; ++t) q[t] = pts[p * D + t];
      self = pid[p];
      orow = static_cast<int64_t>(self) - row_offset;
    } else {
#pragma unroll
      for (int t = 0; t < D; ++t) q[t] = Q[w * D + t];
      orow = qout != nullptr ? qout[w] : w;
      if (excl_arr != nullptr) self = excl_arr[orow];
    }
    int c[3];
    cell_key<D>(q, g, c);
    int cnt = 0;
    double rd = INFINITY;  // heap root (the kk-th best once full)
    int32_t ri = INT_MAX;

    auto consider = [&](int32_t b, int32_t e) {
      for (int32_t p = b; p < e; ++p) {
        const int32_t id = pid[p];
        double x[D];
#pragma unroll
        for (int t = 0; t < D; ++t) x[t] = pts[static_cast<int64_t>(p) * D + t];
        const double sd = dist_sq_fixed<D>(q, x);
        if (id == self) continue;
        if (cnt < kk) {  // push + sift up
          int pos = cnt++;
          while (pos > 0) {
            const int par = (pos - 1) >> 1;
            const double pd = hd[par * T];
            const int32_t pi = hi[par * T];
            if (!pair_less(pd, pi, sd, id)) break;
            hd[pos * T] = pd;
            hi[pos * T] = pi;
            pos = par;
          }
          hd[pos * T] = sd;
          hi[pos * T] = id;
          rd = hd[0];
          ri = hi[0];
        } else if (pair_less(sd, id, rd, ri)) {  // replace the root + sift down
          int pos = 0;
          for (;;) {
            int ch = 2 * pos + 1;
            if (ch >= kk) break;
            double cd = hd[ch * T];
            int32_t ci = hi[ch * T];
            if (ch + 1 < kk) {
              const double d2 = hd[(ch + 1) * T];
              const int32_t i2 = hi[(ch + 1) * T];
              if (pair_less(cd, ci, d2, i2)) {
                cd = d2;
                ci = i2;
                ++ch;
              }
            }
            if (!pair_less(sd, id, cd, ci)) break;
            hd[pos * T] = cd;
            hi[pos * T] = ci;
            pos = ch;
          }
          hd[pos * T] = sd;
          hi[pos * T] = id;
          rd = hd[0];
          ri = hi[0];
        }
      }
    };

    for (int r = 1;; ++r) {
      const bool block = (r == 1);
      const int z0 = D >= 3 ? max(0, c[2] - r) : 0, z1 = D >= 3 ? min(g.G[2] - 1, c[2] + r) : 0;
      const int y0 = D >= 2 ? max(0, c[1] - r) : 0, y1 = D >= 2 ? min(g.G[1] - 1, c[1] + r) : 0;
      const int xl = c[0] - r, xr = c[0] + r;
      const int x0 = max(0, xl), x1 = min(g.G[0] - 1, xr);
      for (int z = z0; z <= z1; ++z) {
        for (int y = y0; y <= y1; ++y) {
          const bool edge = block || (D >= 3 && (z == c[2] - r || z == c[2] + r)) ||
                            (D >= 2 && (y == c[1] - r || y == c[1] + r));
          const int64_t rowkey = (static_cast<int64_t>(z) * g.G[1] + y) * g.G[0];
          if (edge) {
            consider(cstart[rowkey + x0], cstart[rowkey + x1 + 1]);
          } else {
            if (xl >= 0) consider(cstart[rowkey + xl], cstart[rowkey + xl + 1]);
            if (xr < g.G[0]) consider(cstart[rowkey + xr], cstart[rowkey + xr + 1]);
          }
        }
      }
      const double lb2 = outside_lb_sq<D>(g, q, c, r);
      if (lb2 == INFINITY) break;             // the block covers every cell
      if (cnt == kk && rd < lb2) break;       // nothing outside can enter the top-kk
    }
    // heap sort in place: ascending (key, index) in slots 0 .. cnt-1
    for (int end = cnt - 1; end > 0; --end) {
      const double td = hd[end * T];
      const int32_t ti = hi[end * T];
      hd[end * T] = hd[0];
      hi[end * T] = hi[0];
      int pos = 0;
      for (;;) {
        int ch = 2 * pos + 1;
        if (ch >= end) break;
        double cd = hd[ch * T];
        int32_t ci = hi[ch * T];
        if (ch + 1 < end) {
          const double d2 = hd[(ch + 1) * T];
          const int32_t i2 = hi[(ch + 1) * T];
          if (pair_less(cd, ci, d2, i2)) {
            cd = d2;
            ci = i2;
            ++ch;
          }
        }
        if (!pair_less(td, ti, cd, ci)) break;
        hd[pos * T] = cd;
        hi[pos * T] = ci;
        pos = ch;
      }
      hd[pos * T] = td;
      hi[pos * T] = ti;
    }
    const int width = kk + (with_self ? 1 : 0);
    int32_t* row = out + orow * width;
    const int o = with_self ? 1 : 0;
    if (with_self) row[0] = self;
    for (int t = 0; t < kk; ++t) {
      row[o + t] = t < cnt ? hi[t * T] : INT_MAX;
      if (out_d) out_d[orow * kk + t] = t < cnt ? hd[t * T] : INFINITY;
    }
  }
}

// Warp-cooperative exact 1-NN of q (argmin over (key, index), the reference's
// std::min over pairs, nn_index.cpp:351-366): the distance-ordered cell walk
// of grid_query_kernel (the 3^D block first, then chunks of up to 32 cells
// skipped by their box bound, then Chebyshev rings), candidates 32 at a time.
template <int D>
__device__ __forceinline__ Cand warp_nn_walk(const GridParams& g, const double* __restrict__ pts,
                                             const int32_t* __restrict__ pid, const int32_t* __restrict__ cstart,
                                             const double (&q)[D], int32_t* rb, int32_t* rp, int lane) {
    int c[3];
    cell_key<D>(q, g, c);
    Cand best{INFINITY, INT_MAX};
    // argmin over up to 64 ranges (two per lane), then over the warp
    auto scan_ranges = [&](int32_t b0, int32_t l0, int32_t b1, int32_t l1) {
      int32_t incl = l0 + l1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int32_t excl = incl - (l0 + l1);
      rb[2 * lane] = b0;
      rb[2 * lane + 1] = b1;
      rp[2 * lane] = excl;
      rp[2 * lane + 1] = excl + l0;
      const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
      if (lane == 31) rp[kSlots] = total;
      __syncwarp();
      for (int32_t base = 0; base < total; base += 32) {
        const int32_t want = base + lane;
        if (want < total) {
          int j = 0;
#pragma unroll
          for (int step = kSlots / 2; step > 0; step >>= 1)
            if (rp[j + step] <= want) j += step;
          const int64_t p = static_cast<int64_t>(rb[j]) + (want - rp[j]);
          double x[D];
#pragma unroll
          for (int t = 0; t < D; ++t) x[t] = pts[p * D + t];
          const Cand cd{dist_sq_fixed<D>(q, x), pid[p]};
          if (cless(cd, best)) best = cd;
        }
      }
      __syncwarp();
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const Cand other = shfl_xor_c(best, o);
        if (cless(other, best)) best = other;
      }
    };

    int r0 = 1;
    bool done = false;
    if constexpr (D >= 2) {
      constexpr int R = OrdR<D>::R, N = OrdR<D>::N, N0 = D == 3 ? 27 : 9;
      double slack2 = 0.0;
#pragma unroll
      for (int t = 0; t < D; ++t) {
        const double lo = g.lo[t] + c[t] * g.h;
        const double gap = fmax(fmax(lo - q[t], q[t] - (lo + g.h)), 0.0);
        slack2 += gap * gap;
      }
      const double slack = sqrt(slack2), margin = g.margin;
      for (int base = 0; base < N;) {
        const int len = base == 0 ? N0 : min(32, N - base);
        if (base > 0) {
          const int sbv = min(static_cast<int>(static_cast<uint32_t>(ord_entry<D>(base)) >> 24), R * R);
          const double lb = g.h * sqrt(static_cast<double>(sbv)) - slack - margin;
          if (lb > 0.0 && best.d < lb * lb * (1.0 - 1e-12)) {
            done = true;
            break;
          }
        }
        int32_t b0 = 0, l0 = 0;
        if (lane < len) {
          const int32_t e = ord_entry<D>(base + lane);
          int cc[3] = {c[0] + ((e & 0xff) - 128), c[1] + (((e >> 8) & 0xff) - 128),
                       D == 3 ? c[2] + (((e >> 16) & 0xff) - 128) : 0};
          bool in = true;
          double lb2 = 0.0;
#pragma unroll
          for (int t = 0; t < D; ++t) {
            in = in && cc[t] >= 0 && cc[t] < g.G[t];
            const double lo = g.lo[t] + cc[t] * g.h;
            const double gap = fmax(fmax(lo - q[t], q[t] - (lo + g.h)) - margin, 0.0);
            lb2 += gap * gap;
          }
          if (in && !(lb2 * (1.0 - 1e-12) > best.d)) {
            const int64_t key = D == 3 ? (static_cast<int64_t>(cc[2]) * g.G[1] + cc[1]) * g.G[0] + cc[0]
                                       : static_cast<int64_t>(cc[1]) * g.G[0] + cc[0];
            b0 = cstart[key];
            l0 = cstart[key + 1] - b0;
          }
        }
        scan_ranges(b0, l0, 0, 0);
        base += len;
      }
      if (!done) {
        const double lb2 = outside_lb_sq<D>(g, q, c, R);
        done = lb2 == INFINITY || best.d < lb2;
      }
      r0 = R + 1;
    }
    for (int r = r0; !done; ++r) {
      const bool block = (r == 1);
      const int z0 = D >= 3 ? max(0, c[2] - r) : 0, z1 = D >= 3 ? min(g.G[2] - 1, c[2] + r) : 0;
      const int y0 = D >= 2 ? max(0, c[1] - r) : 0, y1 = D >= 2 ? min(g.G[1] - 1, c[1] + r) : 0;
      const int xl = c[0] - r, xr = c[0] + r;
      const int x0 = max(0, xl), x1 = min(g.G[0] - 1, xr);
      const int ny = y1 - y0 + 1;
      const int nrows = (z1 - z0 + 1) * ny;
      for (int rbase = 0; rbase < nrows; rbase += 32) {
        const int ridx = rbase + lane;
        int32_t b0 = 0, l0 = 0, b1 = 0, l1 = 0;
        if (ridx < nrows) {
          const int z = z0 + ridx / ny, y = y0 + ridx % ny;
          const bool edge = block || (D >= 3 && (z == c[2] - r || z == c[2] + r)) ||
                            (D >= 2 && (y == c[1] - r || y == c[1] + r));
          const int64_t rowkey = (static_cast<int64_t>(z) * g.G[1] + y) * g.G[0];
          if (edge) {
            b0 = cstart[rowkey + x0];
            l0 = cstart[rowkey + x1 + 1] - b0;
          } else {
            if (xl >= 0) {
              b0 = cstart[rowkey + xl];
              l0 = cstart[rowkey + xl + 1] - b0;
            }
            if (xr < g.G[0]) {
              b1 = cstart[rowkey + xr];
              l1 = cstart[rowkey + xr + 1] - b1;
            }
          }
        }
        scan_ranges(b0, l0, b1, l1);
      }
      const double lb2 = outside_lb_sq<D>(g, q, c, r);
      if (lb2 == INFINITY) break;
      if (best.d < lb2) break;
    }
    return best;
}

// Fused predict for d <= 3 (fast_predict_one, fast_predict.cpp:132-144).
// Each warp takes 32 consecutive (cell-sorted) test points.
// 1-NN, one lane per test point: the lane scans the 3^D block of cells
// around its point (cells of ~1.5 points in 2-D, ~1 in 3-D; a block row of
// cells is one contiguous range of the cell-ordered points) and keeps the
// (key, index) minimum; the answer is final when it is below the bound on
// every point outside the block (outside_lb_sq, conservative by the grid
// margin). Lanes whose block does not certify (empty neighbourhood, a test
// point outside the training box) are finished by the warp-cooperative walk.
// Gather-kernel-dot, one test point at a time over the warp: lanes t and
// t + 32 take neighbours t, t + 32 of the 1-NN's row (S, C coalesced, X
// gathered), evaluate the cross-covariances (kernel_from_sq_build, KF =
// kernel kind) and reduce the dot by a shuffle tree; the S/C row of the next
// test point and the X rows of the current one are loaded one step ahead, so
// the dependent 1-NN -> S -> X chain overlaps the arithmetic. The sum order
// differs from the reference's sequential loop by rounding only (tolerance
// 1e-9, tested). FMGP_PGRID_WARP=1 selects the warp walk for every point
// (A/B).
template <int D, int KF, bool kThreadNN>
__global__ void __launch_bounds__(kQueryThreads, FMGP_GP_MINB)
grid_predict_kernel(const GridParams* __restrict__ gpp, const double* __restrict__ pts, const int32_t* __restrict__ pid,
                    const int32_t* __restrict__ cstart, int64_t nq, const double* __restrict__ Qs,
                    const int32_t* __restrict__ qout, const double* __restrict__ X, const int32_t* __restrict__ S,
                    const double* __restrict__ Cf, int k, int m, KParams kp, const double* __restrict__ mean_offset,
                    double* __restrict__ out, int32_t* __restrict__ nn_out, const int32_t* __restrict__ pos_of,
                    const int32_t* __restrict__ s_pos, const double* __restrict__ c_perm, int lane_dot) {
  __shared__ int32_t s_beg[kQueryThreads / 32][kSlots];
  __shared__ int32_t s_pre[kQueryThreads / 32][kSlots + 1];
  __shared__ double s_exp[FMGP_BUILD_TAB_N];
  stage_exp_table(s_exp);
  __syncthreads();
  const GridParams g = *gpp;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  int32_t* rb = s_beg[wib];
  int32_t* rp = s_pre[wib];
  const double kc = kernel_scale_build<KF>(kp);
  const int64_t warp0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const bool fast = m == 1 && k <= 2 * kWarp && S != nullptr;
  for (int64_t w0 = warp0 * kWarp; w0 < nq; w0 += nwarps * kWarp) {
    const int nv = nq - w0 < kWarp ? static_cast<int>(nq - w0) : kWarp;
    const bool has = lane < nv;
    double q[D];
#pragma unroll
    for (int t = 0; t < D; ++t) q[t] = has ? Qs[(w0 + lane) * D + t] : 0.0;
    const int64_t orow = !has ? 0 : (qout != nullptr ? qout[w0 + lane] : w0 + lane);
    Cand best{INFINITY, INT_MAX};
    int32_t bpos = 0;  // grid position of best (the grid-ordered model's row)
    // a non-finite test point has no nearest neighbour (every key is NaN or inf): no search,
    // nn = -1 and NaN means below (the host entry points reject such batches with FMGP_EINVAL)
    bool qfin = true;
#pragma unroll
    for (int t = 0; t < D; ++t) qfin = qfin && (__double2hiint(q[t]) & 0x7ff00000) != 0x7ff00000;
    bool certified = !has || !qfin;
    if constexpr (kThreadNN) {
      if (has && qfin) {
        int c[3];
        cell_key<D>(q, g, c);
        const int x0 = max(c[0] - 1, 0), x1 = min(c[0] + 1, g.G[0] - 1);
        const int y0 = D >= 2 ? max(c[1] - 1, 0) : 0, y1 = D >= 2 ? min(c[1] + 1, g.G[1] - 1) : 0;
        const int z0 = D >= 3 ? max(c[2] - 1, 0) : 0, z1 = D >= 3 ? min(c[2] + 1, g.G[2] - 1) : 0;
        for (int z = z0; z <= z1; ++z) {
          for (int y = y0; y <= y1; ++y) {
            const int64_t rowkey = (static_cast<int64_t>(z) * g.G[1] + y) * g.G[0];
            const int32_t pb = __ldg(&cstart[rowkey + x0]), pe = __ldg(&cstart[rowkey + x1 + 1]);
            for (int32_t p = pb; p < pe; ++p) {
              double x[D];
#pragma unroll
              for (int t = 0; t < D; ++t) x[t] = __ldg(&pts[static_cast<int64_t>(p) * D + t]);
              const Cand cd{dist_sq_fixed<D>(q, x), __ldg(&pid[p])};
              if (cless(cd, best)) {
                best = cd;
                bpos = p;
              }
            }
          }
        }
        const double lb2 = outside_lb_sq<D>(g, q, c, 1);
        certified = best.d < INFINITY && (lb2 == INFINITY || best.d < lb2);
      }
    }
    unsigned need = __ballot_sync(0xffffffffu, !certified);
    while (need != 0) {
      const int src = __ffs(need) - 1;
      need &= need - 1;
      double qq[D];
#pragma unroll
      for (int t = 0; t < D; ++t) qq[t] = __shfl_sync(0xffffffffu, q[t], src);
      const Cand r = warp_nn_walk<D>(g, pts, pid, cstart, qq, rb, rp, lane);
      if (lane == src) {
        best = r;
        if (pos_of != nullptr && r.i != INT_MAX) bpos = pos_of[r.i];
      }
    }
    const bool found = best.i != INT_MAX;
    if (has && nn_out != nullptr) nn_out[orow] = found ? best.i : -1;
    if (S == nullptr) continue;  // nearest-only walk (NeighborIndex::nearest_training_point)
    if (has && !found)  // no candidate ranked (non-finite or overflowing z): NaN means, no gather
      for (int cc = 0; cc < m; ++cc) out[orow * m + cc] = __longlong_as_double(0x7ff8000000000000ll);
    if (fast && lane_dot) {
      // Gather-kernel-dot, one lane per test point (the lane that found the point's nearest
      // row walks that row itself): no shuffles, no reduction tree, every lane busy for all k
      // neighbours (a warp spread over one point's k = 50 neighbours fills 50 of 64 lane slots
      // and pays a 5-step reduction per point). Two neighbours per step: one 8-byte load of
      // the S row, one 16-byte load of the C row (each 32-byte sector is consumed by adjacent
      // steps, so the rows stream through L1 once), two coordinate gathers, two evaluations
      // into two accumulators. Sum order: sequential within each parity, as the reference's
      // loop up to rounding (tolerance 1e-9, tested).
      const bool perm = s_pos != nullptr;
      const int32_t* Sr = perm ? s_pos : S;
      const double* Cr = perm ? c_perm : Cf;
      const double* Xr = perm ? pts : X;
      const bool ok = has && found;
      const int64_t j = ok ? (perm ? bpos : best.i) : 0;
      const int2* srow = reinterpret_cast<const int2*>(Sr + j * k);
      const double2* crow = reinterpret_cast<const double2*>(Cr + j * k);
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll kLaneDotUnroll
      for (int t = 0; t < (k >> 1); ++t) {
        const int2 nb = __ldg(srow + t);
        const double2 cv = __ldg(crow + t);
        double xa[D], xb[D];
#pragma unroll
        for (int u = 0; u < D; ++u) {
          xa[u] = __ldg(&Xr[static_cast<int64_t>(nb.x) * D + u]);
          xb[u] = __ldg(&Xr[static_cast<int64_t>(nb.y) * D + u]);
        }
        double da = q[0] - xa[0], db = q[0] - xb[0];
        double sa = da * da, sb = db * db;
#pragma unroll
        for (int u = 1; u < D; ++u) {
          da = q[u] - xa[u];
          db = q[u] - xb[u];
          sa = fma(da, da, sa);
          sb = fma(db, db, sb);
        }
        acc0 = fma(kernel_from_sq_build<KF>(sa, kc, kp, s_exp), cv.x, acc0);
        acc1 = fma(kernel_from_sq_build<KF>(sb, kc, kp, s_exp), cv.y, acc1);
      }
      if (ok) out[orow] = (acc0 + acc1) + mean_offset[0];
      continue;
    }
    if (fast) {
      const int t0 = lane, t1 = lane + kWarp;
      const bool h0 = t0 < k, h1 = t1 < k;
      const double mo = mean_offset[0];
      // the grid-ordered model when attached (rows and neighbour coordinates in
      // cell order), else the model as given
      const bool perm = s_pos != nullptr;
      const int32_t* Sr = perm ? s_pos : S;
      const double* Cr = perm ? c_perm : Cf;
      const double* Xr = perm ? pts : X;
      const int32_t rowid = perm ? bpos : best.i;
      // stage loads of point i: its S/C row (needs j_i) and, one step later, its X rows (need S)
      auto load_sc = [&](int i, int64_t& nb0, int64_t& nb1, double& c0, double& c1) {
        const int32_t jj = __shfl_sync(0xffffffffu, rowid, i);
        const bool ok = i < nv && __shfl_sync(0xffffffffu, best.i, i) != INT_MAX;
        const int64_t j = ok ? jj : 0;
        nb0 = ok && h0 ? __ldg(&Sr[j * k + t0]) : 0;
        nb1 = ok && h1 ? __ldg(&Sr[j * k + t1]) : 0;
        c0 = ok && h0 ? __ldg(&Cr[j * k + t0]) : 0.0;
        c1 = ok && h1 ? __ldg(&Cr[j * k + t1]) : 0.0;
      };
      auto load_x = [&](int64_t nb0, int64_t nb1, double (&x0)[D], double (&x1)[D]) {
#pragma unroll
        for (int u = 0; u < D; ++u) {
          x0[u] = __ldg(&Xr[nb0 * D + u]);
          x1[u] = __ldg(&Xr[nb1 * D + u]);
        }
      };
      int64_t nbA0, nbA1;
      double cA0, cA1, xA0[D], xA1[D];
      load_sc(0, nbA0, nbA1, cA0, cA1);
      load_x(nbA0, nbA1, xA0, xA1);
      int64_t nbB0, nbB1;
      double cB0, cB1;
      load_sc(1, nbB0, nbB1, cB0, cB1);
      for (int i = 0; i < nv; ++i) {
        // prefetch: X rows of point i + 1, S/C of point i + 2
        double xB0[D], xB1[D];
        load_x(nbB0, nbB1, xB0, xB1);
        int64_t nbC0, nbC1;
        double cC0, cC1;
        load_sc(i + 2, nbC0, nbC1, cC0, cC1);
        double qi[D];
#pragma unroll
        for (int u = 0; u < D; ++u) qi[u] = __shfl_sync(0xffffffffu, q[u], i);
        const bool ok = __shfl_sync(0xffffffffu, best.i, i) != INT_MAX;
        double dq0 = qi[0] - xA0[0], dq1 = qi[0] - xA1[0];
        double s0 = dq0 * dq0, s1 = dq1 * dq1;
#pragma unroll
        for (int u = 1; u < D; ++u) {
          dq0 = qi[u] - xA0[u];
          dq1 = qi[u] - xA1[u];
          s0 = fma(dq0, dq0, s0);
          s1 = fma(dq1, dq1, s1);
        }
        double acc = h0 ? kernel_from_sq_build<KF>(s0, kc, kp, s_exp) * cA0 : 0.0;
        if (h1) acc = fma(kernel_from_sq_build<KF>(s1, kc, kp, s_exp), cA1, acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const int64_t orow_i = __shfl_sync(0xffffffffu, orow, i);
        if (lane == 0 && ok) out[orow_i] = acc + mo;
        nbA0 = nbB0; nbA1 = nbB1; cA0 = cB0; cA1 = cB1;
#pragma unroll
        for (int u = 0; u < D; ++u) {
          xA0[u] = xB0[u];
          xA1[u] = xB1[u];
        }
        nbB0 = nbC0; nbB1 = nbC1; cB0 = cC0; cB1 = cC1;
      }
      continue;
    }
    for (int i = 0; i < nv; ++i) {
      const int32_t jj = __shfl_sync(0xffffffffu, best.i, i);
      const int64_t orow_i = __shfl_sync(0xffffffffu, orow, i);
      if (jj == INT_MAX) continue;
      const int64_t j = jj;
      double qi[D];
#pragma unroll
      for (int u = 0; u < D; ++u) qi[u] = __shfl_sync(0xffffffffu, q[u], i);
      for (int cc = 0; cc < m; ++cc) {
        double acc = 0.0;
        for (int t = lane; t < k; t += kWarp) {
          const int64_t nb = S[j * k + t];
          const double* xn = X + nb * D;
          const double d0 = qi[0] - xn[0];
          double dsq = d0 * d0;
#pragma unroll
          for (int u = 1; u < D; ++u) {
            const double du = qi[u] - xn[u];
            dsq = fma(du, du, dsq);
          }
          acc = fma(kernel_from_sq_build<KF>(dsq, kc, kp, s_exp), Cf[(j * k + t) * m + cc], acc);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[orow_i * m + cc] = acc + mean_offset[cc];
      }
    }
  }
}

// Sorted positions of the query rows: ids in [rb, re), and with cyc_pc > 0
// only the block-cyclic row set of member cyc_r of cyc_g (blocks of cyc_pc
// rows dealt round-robin; the multi-GPU layout of group.cu).
__global__ void compact_rows_kernel(const int32_t* __restrict__ pid, int64_t n, int64_t rb, int64_t re,
                                    int64_t cyc_pc, int cyc_g, int cyc_r,
                                    int32_t* __restrict__ qpos, int32_t* __restrict__ counter) {
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t id = pid[p];
    if (id >= rb && id < re && (cyc_pc == 0 || (id / cyc_pc) % cyc_g == cyc_r)) {
      // warp-aggregated append keeps cell order within each warp's run
      const int32_t s = atomicAdd(counter, 1);
      qpos[s] = static_cast<int32_t>(p);
    }
  }
}

unsigned grid1d(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 64) g = 148 * 64;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

// Device scratch for one counting sort of `n` points into `ncap` cells.
struct SortBufs {
  int32_t *counts = nullptr, *key = nullptr, *slot = nullptr, *cstart = nullptr, *bsums = nullptr;
  int32_t* pid = nullptr;
  double* pts = nullptr;
  int64_t nb = 0;
  cudaError_t alloc(int64_t n, int64_t ncap, int D, cudaStream_t s) {
    nb = (ncap + 1 + kScanBlock * kScanItems - 1) / (kScanBlock * kScanItems);
    cudaError_t e = cudaMallocAsync(&counts, sizeof(int32_t) * (ncap + 1), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&cstart, sizeof(int32_t) * (ncap + 2), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&bsums, sizeof(int32_t) * (nb + 1), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&key, sizeof(int32_t) * (n > 0 ? n : 1), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&slot, sizeof(int32_t) * (n > 0 ? n : 1), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&pid, sizeof(int32_t) * (n > 0 ? n : 1), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&pts, sizeof(double) * (n > 0 ? n : 1) * D, s);
    return e;
  }
  void release(cudaStream_t s) {
    for (void* p : {static_cast<void*>(counts), static_cast<void*>(cstart), static_cast<void*>(bsums),
                    static_cast<void*>(key), static_cast<void*>(slot), static_cast<void*>(pid),
                    static_cast<void*>(pts)})
      if (p) cudaFreeAsync(p, s);
  }
};

// Counting sort of P (np x D) by the cells of `gp`: pts/pid in cell order,
// cstart = cell offsets.
template <int D>
void cell_sort(const double* P, int64_t np, const GridParams* gp, int64_t ncap, SortBufs& b, cudaStream_t s,
               int32_t* pos_of = nullptr) {
  cudaMemsetAsync(b.counts, 0, sizeof(int32_t) * (ncap + 1), s);
  count_kernel<D><<<grid1d(np), 256, 0, s>>>(P, np, gp, b.counts, b.key, b.slot);
  const int64_t m = ncap + 1;
  scan_local_kernel<<<static_cast<unsigned>(b.nb), kScanBlock, 0, s>>>(b.counts, m, b.cstart, b.bsums);
  scan_sums_kernel<<<1, kScanBlock, 0, s>>>(b.bsums, b.nb, b.bsums + b.nb);
  scan_add_kernel<<<static_cast<unsigned>(b.nb), kScanBlock, 0, s>>>(b.cstart, m, b.bsums);
  scatter_kernel<D><<<grid1d(np), 256, 0, s>>>(P, np, b.key, b.slot, b.cstart, b.pts, b.pid, pos_of);
  note_launches(5);
}

template <int D, int E>
void launch_query(const GridParams* gp, const double* pts, const int32_t* pid, const int32_t* cstart, int64_t nq,
                  const int32_t* qpos, const double* Q, const int32_t* qout, const int32_t* excl_arr, int kk,
                  int with_self, int64_t row_offset, int32_t* out, double* out_d, int num_sms, cudaStream_t s) {
  int64_t blocks = (nq * 32 + kQueryThreads - 1) / kQueryThreads;
  const char* ce = std::getenv("FMGP_GQ_CTAS");  // CTAs per SM of the grid-stride query kernel (A/B)
  // 128: only four 8-warp CTAs are resident per SM, so a grid of a few long CTAs per SM ends in a tail of
  // idle SMs (8 per SM: 27 of 32 warps active on average, cfg5 kNN 28.6 ms; 128: 25.9 ms)
  const int per_sm = ce != nullptr && std::atoi(ce) > 0 ? std::atoi(ce) : 128;
  const int64_t cap = static_cast<int64_t>(num_sms) * per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  grid_query_kernel<D, E><<<static_cast<unsigned>(blocks), kQueryThreads, 0, s>>>(
      gp, pts, pid, cstart, nq, qpos, Q, qout, excl_arr, kk, with_self, row_offset, out, out_d);
  note_launches(1);
}

template <int D>
void launch_query_e(int E, const GridParams* gp, const double* pts, const int32_t* pid, const int32_t* cstart,
                    int64_t nq, const int32_t* qpos, const double* Q, const int32_t* qout, const int32_t* excl_arr,
                    int kk, int with_self, int64_t row_offset, int32_t* out, double* out_d, int num_sms,
                    cudaStream_t s) {
  // FMGP_KNN_GRID=thread selects the thread-per-query kernel (A/B checks)
  static const bool thread_mode = [] {
    const char* e = std::getenv("FMGP_KNN_GRID");
    return e != nullptr && std::string(e) == "thread";
  }();
  if (thread_mode && kk <= kThreadMaxK) {
    const size_t smem = static_cast<size_t>(kk) * kThreadQueryThreads * (sizeof(double) + sizeof(int32_t));
    cudaFuncSetAttribute(grid_query_thread_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, grid_query_thread_kernel<D>, kThreadQueryThreads, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t blocks = (nq + kThreadQueryThreads - 1) / kThreadQueryThreads;
    const int64_t cap = static_cast<int64_t>(num_sms) * per_sm;
    if (blocks > cap) blocks = cap;
    grid_query_thread_kernel<D><<<static_cast<unsigned>(blocks), kThreadQueryThreads, smem, s>>>(
        gp, pts, pid, cstart, nq, qpos, Q, qout, excl_arr, kk, with_self, row_offset, out, out_d);
    note_launches(1);
    return;
  }
  if (E == 1)
    launch_query<D, 1>(gp, pts, pid, cstart, nq, qpos, Q, qout, excl_arr, kk, with_self, row_offset, out, out_d,
                          num_sms, s);
  else if (E == 2)
    launch_query<D, 2>(gp, pts, pid, cstart, nq, qpos, Q, qout, excl_arr, kk, with_self, row_offset, out, out_d,
                          num_sms, s);
  else
    launch_query<D, 4>(gp, pts, pid, cstart, nq, qpos, Q, qout, excl_arr, kk, with_self, row_offset, out, out_d,
                          num_sms, s);
}

// cyc_pc > 0 (self mode only): the queries are the block-cyclic row set of
// member cyc_r of cyc_g over all np rows (nq of them), written at their
// global rows of `out` (row_offset 0).
template <int D>
cudaError_t knn_grid_d(const double* Q, int64_t nq, const double* P, int64_t np, int kk, int64_t self_offset,
                       const int32_t* excl_arr, int with_self, int32_t* out, double* out_d, int num_sms,
                       cudaStream_t s, int64_t cyc_pc = 0, int cyc_g = 1, int cyc_r = 0) {
  const int E = kk <= 32 ? 1 : (kk <= 64 ? 2 : 4);
  // Points per cell: enough that the radius-1 block usually holds the kk-th neighbour.
  // Points per cell. d = 1: enough that the radius-1 block usually holds the
  // kk-th neighbour; d = 2, 3: smaller cells for the distance-ordered walk
  // (the 3^D block holds ~1.8 kk in 2-D, ~2.2 kk in 3-D; later cells are
  // skipped by their distance). A/B at cfg2: kk/4 2.54, kk/5 2.40, kk/6 2.44,
  // kk/7 2.58, kk/8 2.85 ms; cfg5: kk/10 29.6, kk/13 29.6, kk/16 29.9,
  // kk/20 31.7 ms.
  static const double div2 = [] {  // FMGP_GRID_DIV2 / FMGP_GRID_DIV3: A/B of the cell size
    const char* e = std::getenv("FMGP_GRID_DIV2");
    return e != nullptr ? std::atof(e) : 5.0;
  }();
  static const double div3 = [] {
    const char* e = std::getenv("FMGP_GRID_DIV3");
    return e != nullptr ? std::atof(e) : 12.0;
  }();
  const double per_cell = (D == 1) ? fmax(4.0, 0.6 * kk) : (D == 2 ? fmax(4.0, kk / div2) : fmax(2.0, kk / div3));
  const int64_t ncap = np;  // cells never exceed the point count
  GridParams* gp = nullptr;
  unsigned long long* mm = nullptr;
  SortBufs pb, qb;
  int32_t *qpos = nullptr, *cnt = nullptr;
  cudaError_t err = cudaMallocAsync(&gp, sizeof(GridParams), s);
  if (err == cudaSuccess) err = cudaMallocAsync(&mm, sizeof(unsigned long long) * 6, s);
  if (err == cudaSuccess) err = pb.alloc(np, ncap, D, s);
  if (err != cudaSuccess) return err;
  // bounding box -> grid parameters -> counting sort of the reference points
  cudaMemsetAsync(mm, 0, sizeof(unsigned long long) * 6, s);
  for (int t = 0; t < D; ++t) cudaMemsetAsync(mm + 2 * t, 0xFF, sizeof(unsigned long long), s);
  bbox_kernel<<<grid1d(np), 256, 0, s>>>(P, np, D, mm);
  grid_params_kernel<<<1, 1, 0, s>>>(mm, np, D, per_cell, ncap, gp);
  note_launches(2);
  cell_sort<D>(P, np, gp, ncap, pb, s);

  const bool self_mode = excl_arr == nullptr && self_offset >= 0 && Q == P + self_offset * D;
  if (cyc_pc > 0) {
    err = cudaMallocAsync(&qpos, sizeof(int32_t) * (nq > 0 ? nq : 1), s);
    if (err == cudaSuccess) err = cudaMallocAsync(&cnt, sizeof(int32_t), s);
    if (err != cudaSuccess) return err;
    cudaMemsetAsync(cnt, 0, sizeof(int32_t), s);
    compact_rows_kernel<<<grid1d(np), 256, 0, s>>>(pb.pid, np, 0, np, cyc_pc, cyc_g, cyc_r, qpos, cnt);
    note_launches(1);
    launch_query_e<D>(E, gp, pb.pts, pb.pid, pb.cstart, nq, qpos, nullptr, nullptr, nullptr, kk, with_self, 0, out,
                      out_d, num_sms, s);
  } else if (self_mode && self_offset == 0 && nq == np) {
    // every training row is a query: walk them in cell order
    launch_query_e<D>(E, gp, pb.pts, pb.pid, pb.cstart, nq, nullptr, nullptr, nullptr, nullptr, kk, with_self, 0,
                      out, out_d, num_sms, s);
  } else if (self_mode) {
    // a row shard: its sorted positions, mostly in cell order
    err = cudaMallocAsync(&qpos, sizeof(int32_t) * (nq > 0 ? nq : 1), s);
    if (err == cudaSuccess) err = cudaMallocAsync(&cnt, sizeof(int32_t), s);
    if (err != cudaSuccess) return err;
    cudaMemsetAsync(cnt, 0, sizeof(int32_t), s);
    compact_rows_kernel<<<grid1d(np), 256, 0, s>>>(pb.pid, np, self_offset, self_offset + nq, 0, 1, 0, qpos, cnt);
    note_launches(1);
    launch_query_e<D>(E, gp, pb.pts, pb.pid, pb.cstart, nq, qpos, nullptr, nullptr, nullptr, kk, with_self,
                      self_offset, out, out_d, num_sms, s);
  } else {
    // external queries (predict): sort them by the same cells for locality
    err = qb.alloc(nq, ncap, D, s);
    if (err != cudaSuccess) return err;
    cell_sort<D>(Q, nq, gp, ncap, qb, s);
    launch_query_e<D>(E, gp, pb.pts, pb.pid, pb.cstart, nq, nullptr, qb.pts, qb.pid, excl_arr, kk, with_self, 0,
                      out, out_d, num_sms, s);
  }
  err = cudaGetLastError();
  cudaFreeAsync(gp, s);
  cudaFreeAsync(mm, s);
  pb.release(s);
  qb.release(s);
  if (qpos) cudaFreeAsync(qpos, s);
  if (cnt) cudaFreeAsync(cnt, s);
  return err;
}

// The training-point grid of the predict walk (bbox -> cubic cells of ~1.5
// points in 2-D, ~1 in 3-D -> counting sort): built per call, or once per
// model handle (PredictGridCache) and reused by every predict on it.
constexpr int64_t kPredictSortMin = 4096;  // test batches at least this large are cell-sorted first

// Grid-ordered copy of a model: row p of (s_pos, c_perm) is training point
// pid[p]'s row of (S, C) with neighbour ids mapped to grid positions. One
// warp per row (k <= 64: lanes t and t + 32).
__global__ void permute_model_kernel(int64_t n, int k, int m, const int32_t* __restrict__ pid,
                                     const int32_t* __restrict__ pos_of, const int32_t* __restrict__ S,
                                     const double* __restrict__ C, int32_t* __restrict__ s_pos,
                                     double* __restrict__ c_perm) {
  const int lane = threadIdx.x & 31;
  for (int64_t p = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; p < n;
       p += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    const int64_t j = pid[p];
    for (int t = lane; t < k; t += 32) s_pos[p * k + t] = pos_of[S[j * k + t]];
    for (int t = lane; t < k * m; t += 32) c_perm[p * k * m + t] = C[j * k * m + t];
  }
}

struct PredictGridCache {
  int d = 0;
  int64_t n = 0;
  GridParams* gp = nullptr;
  SortBufs pb;
  int32_t* pos_of = nullptr;  // n: grid position of training point i (inverse of pb.pid)
  // grid-ordered model (predict_grid_cache_attach): row p = training point
  // pid[p]; neighbour ids as grid positions, so a test point's 1-NN row and
  // the neighbours' coordinates (pb.pts) are read in cell order
  int32_t* s_pos = nullptr;
  double* c_perm = nullptr;
  int pk = 0, pm = 0;
};

template <int D>
cudaError_t build_predict_grid(const double* X, int64_t n, PredictGridCache& g, cudaStream_t s) {
  static const double pc2 = [] {  // FMGP_PGRID_PC2 / FMGP_PGRID_PC3: A/B of the cell size
    const char* e = std::getenv("FMGP_PGRID_PC2");
    return e != nullptr ? std::atof(e) : 1.5;
  }();
  static const double pc3 = [] {
    const char* e = std::getenv("FMGP_PGRID_PC3");
    return e != nullptr ? std::atof(e) : 1.0;
  }();
  const double per_cell = (D == 1) ? 4.0 : (D == 2 ? pc2 : pc3);
  const int64_t ncap = n;
  unsigned long long* mm = nullptr;
  g.d = D;
  g.n = n;
  cudaError_t err = cudaMallocAsync(&g.gp, sizeof(GridParams), s);
  if (err == cudaSuccess) err = cudaMallocAsync(&mm, sizeof(unsigned long long) * 6, s);
  if (err == cudaSuccess) err = g.pb.alloc(n, ncap, D, s);
  if (err != cudaSuccess) return err;
  cudaMemsetAsync(mm, 0, sizeof(unsigned long long) * 6, s);
  for (int t = 0; t < D; ++t) cudaMemsetAsync(mm + 2 * t, 0xFF, sizeof(unsigned long long), s);
  bbox_kernel<<<grid1d(n), 256, 0, s>>>(X, n, D, mm);
  grid_params_kernel<<<1, 1, 0, s>>>(mm, n, D, per_cell, ncap, g.gp);
  note_launches(2);
  err = cudaMallocAsync(&g.pos_of, sizeof(int32_t) * n, s);
  if (err != cudaSuccess) return err;
  cell_sort<D>(X, n, g.gp, ncap, g.pb, s, g.pos_of);
  cudaFreeAsync(mm, s);
  return cudaGetLastError();
}

void release_predict_grid(PredictGridCache& g, cudaStream_t s) {
  if (g.gp) cudaFreeAsync(g.gp, s);
  g.gp = nullptr;
  for (void* p : {static_cast<void*>(g.pos_of), static_cast<void*>(g.s_pos), static_cast<void*>(g.c_perm)})
    if (p) cudaFreeAsync(p, s);
  g.pos_of = g.s_pos = nullptr;
  g.c_perm = nullptr;
  g.pb.release(s);
  g.pb = SortBufs{};
}

// Test points sorted by the same cells (locality), then the fused kernel.
template <int D>
cudaError_t run_predict_grid(const PredictGridCache& g, const double* X, const int32_t* S, const double* Cf, int k,
                             int m, const KParams& kp, const double* mean_offset_dev, const double* Z, int64_t nz,
                             double* out, int32_t* nn_out, int num_sms, cudaStream_t s) {
  // Large batches are sorted by cell for locality; a small one (a few warps'
  // worth, e.g. fast_predict_one) goes in input order: the sort's cell-count
  // scan is O(cells), which would dominate its latency.
  SortBufs qb;
  const double* Qs = Z;
  const int32_t* qo = nullptr;
  cudaError_t err = cudaSuccess;
  if (nz >= kPredictSortMin) {
    err = qb.alloc(nz, g.n, D, s);
    if (err != cudaSuccess) return err;
    cell_sort<D>(Z, nz, g.gp, g.n, qb, s);
    Qs = qb.pts;
    qo = qb.pid;
  }
  int64_t blocks = (nz + kQueryThreads - 1) / kQueryThreads;  // 32 test points per warp
  const char* pce = std::getenv("FMGP_PGRID_CTAS");  // CTAs per SM of the grid-stride predict kernel (A/B)
  const int64_t cap = static_cast<int64_t>(num_sms) * (pce != nullptr && std::atoi(pce) > 0 ? std::atoi(pce) : 256);  // 8 per SM left a tail: cfg5 4.93 -> 4.40 ms
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  // the grid-ordered model replica, when attached to this grid for these S/C shapes
  const bool use_perm = g.s_pos != nullptr && S != nullptr && g.pk == k && g.pm == m && m == 1;
  const int32_t* sp = use_perm ? g.s_pos : nullptr;
  const double* cp = use_perm ? g.c_perm : nullptr;
  static const bool warp_nn = [] {  // FMGP_PGRID_WARP=1: warp-cooperative 1-NN walk for every point (A/B)
    const char* e = std::getenv("FMGP_PGRID_WARP");
    return e != nullptr && e[0] == '1';
  }();
  // lane-per-point gather-kernel-dot (FMGP_PGRID_LANEDOT=0: a warp per point's neighbours, A/B);
  // needs an even k and 8- / 16-byte aligned S / C rows for its vector loads
  const char* ld_env = std::getenv("FMGP_PGRID_LANEDOT");
  const int32_t* s_rows = use_perm ? sp : S;
  const double* c_rows = use_perm ? cp : Cf;
  // (and the cell-ordered model replica: without it the lanes' rows are scattered over the model)
  const int lane_dot = !(ld_env != nullptr && ld_env[0] == '0') && use_perm && (k & 1) == 0 && S != nullptr &&
                       (reinterpret_cast<uintptr_t>(s_rows) & 7) == 0 && (reinterpret_cast<uintptr_t>(c_rows) & 15) == 0;
  switch (kp.kind == 1 ? 0 : 1 + kp.nu_code) {  // kernel_code(), evaluated on the host
#define FMGP_PRED_CASE(KF)                                                                                      \
  case KF:                                                                                                      \
    if (warp_nn)                                                                                                \
      grid_predict_kernel<D, KF, false><<<static_cast<unsigned>(blocks), kQueryThreads, 0, s>>>(                \
          g.gp, g.pb.pts, g.pb.pid, g.pb.cstart, nz, Qs, qo, X, S, Cf, k, m, kp, mean_offset_dev, out, nn_out,    \
          g.pos_of, sp, cp, lane_dot);                                                                                  \
    else                                                                                                        \
      grid_predict_kernel<D, KF, true><<<static_cast<unsigned>(blocks), kQueryThreads, 0, s>>>(                 \
          g.gp, g.pb.pts, g.pb.pid, g.pb.cstart, nz, Qs, qo, X, S, Cf, k, m, kp, mean_offset_dev, out, nn_out,    \
          g.pos_of, sp, cp, lane_dot);                                                                                  \
    break;
    FMGP_PRED_CASE(0)
    FMGP_PRED_CASE(1)
    FMGP_PRED_CASE(2)
    FMGP_PRED_CASE(3)
    default:
      FMGP_PRED_CASE(4)
#undef FMGP_PRED_CASE
  }
  note_launches(1);
  err = cudaGetLastError();
  qb.release(s);
  return err;
}

template <int D>
cudaError_t predict_grid_d(const double* X, int64_t n, const int32_t* S, const double* Cf, int k, int m,
                           const KParams& kp, const double* mean_offset_dev, const double* Z, int64_t nz, double* out,
                           int32_t* nn_out, int num_sms, cudaStream_t s) {
  PredictGridCache g;
  cudaError_t err = build_predict_grid<D>(X, n, g, s);
  if (err == cudaSuccess) err = run_predict_grid<D>(g, X, S, Cf, k, m, kp, mean_offset_dev, Z, nz, out, nn_out, num_sms, s);
  release_predict_grid(g, s);
  return err;
}

}  // namespace

cudaError_t predict_grid(const double* X, int64_t n, int d, const int32_t* S, const double* Cf, int k, int m,
                         const KParams& kp, const double* mean_offset_dev, const double* Z, int64_t nz, double* out,
                         int32_t* nn_out, int num_sms, cudaStream_t stream) {
  if (nz <= 0) return cudaSuccess;
  switch (d) {
    case 1: return predict_grid_d<1>(X, n, S, Cf, k, m, kp, mean_offset_dev, Z, nz, out, nn_out, num_sms, stream);
    case 2: return predict_grid_d<2>(X, n, S, Cf, k, m, kp, mean_offset_dev, Z, nz, out, nn_out, num_sms, stream);
    case 3: return predict_grid_d<3>(X, n, S, Cf, k, m, kp, mean_offset_dev, Z, nz, out, nn_out, num_sms, stream);
    default: return cudaErrorInvalidValue;
  }
}

void* predict_grid_cache_build(const double* X, int64_t n, int d, cudaStream_t stream, cudaError_t* err) {
  *err = cudaErrorInvalidValue;
  if (d < 1 || d > 3 || n < 1) return nullptr;
  auto* g = new PredictGridCache();
  switch (d) {
    case 1: *err = build_predict_grid<1>(X, n, *g, stream); break;
    case 2: *err = build_predict_grid<2>(X, n, *g, stream); break;
    default: *err = build_predict_grid<3>(X, n, *g, stream); break;
  }
  if (*err == cudaSuccess) *err = cudaStreamSynchronize(stream);  // the handle is used from other streams
  if (*err != cudaSuccess) {
    predict_grid_cache_free(g);
    return nullptr;
  }
  return g;
}

void predict_grid_cache_free(void* cache) {
  auto* g = static_cast<PredictGridCache*>(cache);
  if (g == nullptr) return;
  release_predict_grid(*g, 0);
  cudaStreamSynchronize(0);
  delete g;
}

cudaError_t predict_grid_cache_attach(void* cache, const int32_t* S, const double* C, int k, int m,
                                      cudaStream_t stream) {
  auto* g = static_cast<PredictGridCache*>(cache);
  if (g == nullptr || m != 1 || k > 2 * kWarp || g->s_pos != nullptr) return cudaSuccess;
  static const bool off = [] {  // FMGP_PGRID_PERM=0: predict from the model as given (A/B)
    const char* e = std::getenv("FMGP_PGRID_PERM");
    return e != nullptr && e[0] == '0';
  }();
  if (off) return cudaSuccess;
  cudaError_t e = cudaMallocAsync(&g->s_pos, sizeof(int32_t) * g->n * k, stream);
  if (e == cudaSuccess) e = cudaMallocAsync(&g->c_perm, sizeof(double) * g->n * k * m, stream);
  if (e != cudaSuccess) return e;
  const int64_t blocks = std::min<int64_t>((g->n * 32 + 255) / 256, 65535);
  permute_model_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(g->n, k, m, g->pb.pid, g->pos_of, S, C,
                                                                          g->s_pos, g->c_perm);
  note_launches(1);
  g->pk = k;
  g->pm = m;
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  return e;
}

cudaError_t predict_grid_cached(const void* cache, const double* X, const int32_t* S, const double* Cf, int k, int m,
                                const KParams& kp, const double* mean_offset_dev, const double* Z, int64_t nz,
                                double* out, int32_t* nn_out, int num_sms, cudaStream_t stream) {
  const auto* g = static_cast<const PredictGridCache*>(cache);
  if (nz <= 0) return cudaSuccess;
  switch (g->d) {
    case 1: return run_predict_grid<1>(*g, X, S, Cf, k, m, kp, mean_offset_dev, Z, nz, out, nn_out, num_sms, stream);
    case 2: return run_predict_grid<2>(*g, X, S, Cf, k, m, kp, mean_offset_dev, Z, nz, out, nn_out, num_sms, stream);
    default: return run_predict_grid<3>(*g, X, S, Cf, k, m, kp, mean_offset_dev, Z, nz, out, nn_out, num_sms, stream);
  }
}

// Processing order of the fused solve (d <= 3): the rows [0, n) of P sorted by
// a coarse cell grid (~16 points per cell, counting sort), so the warps in
// flight work on spatially close neighbourhoods and their coordinate gathers
// hit L2 instead of HBM. Any permutation gives the same per-row results.
namespace {
__global__ void order_scatter_kernel(int64_t n, const int32_t* __restrict__ key, const int32_t* __restrict__ slot,
                                     const int32_t* __restrict__ start, int32_t* __restrict__ order) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    order[start[key[i]] + slot[i]] = static_cast<int32_t>(i);
}

template <int D>
cudaError_t spatial_order_d(const double* P, int64_t n, int32_t* order, cudaStream_t s) {
  const int64_t ncap = n / 16 + 1;
  GridParams* gp = nullptr;
  unsigned long long* mm = nullptr;
  SortBufs b;
  b.nb = (ncap + 1 + kScanBlock * kScanItems - 1) / (kScanBlock * kScanItems);
  cudaError_t e = cudaMallocAsync(&gp, sizeof(GridParams), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&mm, sizeof(unsigned long long) * 6, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&b.counts, sizeof(int32_t) * (ncap + 1), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&b.cstart, sizeof(int32_t) * (ncap + 2), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&b.bsums, sizeof(int32_t) * (b.nb + 1), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&b.key, sizeof(int32_t) * n, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&b.slot, sizeof(int32_t) * n, s);
  if (e == cudaSuccess) {
    cudaMemsetAsync(mm, 0, sizeof(unsigned long long) * 6, s);
    for (int t = 0; t < D; ++t) cudaMemsetAsync(mm + 2 * t, 0xFF, sizeof(unsigned long long), s);
    bbox_kernel<<<grid1d(n), 256, 0, s>>>(P, n, D, mm);
    grid_params_kernel<<<1, 1, 0, s>>>(mm, n, D, 16.0, ncap, gp);
    cudaMemsetAsync(b.counts, 0, sizeof(int32_t) * (ncap + 1), s);
    count_kernel<D><<<grid1d(n), 256, 0, s>>>(P, n, gp, b.counts, b.key, b.slot);
    const int64_t m = ncap + 1;
    scan_local_kernel<<<static_cast<unsigned>(b.nb), kScanBlock, 0, s>>>(b.counts, m, b.cstart, b.bsums);
    scan_sums_kernel<<<1, kScanBlock, 0, s>>>(b.bsums, b.nb, b.bsums + b.nb);
    scan_add_kernel<<<static_cast<unsigned>(b.nb), kScanBlock, 0, s>>>(b.cstart, m, b.bsums);
    order_scatter_kernel<<<grid1d(n), 256, 0, s>>>(n, b.key, b.slot, b.cstart, order);
    note_launches(7);
    e = cudaGetLastError();
  }
  if (gp) cudaFreeAsync(gp, s);
  if (mm) cudaFreeAsync(mm, s);
  b.release(s);
  return e;
}
}  // namespace

cudaError_t spatial_row_order(const double* P, int64_t n, int d, int32_t* order, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  switch (d) {
    case 1: return spatial_order_d<1>(P, n, order, stream);
    case 2: return spatial_order_d<2>(P, n, order, stream);
    case 3: return spatial_order_d<3>(P, n, order, stream);
    default: return cudaErrorInvalidValue;
  }
}

bool knn_grid_supported(int d, int kk) { return d >= 1 && d <= 3 && kk >= 1 && kk <= 128; }

cudaError_t knn_grid(const double* Q, int64_t nq, const double* P, int64_t np, int d, int kk, int64_t self_offset,
                     const int32_t* excl_arr, int with_self, int32_t* out, double* out_d, int num_sms,
                     cudaStream_t stream) {
  if (nq <= 0) return cudaSuccess;
  switch (d) {
    case 1: return knn_grid_d<1>(Q, nq, P, np, kk, self_offset, excl_arr, with_self, out, out_d, num_sms, stream);
    case 2: return knn_grid_d<2>(Q, nq, P, np, kk, self_offset, excl_arr, with_self, out, out_d, num_sms, stream);
    case 3: return knn_grid_d<3>(Q, nq, P, np, kk, self_offset, excl_arr, with_self, out, out_d, num_sms, stream);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t knn_grid_rows_cyclic(const double* P, int64_t np, int d, int kk, int64_t nrows, int64_t pc, int g, int r,
                                 int32_t* out, int num_sms, cudaStream_t stream) {
  if (nrows <= 0) return cudaSuccess;
  switch (d) {
    case 1: return knn_grid_d<1>(P, nrows, P, np, kk, 0, nullptr, 1, out, nullptr, num_sms, stream, pc, g, r);
    case 2: return knn_grid_d<2>(P, nrows, P, np, kk, 0, nullptr, 1, out, nullptr, num_sms, stream, pc, g, r);
    case 3: return knn_grid_d<3>(P, nrows, P, np, kk, 0, nullptr, 1, out, nullptr, num_sms, stream, pc, g, r);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace fmgp
