// K1 — exact k-nearest-neighbour search (brute force), bit-exact with the
// reference's Exact NeighborIndex (proj/core/src/nn_index.cpp:254-287 query_knn,
// :351-366 nearest_training_point).
//
// The ranking key is the reference's computed fp64 dist_sq (sequential
// sum of (q_t - p_t)^2, no FMA; nn_index.cpp:73-81) with ties broken by the
// lower index. Each (query, reference-chunk) pair keeps a sorted top-kk list;
// references are scanned in ascending index inside a chunk, so a candidate
// equal to the current kk-th distance always has the larger index and is
// rejected (strict <), exactly like the reference's max-heap (:276-281).
// Chunks are merged by (dist, idx) in knn_merge_kernel.
//
// Two scan kernels:
//  * knn_scan_reg<D> (d <= 8): one thread per query (QPT queries per thread,
//    coordinates in registers); reference tiles are staged in shared memory
//    and broadcast. FP64-pipe bound: 3d-1 DFMA-pipe ops + 1 compare per pair.
//  * knn_scan_tiled (any d): 64x64 (query, ref) tiles, 4x4 register blocking,
//    dims streamed through shared memory in 8-wide chunks; per-pair sums stay
//    in ascending-t order so the key is still bit-exact.
#include <cfloat>
#include <climits>
#include <cstdlib>
#include <string>

#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

constexpr int kScanThreads = 128;
constexpr int kRegTile = 256;   // references per shared-memory tile
constexpr int kQPT = 2;         // queries per thread (register kernel)

// Insert (s, j) into the sorted list (ld, li) of length cnt <= kk, where j is
// larger than every index already present. Updates thr to the kk-th distance
// once the list is full.
__device__ __forceinline__ void list_insert(double* ld, int32_t* li, int& cnt, int kk, double s,
                                            int32_t j, double& thr) {
  int pos = cnt < kk ? cnt : kk - 1;
  while (pos > 0) {
    double pd = ld[pos - 1];
    if (pd > s) {
      ld[pos] = pd;
      li[pos] = li[pos - 1];
      --pos;
    } else {
      break;
    }
  }
  ld[pos] = s;
  li[pos] = j;
  if (cnt < kk) ++cnt;
  if (cnt == kk) thr = ld[kk - 1];
}

template <int D>
__global__ void __launch_bounds__(kScanThreads)
knn_scan_reg(const double* __restrict__ Q, int64_t nq, const double* __restrict__ P, int64_t np,
             int kk, int64_t self_offset, const int32_t* __restrict__ excl_arr, int nchunks,
             int64_t chunk_len, double* __restrict__ wd, int32_t* __restrict__ wi) {
  __shared__ double sp[kRegTile * D];
  const int chunk = blockIdx.y;
  const int64_t r0 = static_cast<int64_t>(chunk) * chunk_len;
  const int64_t r1 = min(np, r0 + chunk_len);

  double q[kQPT][D];
  double thr[kQPT];
  int cnt[kQPT];
  int64_t excl[kQPT];
  int64_t base[kQPT];
  bool valid[kQPT];
#pragma unroll
  for (int u = 0; u < kQPT; ++u) {
    int64_t qi = static_cast<int64_t>(blockIdx.x) * kScanThreads * kQPT + u * kScanThreads + threadIdx.x;
    valid[u] = qi < nq;
#pragma unroll
    for (int c = 0; c < D; ++c) q[u][c] = valid[u] ? Q[qi * D + c] : 0.0;
    thr[u] = valid[u] ? INFINITY : -INFINITY;  // -inf never admits a candidate
    cnt[u] = 0;
    excl[u] = excl_arr != nullptr ? (valid[u] ? excl_arr[qi] : -1) : ((self_offset >= 0) ? qi + self_offset : -1);
    base[u] = (qi * nchunks + chunk) * kk;
  }

  for (int64_t t0 = r0; t0 < r1; t0 += kRegTile) {
    const int nt = static_cast<int>((r1 - t0 < kRegTile ? r1 - t0 : kRegTile));
    __syncthreads();
    for (int e = threadIdx.x; e < nt * D; e += kScanThreads) sp[e] = P[t0 * D + e];
    __syncthreads();
    for (int r = 0; r < nt; ++r) {
      double p[D];
#pragma unroll
      for (int c = 0; c < D; ++c) p[c] = sp[r * D + c];
#pragma unroll
      for (int u = 0; u < kQPT; ++u) {
        double s = dist_sq_fixed<D>(q[u], p);
        if (s < thr[u]) {
          int64_t j = t0 + r;
          if (j != excl[u]) list_insert(wd + base[u], wi + base[u], cnt[u], kk, s, static_cast<int32_t>(j), thr[u]);
        }
      }
    }
  }
  // Pad short lists (a chunk with fewer than kk admissible references).
#pragma unroll
  for (int u = 0; u < kQPT; ++u) {
    if (!valid[u]) continue;
    for (int t = cnt[u]; t < kk; ++t) {
      wd[base[u] + t] = INFINITY;
      wi[base[u] + t] = INT_MAX;
    }
  }
}

constexpr int kTileQ = 64;
constexpr int kTileR = 64;
constexpr int kTileD = 8;
constexpr int kTiledThreads = 256;

__global__ void __launch_bounds__(kTiledThreads)
knn_scan_tiled(const double* __restrict__ Q, int64_t nq, const double* __restrict__ P, int64_t np, int d,
               int kk, int64_t self_offset, const int32_t* __restrict__ excl_arr, int nchunks,
               int64_t chunk_len, double* __restrict__ wd, int32_t* __restrict__ wi) {
  __shared__ double qs[kTileD][kTileQ + 1];
  __shared__ double ps[kTileD][kTileR + 1];
  __shared__ double dt[kTileQ][kTileR + 1];
  const int chunk = blockIdx.y;
  const int64_t r0 = static_cast<int64_t>(chunk) * chunk_len;
  const int64_t r1 = min(np, r0 + chunk_len);
  const int64_t q0 = static_cast<int64_t>(blockIdx.x) * kTileQ;
  const int tid = threadIdx.x;
  const int tq = tid / 16;  // 16 x 16 thread grid, 4 x 4 pairs each
  const int tr = tid % 16;

  // Owner state (threads 0..63 own one query each).
  int cnt = 0;
  double thr = INFINITY;
  const int64_t my_q = q0 + tid;
  const bool owner = tid < kTileQ && my_q < nq;
  const int64_t my_excl = excl_arr != nullptr ? (owner ? excl_arr[my_q] : -1)
                                               : (self_offset >= 0 ? my_q + self_offset : -1);
  const int64_t my_base = (my_q * nchunks + chunk) * kk;

  for (int64_t t0 = r0; t0 < r1; t0 += kTileR) {
    const int nr = static_cast<int>((r1 - t0 < kTileR ? r1 - t0 : kTileR));
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int c0 = 0; c0 < d; c0 += kTileD) {
      const int dc = min(kTileD, d - c0);
      __syncthreads();
      for (int e = tid; e < kTileQ * kTileD; e += kTiledThreads) {
        int qq = e / kTileD, c = e % kTileD;
        int64_t gq = q0 + qq;
        qs[c][qq] = (c < dc && gq < nq) ? Q[gq * d + c0 + c] : 0.0;
        int64_t gr = t0 + qq;
        ps[c][qq] = (c < dc && qq < nr) ? P[gr * d + c0 + c] : 0.0;
      }
      __syncthreads();
      for (int c = 0; c < dc; ++c) {
        double qa[4], pb[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) qa[a] = qs[c][tq * 4 + a];
#pragma unroll
        for (int b = 0; b < 4; ++b) pb[b] = ps[c][tr * 4 + b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            double diff = __dsub_rn(qa[a], pb[b]);
            acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(diff, diff));
          }
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dt[tq * 4 + a][tr * 4 + b] = acc[a][b];
    __syncthreads();
    if (owner) {
      for (int r = 0; r < nr; ++r) {
        double s = dt[tid][r];
        if (s < thr) {
          int64_t j = t0 + r;
          if (j != my_excl) list_insert(wd + my_base, wi + my_base, cnt, kk, s, static_cast<int32_t>(j), thr);
        }
      }
    }
  }
  if (owner) {
    for (int t = cnt; t < kk; ++t) {
      wd[my_base + t] = INFINITY;
      wi[my_base + t] = INT_MAX;
    }
  }
}

// Merge the nchunks sorted lists of each query by (dist, idx) and write the
// output row. with_self: row = [q + self_offset, top kk] (precompute's
// S[i,0] = i, fast_predict.cpp:90); otherwise row = [top kk].
__global__ void knn_merge_kernel(const double* __restrict__ wd, const int32_t* __restrict__ wi, int64_t nq,
                                 int nchunks, int kk, int with_self, int64_t self_offset,
                                 int32_t* __restrict__ out, double* __restrict__ out_d) {
  int64_t qi = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (qi >= nq) return;
  const int width = kk + (with_self ? 1 : 0);
  int32_t* row = out + qi * width;
  int o = 0;
  if (with_self) row[o++] = static_cast<int32_t>(qi + self_offset);
  if (nchunks == 1) {
    const int64_t b = qi * kk;
    for (int t = 0; t < kk; ++t) {
      row[o + t] = wi[b + t];
      if (out_d) out_d[qi * kk + t] = wd[b + t];
    }
    return;
  }
  int head[64];
  for (int c = 0; c < nchunks; ++c) head[c] = 0;
  for (int t = 0; t < kk; ++t) {
    int best = -1;
    double bd = INFINITY;
    int32_t bi = INT_MAX;
    for (int c = 0; c < nchunks; ++c) {
      if (head[c] >= kk) continue;
      int64_t e = (qi * nchunks + c) * kk + head[c];
      double dd = wd[e];
      int32_t ii = wi[e];
      if (best < 0 || pair_less(dd, ii, bd, bi)) {
        best = c;
        bd = dd;
        bi = ii;
      }
    }
    head[best]++;
    row[o + t] = bi;
    if (out_d) out_d[qi * kk + t] = bd;
  }
}

// Merge for many chunks (few queries, e.g. the tensor-core path's overflow
// redo): one warp per query, each lane owns chunks lane, lane+32, ...; every
// output step is a warp-wide (key, index) argmin over the lanes' heads.
__global__ void knn_merge_warp_kernel(const double* __restrict__ wd, const int32_t* __restrict__ wi, int64_t nq,
                                      int nchunks, int kk, int with_self, int64_t self_offset,
                                      int32_t* __restrict__ out, double* __restrict__ out_d) {
  const int lane = threadIdx.x & 31;
  const int64_t qi = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (qi >= nq) return;
  const int width = kk + (with_self ? 1 : 0);
  int32_t* row = out + qi * width;
  int o = 0;
  if (with_self) {
    if (lane == 0) row[0] = static_cast<int32_t>(qi + self_offset);
    o = 1;
  }
  constexpr int kMaxPerLane = 16;  // nchunks <= 512
  int head[kMaxPerLane];
#pragma unroll
  for (int s = 0; s < kMaxPerLane; ++s) head[s] = 0;
  for (int t = 0; t < kk; ++t) {
    // this lane's best head
    double bd = INFINITY;
    int32_t bi = INT_MAX;
    int bs = -1;
#pragma unroll
    for (int s = 0; s < kMaxPerLane; ++s) {
      const int c = s * 32 + lane;
      if (c >= nchunks || head[s] >= kk) continue;
      const int64_t e = (qi * nchunks + c) * kk + head[s];
      const double dd = wd[e];
      const int32_t ii = wi[e];
      if (bs < 0 || pair_less(dd, ii, bd, bi)) {
        bd = dd;
        bi = ii;
        bs = s;
      }
    }
    double wdv = bd;
    int32_t wiv = bi;
    for (int off = 16; off > 0; off >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, wdv, off);
      const int32_t oi = __shfl_xor_sync(0xffffffffu, wiv, off);
      if (pair_less(od, oi, wdv, wiv)) {
        wdv = od;
        wiv = oi;
      }
    }
    // the winning head advances (indices are unique across chunks)
    if (bs >= 0 && bi == wiv && bd == wdv) {
#pragma unroll
      for (int s = 0; s < kMaxPerLane; ++s)
        if (s == bs) ++head[s];
    }
    if (lane == 0) {
      row[o + t] = wiv;
      if (out_d) out_d[qi * kk + t] = wdv;
    }
  }
}

}  // namespace

cudaError_t knn_bruteforce(const double* Q, int64_t nq, const double* P, int64_t np, int d, int kk,
                           int64_t self_offset, const int32_t* excl_arr, int with_self, int32_t* out,
                           double* out_d, int num_sms, cudaStream_t stream) {
  if (nq <= 0) return cudaSuccess;
  // Enough (query, chunk) work items for ~2 waves of the whole chip.
  const bool reg = d <= 8;
  const int64_t per_block = reg ? static_cast<int64_t>(kScanThreads) * kQPT : kTileQ;
  const int64_t qblocks = (nq + per_block - 1) / per_block;
  const int64_t want_blocks = static_cast<int64_t>(num_sms) * (reg ? 16 : 4);
  // few query blocks (e.g. the tensor-core overflow redo): many point chunks, warp merge
  const int max_chunks = qblocks * 64 < want_blocks ? 512 : 64;
  int nchunks = static_cast<int>(std::min<int64_t>(max_chunks, std::max<int64_t>(1, want_blocks / qblocks)));
  // Every chunk must hold at least kk admissible references.
  while (nchunks > 1 && np / nchunks < 2 * (kk + 1)) --nchunks;
  const int64_t chunk_len = (np + nchunks - 1) / nchunks;

  double* wd = nullptr;
  int32_t* wi = nullptr;
  const size_t nent = static_cast<size_t>(nq) * nchunks * kk;
  cudaError_t err = cudaMallocAsync(&wd, nent * sizeof(double), stream);
  if (err != cudaSuccess) return err;
  err = cudaMallocAsync(&wi, nent * sizeof(int32_t), stream);
  if (err != cudaSuccess) return err;

  dim3 grid(static_cast<unsigned>(qblocks), static_cast<unsigned>(nchunks));
  if (reg) {
    switch (d) {
#define FMGP_KNN_CASE(DD)                                                                          \
  case DD:                                                                                         \
    knn_scan_reg<DD><<<grid, kScanThreads, 0, stream>>>(Q, nq, P, np, kk, self_offset, excl_arr,   \
                                                        nchunks, chunk_len, wd, wi);               \
    break;
      FMGP_KNN_CASE(1) FMGP_KNN_CASE(2) FMGP_KNN_CASE(3) FMGP_KNN_CASE(4)
      FMGP_KNN_CASE(5) FMGP_KNN_CASE(6) FMGP_KNN_CASE(7) FMGP_KNN_CASE(8)
#undef FMGP_KNN_CASE
    }
  } else {
    knn_scan_tiled<<<grid, kTiledThreads, 0, stream>>>(Q, nq, P, np, d, kk, self_offset, excl_arr, nchunks,
                                                       chunk_len, wd, wi);
  }
  note_launches(1);
  err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  if (nchunks > 64)
    knn_merge_warp_kernel<<<static_cast<unsigned>((nq * 32 + 127) / 128), 128, 0, stream>>>(
        wd, wi, nq, nchunks, kk, with_self, self_offset, out, out_d);
  else
    knn_merge_kernel<<<static_cast<unsigned>((nq + 127) / 128), 128, 0, stream>>>(
        wd, wi, nq, nchunks, kk, with_self, self_offset, out, out_d);
  note_launches(1);
  err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  cudaFreeAsync(wd, stream);
  cudaFreeAsync(wi, stream);
  return cudaGetLastError();
}

}  // namespace fmgp

namespace fmgp {

cudaError_t knn_exact(const double* Q, int64_t nq, const double* P, int64_t np, int d, int kk, int64_t self_offset,
                      const int32_t* excl_arr, int with_self, int32_t* out, double* out_d, int num_sms,
                      cudaStream_t stream) {
  // FMGP_KNN = brute forces the fp64 brute-force scan (A/B checks).
  static const bool force_brute = [] {
    const char* e = std::getenv("FMGP_KNN");
    return e != nullptr && std::string(e) == "brute";
  }();
  if (!force_brute && knn_grid_supported(d, kk))
    return knn_grid(Q, nq, P, np, d, kk, self_offset, excl_arr, with_self, out, out_d, num_sms, stream);
  if (!force_brute && knn_tc_supported(d, kk))
    return knn_tc(Q, nq, P, np, d, kk, self_offset, excl_arr, with_self, out, out_d, num_sms, stream, nullptr);
  return knn_bruteforce(Q, nq, P, np, d, kk, self_offset, excl_arr, with_self, out, out_d, num_sms, stream);
}

}  // namespace fmgp
