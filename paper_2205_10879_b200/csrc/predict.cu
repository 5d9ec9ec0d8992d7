// K3 — predict gather–kernel–dot (bandwidth bound), one warp per test point.
//
// Replaces fast_predict_one's body (proj/core/src/fast_predict.cpp:135-143):
//   acc = sum_{t<k} kernel_value(distance_to(z, S[j,t])) * C[j,t];  acc + mean_offset
// with distance_to = sqrt(dist_sq) (nn_index.cpp:344-349). j is the 1-NN
// index from K1 (nearest_training_point, :351-366). The k kernel values are
// computed once per test point (lanes in parallel for small d; for d >= 32 the
// warp computes each distance cooperatively with coalesced row loads, tree
// reduction order) and reused for every output column; each sum is then
// accumulated in the reference's sequential t order (shuffle chain).
#include <climits>

#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

constexpr int kPredWarps = 8;
constexpr int kMaxKv = 4;  // kernel values held per lane (k <= 128); larger k recomputes per output

// Kernel value k(z, x_nb) for neighbour slot t: lane-private distance for small
// d (sequential dist_sq, the reference's key order), or a warp-cooperative
// distance for large d (coalesced row loads, tree reduction). Returns the value
// on lane (t % 32) of the cooperative path and on every lane of the private one.
__device__ __forceinline__ double neighbour_kernel(const double* __restrict__ X, const double* z, int64_t nb, int d,
                                                   bool coop, int lane, const KParams& kp) {
  if (!coop) return kernel_eval(sqrt(dist_sq_dyn(z, X + nb * d, d)), kp);
  const double* x = X + nb * d;
  double part = 0.0;
  for (int c = lane; c < d; c += kWarp) {
    const double e = z[c] - x[c];
    part = fma(e, e, part);
  }
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  return kernel_eval(sqrt(part), kp);
}

__global__ void __launch_bounds__(kPredWarps * kWarp)
predict_kernel(const double* __restrict__ X, const int32_t* __restrict__ S, const double* __restrict__ C,
               int d, int k, int m, KParams kp, const double* __restrict__ mean_offset,
               const double* __restrict__ Z, int64_t nz, const int32_t* __restrict__ nn,
               double* __restrict__ out) {
  const int lane = threadIdx.x % kWarp;
  const int64_t warp_global = static_cast<int64_t>(blockIdx.x) * kPredWarps + threadIdx.x / kWarp;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kPredWarps;
  const bool coop = d >= kWarp;
  for (int64_t zi = warp_global; zi < nz; zi += nwarps) {
    const int64_t j = nn[zi];
    if (j < 0 || j == INT_MAX) {  // no nearest point (non-finite or overflowing z): NaN, no gather
      for (int c = lane; c < m; c += kWarp) out[zi * m + c] = __longlong_as_double(0x7ff8000000000000ll);
      continue;
    }
    const double* z = Z + zi * d;
    // kernel values of the k neighbours, once per test point: lane l holds t = l + 32 s
    double kv[kMaxKv];
#pragma unroll
    for (int s = 0; s < kMaxKv; ++s) kv[s] = 0.0;
    const bool held = k <= kMaxKv * kWarp;
    if (held) {
      if (coop) {
        for (int t = 0; t < k; ++t) {  // warp-uniform: one cooperative distance per neighbour
          const double v = neighbour_kernel(X, z, S[j * k + t], d, true, lane, kp);
#pragma unroll
          for (int s = 0; s < kMaxKv; ++s)
            if ((t >> 5) == s && (t & 31) == lane) kv[s] = v;
        }
      } else {
#pragma unroll
        for (int s = 0; s < kMaxKv; ++s) {
          const int t = s * kWarp + lane;
          if (t < k) kv[s] = neighbour_kernel(X, z, S[j * k + t], d, false, lane, kp);
        }
      }
    }
    for (int c = 0; c < m; ++c) {
      double acc = 0.0;
      for (int t0 = 0; t0 < k; t0 += kWarp) {
        const int t = t0 + lane;
        double kval = 0.0;
        if (held) {
#pragma unroll
          for (int s = 0; s < kMaxKv; ++s)
            if ((t0 >> 5) == s) kval = kv[s];
        } else if (coop) {
          for (int tt = t0; tt < min(k, t0 + kWarp); ++tt) {
            const double v = neighbour_kernel(X, z, S[j * k + tt], d, true, lane, kp);
            if (tt == t) kval = v;
          }
        } else if (t < k) {
          kval = neighbour_kernel(X, z, S[j * k + t], d, false, lane, kp);
        }
        const double prod = t < k ? __dmul_rn(kval, C[(j * k + t) * m + c]) : 0.0;
        const int cnt = min(kWarp, k - t0);
        for (int s = 0; s < cnt; ++s) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, prod, s));
      }
      if (lane == 0) out[zi * m + c] = __dadd_rn(acc, mean_offset[c]);
    }
  }
}

}  // namespace

cudaError_t predict_gather(const double* X, const int32_t* S, const double* C, int d, int k, int m,
                           const KParams& kp, const double* mean_offset_dev, const double* Z, int64_t nz,
                           const int32_t* nn, double* out, int num_sms, cudaStream_t stream) {
  if (nz <= 0) return cudaSuccess;
  int64_t need = (nz + kPredWarps - 1) / kPredWarps;
  int64_t grid = std::min<int64_t>(need, static_cast<int64_t>(num_sms) * 64);  // many short CTAs: no tail of idle SMs
  predict_kernel<<<static_cast<unsigned>(grid), kPredWarps * kWarp, 0, stream>>>(X, S, C, d, k, m, kp,
                                                                                 mean_offset_dev, Z, nz, nn, out);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace fmgp
