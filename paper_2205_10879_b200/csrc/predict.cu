// K3 — predict gather–kernel–dot (bandwidth bound), one warp per test point.
//
// Replaces fast_predict_one's body (proj/core/src/fast_predict.cpp:135-143):
//   acc = sum_{t<k} kernel_value(distance_to(z, S[j,t])) * C[j,t];  acc + mean_offset
// with distance_to = sqrt(dist_sq) (nn_index.cpp:344-349). j is the 1-NN
// index from K1 (nearest_training_point, :351-366). Lanes evaluate the k
// kernel values in parallel; the sum is then accumulated in the reference's
// sequential t order (shuffle chain), so the only deviation from the CPU is
// the last-ulp behaviour of exp().
#include "fmgp_common.cuh"
#include "fmgp_internal.h"

namespace fmgp {

namespace {

constexpr int kPredWarps = 8;

__global__ void __launch_bounds__(kPredWarps * kWarp)
predict_kernel(const double* __restrict__ X, const int32_t* __restrict__ S, const double* __restrict__ C,
               int d, int k, int m, KParams kp, const double* __restrict__ mean_offset,
               const double* __restrict__ Z, int64_t nz, const int32_t* __restrict__ nn,
               double* __restrict__ out) {
  const int lane = threadIdx.x % kWarp;
  const int64_t warp_global = static_cast<int64_t>(blockIdx.x) * kPredWarps + threadIdx.x / kWarp;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kPredWarps;
  for (int64_t zi = warp_global; zi < nz; zi += nwarps) {
    const int64_t j = nn[zi];
    const double* z = Z + zi * d;
    for (int c = 0; c < m; ++c) {
      double acc = 0.0;
      for (int t0 = 0; t0 < k; t0 += kWarp) {
        const int t = t0 + lane;
        double prod = 0.0;
        if (t < k) {
          const int64_t nb = S[j * k + t];
          const double dist = sqrt(dist_sq_dyn(z, X + nb * d, d));
          prod = __dmul_rn(kernel_eval(dist, kp), C[(j * k + t) * m + c]);
        }
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
  int64_t grid = std::min<int64_t>(need, static_cast<int64_t>(num_sms) * 8);
  predict_kernel<<<static_cast<unsigned>(grid), kPredWarps * kWarp, 0, stream>>>(X, S, C, d, k, m, kp,
                                                                                 mean_offset_dev, Z, nz, nn, out);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace fmgp
