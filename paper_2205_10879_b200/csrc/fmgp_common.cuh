// Shared device helpers for the FastMuyGPs B200 path (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fmgp {

constexpr int kWarp = 32;
constexpr int kMaxK = 160;  // largest neighbourhood the fused solve stages in smem

// Kernel hyper-parameters as the device sees them. kind: 0 Matern, 1 RBF
// (kernel.hpp:7). `diag` = sigma^2 (1 + tau^2), the d == 0 value
// (kernel.cpp:58-60, :81-83); diag_jit[a] is the diagonal after jitter
// attempt a of linalg.cpp:13-19 (cumulative `+= jitter - previous`).
struct KParams {
  int kind;
  int nu_code;  // 0: nu=0.5, 1: nu=1.5, 2: nu=2.5 (Matern); unused for RBF
  double s2, rho, diag;
  double diag_jit[4];
};

// The reference's neighbour key, nn_index.cpp:73-81: s = 0; s += diff*diff in
// ascending t, with no FMA contraction (explicit _rn intrinsics). The first
// step 0 + x == x exactly, so it starts from diff0*diff0.
template <int D>
__device__ __forceinline__ double dist_sq_fixed(const double* a, const double* b) {
  double diff = __dsub_rn(a[0], b[0]);
  double s = __dmul_rn(diff, diff);
#pragma unroll
  for (int t = 1; t < D; ++t) {
    diff = __dsub_rn(a[t], b[t]);
    s = __dadd_rn(s, __dmul_rn(diff, diff));
  }
  return s;
}

__device__ __forceinline__ double dist_sq_dyn(const double* a, const double* b, int d) {
  double s = 0.0;
  for (int t = 0; t < d; ++t) {
    double diff = __dsub_rn(a[t], b[t]);
    s = __dadd_rn(s, __dmul_rn(diff, diff));
  }
  return s;
}

// kernel_value(dist) (kernel.cpp:55-90), evaluated in the reference's
// left-to-right operation order with contraction disabled; exp() is CUDA's
// (within 1 ulp of glibc).
__device__ __forceinline__ double kernel_eval(double dist, const KParams& p) {
  if (dist == 0.0) return p.diag;
  double br;
  if (p.kind == 1) {  // rbf_value :78-86 — s2 * exp(-0.5 * u * u)
    double u = __ddiv_rn(dist, p.rho);
    br = exp(__dmul_rn(__dmul_rn(-0.5, u), u));
  } else if (p.nu_code == 0) {  // exp(-d / rho)
    br = exp(__ddiv_rn(-dist, p.rho));
  } else if (p.nu_code == 1) {  // a = sqrt(3) d / rho; (1 + a) e^{-a}
    double a = __ddiv_rn(__dmul_rn(1.7320508075688772, dist), p.rho);
    br = __dmul_rn(__dadd_rn(1.0, a), exp(-a));
  } else {  // a = sqrt(5) d / rho; (1 + a + a^2/3) e^{-a}
    double a = __ddiv_rn(__dmul_rn(2.2360679774997898, dist), p.rho);
    br = __dmul_rn(__dadd_rn(__dadd_rn(1.0, a), __ddiv_rn(__dmul_rn(a, a), 3.0)), exp(-a));
  }
  return __dmul_rn(p.s2, br);
}

// (dist, idx) lexicographic order of std::pair<double,int> (nn_index.cpp:275-281, :363).
__device__ __forceinline__ bool pair_less(double da, int32_t ia, double db, int32_t ib) {
  return da < db || (da == db && ia < ib);
}

}  // namespace fmgp
