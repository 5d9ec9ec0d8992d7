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
  int nu_code;  // 0: nu=0.5, 1: nu=1.5, 2: nu=2.5, 3: general nu (Matern); unused for RBF
  double s2, rho, diag;
  double diag_jit[4];
  // general nu (kernel.cpp:40-51, :72-74): x = sqrt(2 nu) d / rho and
  // log bracket = c0 + nu log x + log K_nu(x), c0 = (1 - nu) ln 2 - lgamma(nu)
  // (host-evaluated with the reference's own std:: calls).
  double nu, sqrt2nu, c0;
  double inv_rho;  // 1 / rho, for the kernel-matrix build (kernel_eval_fast)
};

// log K_nu(x) for x > 0, nu >= 0 — the quantity the reference takes from
// GSL's gsl_sf_bessel_lnKnu_e (kernel.cpp:42). Own implementation:
// K_mu and K_{mu+1} for mu = nu - round(nu) in [-1/2, 1/2) from Temme's
// series (x <= 2) or Steed's continued fraction CF2 (x > 2), then the stable
// upward recurrence K_{m+1} = 2m/x K_m + K_{m-1}, with a running log scale so
// large nu cannot overflow. The 1/Gamma(1 +- mu) terms of Temme's series come
// from the zeta-series of log Gamma(1+z) split into even/odd parts, which
// keeps gam1 = (1/G(1-mu) - 1/G(1+mu)) / (2 mu) free of cancellation.
// zeta(k), k = 2..10 (index k); larger k are summed directly.
__constant__ double kZeta[11] = {0, 0, 1.6449340668482264, 1.2020569031595943, 1.0823232337111382,
                                 1.0369277551433699, 1.0173430619844491, 1.0083492773819228, 1.0040773561979443,
                                 1.0020083928260822, 1.0009945751278181};

__device__ inline double ln_bessel_k(double nu, double x) {
  const double kEps = 1e-16;
  const double kEuler = 0.57721566490153286061;
  const double kPi = 3.14159265358979323846;
  const int nl = static_cast<int>(nu + 0.5);
  const double mu = nu - nl;
  const double mu2 = mu * mu;
  const double xi = 1.0 / x, xi2 = 2.0 * xi;
  double rkmu, rk1;
  if (x < 2.0) {
    double even = 0.0, odd_over_mu = kEuler, pw = mu;  // pw = mu^(k-1)
    for (int k = 2; k <= 60; ++k) {
      double z;
      if (k <= 10) {
        z = kZeta[k];
      } else {
        z = 1.0;
        for (int j = 2; j <= 12; ++j) z += pow(static_cast<double>(j), -static_cast<double>(k));
      }
      pw *= (k == 2 ? 1.0 : mu);  // mu^(k-1) for k >= 2 starting at mu^1
      const double term = z / k;
      if (k % 2 == 0) even -= term * pw * mu;   // -zeta(k) mu^k / k
      else odd_over_mu += term * pw;            // zeta(k) mu^(k-1) / k
      if (fabs(term * pw) < 1e-18) break;
    }
    const double odd = odd_over_mu * mu;
    const double eev = exp(even);
    const double shc = fabs(odd) < 1e-8 ? 1.0 + odd * odd / 6.0 : sinh(odd) / odd;
    const double gam1 = -eev * shc * odd_over_mu;     // (1/G(1-mu) - 1/G(1+mu)) / (2 mu)
    const double gam2 = eev * cosh(odd);              // (1/G(1-mu) + 1/G(1+mu)) / 2
    const double gampl = exp(even + odd);             // 1/G(1+mu)
    const double gammi = exp(even - odd);             // 1/G(1-mu)
    const double x2 = 0.5 * x;
    const double pimu = kPi * mu;
    const double fact = fabs(pimu) < kEps ? 1.0 : pimu / sin(pimu);
    double d = -log(x2);
    double e = mu * d;
    const double fact2 = fabs(e) < kEps ? 1.0 : sinh(e) / e;
    double ff = fact * (gam1 * cosh(e) + gam2 * fact2 * d);
    double sum = ff;
    e = exp(e);
    double p = 0.5 * e / gampl;
    double q = 0.5 / (e * gammi);
    double c = 1.0;
    d = x2 * x2;
    double sum1 = p;
    for (int i = 1; i < 1000; ++i) {
      ff = (i * ff + p + q) / (i * static_cast<double>(i) - mu2);
      c *= d / i;
      p /= (i - mu);
      q /= (i + mu);
      const double del = c * ff;
      sum += del;
      sum1 += c * (p - i * ff);
      if (fabs(del) < fabs(sum) * kEps) break;
    }
    rkmu = sum;
    rk1 = sum1 * xi2;
  } else {
    double b = 2.0 * (1.0 + x);
    double d = 1.0 / b;
    double h = d, delh = d;
    double q1 = 0.0, q2 = 1.0;
    const double a1 = 0.25 - mu2;
    double q = a1, c = a1, a = -a1;
    double s = 1.0 + q * delh;
    for (int i = 2; i < 100000; ++i) {
      a -= 2 * (i - 1);
      c = -a * c / i;
      const double qnew = (q1 - b * q2) / a;
      q1 = q2;
      q2 = qnew;
      q += c * qnew;
      b += 2.0;
      d = 1.0 / (b + a * d);
      delh = (b * d - 1.0) * delh;
      h += delh;
      const double dels = q * delh;
      s += dels;
      if (fabs(dels / s) < kEps) break;
    }
    h = a1 * h;
    rkmu = sqrt(kPi / (2.0 * x)) * exp(-x) / s;
    rk1 = rkmu * (mu + x + 0.5 - h) * xi;
  }
  double logscale = 0.0;
  for (int i = 1; i <= nl; ++i) {
    const double t = (mu + i) * xi2 * rk1 + rkmu;
    rkmu = rk1;
    rk1 = t;
    if (rk1 > 1e250) {
      rkmu *= 1e-250;
      rk1 *= 1e-250;
      logscale += 575.64627324851142;  // 250 ln 10
    }
  }
  return log(rkmu) + logscale;
}

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
  } else if (p.nu_code == 2) {  // a = sqrt(5) d / rho; (1 + a + a^2/3) e^{-a}
    double a = __ddiv_rn(__dmul_rn(2.2360679774997898, dist), p.rho);
    br = __dmul_rn(__dadd_rn(__dadd_rn(1.0, a), __ddiv_rn(__dmul_rn(a, a), 3.0)), exp(-a));
  } else {  // general nu: exp(c0 + nu log x + log K_nu(x)), x = sqrt(2 nu) d / rho
    double x = __ddiv_rn(__dmul_rn(p.sqrt2nu, dist), p.rho);
    br = exp(__dadd_rn(__dadd_rn(p.c0, __dmul_rn(p.nu, log(x))), ln_bessel_k(p.nu, x)));
  }
  return __dmul_rn(p.s2, br);
}

// exp(-a) for a >= 0 (the only sign the kernels need): a = (m ln2)/64 - r with
// m = rint(64 a / ln2), Cody-Waite r (|r| <= ln2/128), exp(-a) = 2^-(m>>6) *
// 2^-((m&63)/64) * exp(r): a 64-entry table of 2^(-j/64) (correctly rounded),
// a degree-5 polynomial (truncation < 4e-17 relative), 2^-(m>>6) built in the
// exponent field. Within 2 ulp of exp(-a) (exact-arithmetic emulation over
// 3e4 samples); a >= 708 (exp < 3.3e-308) returns 0; NaN passes.
namespace {
__device__ const double kExp2NegTab[64] = {
    1.0, 0.9892280131939755, 0.9785720620877001, 0.9680308967461472,
    0.9576032806985737, 0.9472879907934828, 0.93708381705515, 0.9269895625416927,
    0.9170040432046712, 0.9071260877501994, 0.8973545375015536, 0.8876882462632606,
    0.8781260801866497, 0.8686669176368531, 0.859309649061239, 0.8500531768592617,
    0.8408964152537145, 0.8318382901633682, 0.8228777390769825, 0.8140137109286739,
    0.8052451659746271, 0.7965710756711335, 0.7879904225539432, 0.7795022001189185,
    0.7711054127039704, 0.7627990753722692, 0.7545822137967114, 0.7464538641456324,
    0.7384130729697497, 0.7304588970903235, 0.7225904034885233, 0.714806669195985,
    0.7071067811865476, 0.6994898362691556, 0.691954940981916, 0.6845012114872953,
    0.6771277734684463, 0.6698337620266515, 0.6626183215798707, 0.6554806057623822,
    0.6484197773255048, 0.6414350080393891, 0.6345254785958666, 0.6276903785123455,
    0.620928906036742, 0.614240268053435, 0.6076236799902345, 0.6010783657263515,
    0.5946035575013605, 0.5881984958251406, 0.5818624293887887, 0.5755946149764913,
    0.5693943173783458, 0.5632608093041209, 0.5571933712979462, 0.5511912916539204,
    0.5452538663326288, 0.5393803988785599, 0.5335702003384118, 0.5278225891802786,
    0.5221368912137069, 0.5165124395106142, 0.5109485743270583, 0.5054446430258502,
};
}  // namespace
__device__ __forceinline__ double exp_neg(double a) {
  if (!(a < 708.0)) return a == a ? 0.0 : a;
  const double t = a * 92.33248261689366;  // 64 / ln2
  const double mf = rint(t);
  const int m = static_cast<int>(mf);
  double r = fma(mf, 0.01083042469326756, -a);  // (ln2/64)_hi, 32 significant bits
  r = fma(mf, 2.9815858269852933e-12, r);        // (ln2/64)_lo
  double q = fma(r, 8.333333333333333e-03, 4.1666666666666664e-02);
  q = fma(q, r, 1.6666666666666666e-01);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = fma(q, r, 1.0);
  const double tj = __ldg(&kExp2NegTab[m & 63]);
  return (tj * q) * __hiloint2double((1023 - (m >> 6)) << 20, 0);
}

// exp(-a) for finite a >= 0 on the kernel-matrix build path: the same
// reduction and table as exp_neg, branch-free (a clamped to 708: results
// below 3.3e-308 are returned as exp(-708) instead of a smaller value or 0),
// polynomial coefficients in the constant bank.
__constant__ double kExpPoly[8] = {8.333333333333333e-03, 4.1666666666666664e-02, 1.6666666666666666e-01, 0.5,
                                   92.33248261689366, 0.01083042469326756, 2.9815858269852933e-12, 708.0};
__device__ __forceinline__ double exp_neg_fin(double a) {
  a = fmin(a, kExpPoly[7]);
  const double mf = rint(a * kExpPoly[4]);
  const int m = static_cast<int>(mf);
  double r = fma(mf, kExpPoly[5], -a);
  r = fma(mf, kExpPoly[6], r);
  double q = fma(r, kExpPoly[0], kExpPoly[1]);
  q = fma(q, r, kExpPoly[2]);
  q = fma(q, r, kExpPoly[3]);
  q = fma(q, r, 1.0);
  q = fma(q, r, 1.0);
  const double tj = __ldg(&kExp2NegTab[m & 63]);
  return (tj * q) * __hiloint2double((1023 - (m >> 6)) << 20, 0);
}

// Kernel value from the squared distance for the fused-solve build, the
// kernel kind fixed at compile time (KF: 0 RBF, 1/2/3 Matern nu = 0.5/1.5/2.5,
// 4 any other nu through kernel_eval): no per-pair dispatch; the exact-zero
// distance keeps the nugget (kernel.cpp:58-60, :81-83).
__device__ __forceinline__ int kernel_code(const KParams& p) { return p.kind == 1 ? 0 : 1 + p.nu_code; }

template <int KF>
__device__ __forceinline__ double kernel_from_sq(double acc, const KParams& p) {
  double v;
  if constexpr (KF == 0) {
    v = p.s2 * exp_neg_fin(0.5 * acc * (p.inv_rho * p.inv_rho));
  } else if constexpr (KF == 1) {
    v = p.s2 * exp_neg_fin(sqrt(acc) * p.inv_rho);
  } else if constexpr (KF == 2) {
    const double a = 1.7320508075688772 * sqrt(acc) * p.inv_rho;
    v = p.s2 * ((1.0 + a) * exp_neg_fin(a));
  } else if constexpr (KF == 3) {
    const double a = 2.2360679774997898 * sqrt(acc) * p.inv_rho;
    v = p.s2 * (fma(a, a * (1.0 / 3.0), 1.0 + a) * exp_neg_fin(a));
  } else {
    v = kernel_eval(sqrt(acc), p);  // general nu (its d == 0 branch is the same nugget rule)
  }
  return acc == 0.0 ? p.diag : v;
}

// Build-path arithmetic for the register solve (solve_reg.cu), branch-free:
// the kernel-matrix entries only have to be accurate to a few ulps (the
// coefficient tolerance is 1e-9 relative), so the special-case paths of the
// libdevice sqrt/rsqrt are replaced by a MUFU seed plus Newton/Goldschmidt
// refinement, and exp(-a) rounds with the 1.5*2^52 shift instead of
// FRND/F2I and folds 2^-(m>>6) into the table value's exponent field.
//
// sqrt(x) for finite x >= 0: MUFU rsqrt seed (~2^-22) and one third-order
// correction (< 1 ulp + rounding). x == 0 gives NaN (0 * inf); every caller
// replaces the d == 0 entry by the nugget.
#ifndef FMGP_SQRT_BUILD3
#define FMGP_SQRT_BUILD3 1
#endif
__device__ __forceinline__ double sqrt_build(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#if FMGP_SQRT_BUILD3
  // one third-order step: r = x y, e = 1 - r y (exact residual of the rounded r),
  // sqrt(x) = r / sqrt(1 - e) = r (1 + e/2 + 3 e^2/8 + O(e^3)), e ~ 2^-22: five FP64
  // operations, four of them dependent, instead of seven (A/B: FMGP_SQRT_BUILD3=0)
  const double r = x * y;
  const double e = fma(-r, y, 1.0);
  return fma(r * e, fma(e, 0.375, 0.5), r);
#else
  double r = x * y, h = 0.5 * y;
  const double e = fma(-r, h, 0.5);
  r = fma(r, e, r);
  h = fma(h, e, h);
  const double dd = fma(-r, r, x);
  return fma(dd, h, r);
#endif
}

// 1/sqrt(x) for a Cholesky pivot x > 0: MUFU seed and two Newton steps
// (quadratic: 2^-22 -> 2^-43 -> rounding). x <= 0 returns garbage; the
// caller has already recorded the failed pivot.
__device__ __forceinline__ double rsqrt_pivot(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  double t = fma(-h * y, y, 0.5);
  y = fma(y, t, y);
  t = fma(-h * y, y, 0.5);
  return fma(y, t, y);
}

// exp(-a) for a >= 0 (NaN-free) on the build paths (kernel-matrix and
// cross-covariance entries): m = rint(64 a / ln2) by the 1.5*2^52 shift (m is
// the low word of the shifted value), Cody-Waite r = m ln2/64 - a
// (|r| <= ln2/128), exp(-a) = 2^-(m>>6) * 2^-((m&63)/64) * e^r with a degree-5
// polynomial and the 64-entry table of 2^(-j/64) (read from a shared-memory
// copy, `tab`); 2^-(m>>6) is an exponent-field subtraction on the table value
// (a <= 708 keeps the result normal). Within 2 ulp of exp(-a). A/B variant
// (FMGP_EXP_TAB32): a 32-entry table (fewer bank conflicts) and a degree-6
// polynomial; measured slower at cfg5 in the spatially ordered solve
// (profiles/r02/ab_exp_table.txt), so not the default.
__device__ const double kExp2NegTab32[32] = {
    1.0, 0.9785720620877001, 0.9576032806985737, 0.93708381705515,
    0.9170040432046712, 0.8973545375015536, 0.8781260801866497, 0.859309649061239,
    0.8408964152537145, 0.8228777390769825, 0.8052451659746271, 0.7879904225539432,
    0.7711054127039704, 0.7545822137967114, 0.7384130729697497, 0.7225904034885233,
    0.7071067811865476, 0.691954940981916, 0.6771277734684463, 0.6626183215798707,
    0.6484197773255048, 0.6345254785958666, 0.620928906036742, 0.6076236799902345,
    0.5946035575013605, 0.5818624293887887, 0.5693943173783458, 0.5571933712979462,
    0.5452538663326288, 0.5335702003384118, 0.5221368912137069, 0.5109485743270583,
};
#ifndef FMGP_EXP_TAB32
__device__ __forceinline__ double exp_neg_build(double a, const double* tab = kExp2NegTab) {
  // a >= 0: clamp at 708 (0x40862000'00000000) by the high word, an integer
  // compare + two selects (a double compare compiles to fmin with NaN fix-ups);
  // NaN (an overflowed distance) also maps to the clamp
  a = __double2hiint(a) < 0x40862000 ? a : 708.0;
  const double tm = fma(a, 92.33248261689366, 6755399441055744.0);
  const int m = __double2loint(tm);
  const double mf = tm - 6755399441055744.0;
  double r = fma(mf, 0.01083042469326756, -a);
  r = fma(mf, 2.9815858269852933e-12, r);
  double q = fma(r, 8.333333333333333e-03, 4.1666666666666664e-02);
  q = fma(q, r, 1.6666666666666666e-01);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = fma(q, r, 1.0);
  const double tj = tab[m & 63];
  const double sj = __hiloint2double(__double2hiint(tj) - ((m >> 6) << 20), __double2loint(tj));
  return sj * q;
}
#define FMGP_BUILD_TAB kExp2NegTab
#define FMGP_BUILD_TAB_N 64
#else
#define FMGP_BUILD_TAB kExp2NegTab32
#define FMGP_BUILD_TAB_N 32
__device__ __forceinline__ double exp_neg_build(double a, const double* tab = kExp2NegTab32) {
  a = __double2hiint(a) < 0x40862000 ? a : 708.0;
  const double tm = fma(a, 46.16624130844683, 6755399441055744.0);
  const int m = __double2loint(tm);
  const double mf = tm - 6755399441055744.0;
  double r = fma(mf, 0.02166084938653512, -a);  // (ln2/32)_hi, 33 significant bits: mf * hi exact
  r = fma(mf, 5.9631716539705866e-12, r);        // (ln2/32)_lo
  double q = fma(r, 1.388888888888889e-03, 8.333333333333333e-03);
  q = fma(q, r, 4.1666666666666664e-02);
  q = fma(q, r, 1.6666666666666666e-01);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  q = fma(q, r, 1.0);
  const double tj = tab[m & 31];
  const double sj = __hiloint2double(__double2hiint(tj) - ((m >> 5) << 20), __double2loint(tj));
  return sj * q;
}
#endif

// Kernel value from the squared distance on the register-solve build path
// (KF as in kernel_from_sq; `c` = the kind's distance scale: sqrt(3)/rho,
// sqrt(5)/rho, 1/rho, or 0.5/rho^2 for RBF). d == 0 keeps the nugget.
// General nu (GSL lnKnu path, no BASELINE config): out of line, so its
// register demand does not set the register budget of the solve kernels.
static __device__ __noinline__ double kernel_eval_general(double dist, const KParams& p);

// Copy of the build exp table into shared memory (32 doubles; call with
// every thread of the CTA, then __syncthreads).
__device__ __forceinline__ void stage_exp_table(double* dst) {
  for (int i = threadIdx.x; i < FMGP_BUILD_TAB_N; i += blockDim.x) dst[i] = FMGP_BUILD_TAB[i];
}


// `tab`: the 2^(-j/64) table of exp_neg_build; the fused solves pass a copy
// in shared memory (the global table's divergent lookups were ~90% of the
// solve's L1 sector traffic, profiles/r02/ncu_solve_cfg5_full.txt).
template <int KF>
__device__ __forceinline__ double kernel_from_sq_build(double acc, double c, const KParams& p,
                                                       const double* tab = FMGP_BUILD_TAB) {
  double v;
  if constexpr (KF == 0) {
    v = p.s2 * exp_neg_build(acc * c, tab);
  } else if constexpr (KF == 1) {
    v = p.s2 * exp_neg_build(sqrt_build(acc) * c, tab);
  } else if constexpr (KF == 2) {
    const double a = sqrt_build(acc) * c;
    const double e = exp_neg_build(a, tab);
    v = p.s2 * fma(a, e, e);
  } else if constexpr (KF == 3) {
    const double a = sqrt_build(acc) * c;
    v = p.s2 * (fma(a, a * (1.0 / 3.0), 1.0 + a) * exp_neg_build(a, tab));
  } else {
    v = kernel_eval_general(sqrt(acc), p);
  }
  return acc == 0.0 ? p.diag : v;
}

static __device__ __noinline__ double kernel_eval_general(double dist, const KParams& p) { return kernel_eval(dist, p); }

template <int KF>
__device__ __forceinline__ double kernel_scale_build(const KParams& p) {
  if constexpr (KF == 0) return 0.5 * (p.inv_rho * p.inv_rho);
  if constexpr (KF == 1) return p.inv_rho;
  if constexpr (KF == 2) return 1.7320508075688772 * p.inv_rho;
  if constexpr (KF == 3) return 2.2360679774997898 * p.inv_rho;
  return 0.0;
}

// kernel_value for the neighbourhood matrices of the fused solve: the same
// formulas with 1/rho multiplied instead of divided and contraction allowed.
// The matrix entries differ from kernel_eval by at most a few ulps, far inside
// the coefficient tolerance; predictions use the exact-order kernel_eval.
__device__ __forceinline__ double kernel_eval_fast(double dist, const KParams& p) {
  if (dist == 0.0) return p.diag;
  double br;
  if (p.kind == 1) {
    const double u = dist * p.inv_rho;
    br = exp_neg(0.5 * u * u);
  } else if (p.nu_code == 0) {
    br = exp_neg(dist * p.inv_rho);
  } else if (p.nu_code == 1) {
    const double a = 1.7320508075688772 * dist * p.inv_rho;
    br = (1.0 + a) * exp_neg(a);
  } else if (p.nu_code == 2) {
    const double a = 2.2360679774997898 * dist * p.inv_rho;
    br = fma(a, a * (1.0 / 3.0), 1.0 + a) * exp_neg(a);
  } else {
    return kernel_eval(dist, p);
  }
  return p.s2 * br;
}

// (dist, idx) lexicographic order of std::pair<double,int> (nn_index.cpp:275-281, :363).
__device__ __forceinline__ bool pair_less(double da, int32_t ia, double db, int32_t ib) {
  return da < db || (da == db && ia < ib);
}

}  // namespace fmgp
