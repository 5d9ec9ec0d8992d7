// MuyGPs training inner loop and the localized baseline predictor on the
// device, built from the precompute path's kernels:
//  * local_prediction / loocv_loss (muygps.cpp:32-78): the batch's neighbour
//    lists play the role of S, so one fused_solve (gather -> K -> jitter
//    Cholesky -> solve, K2) yields every entry's coefficients, and
//    cross_dot_kernel takes cross . coeff with cross = kernel(list distance);
//  * train (muygps.cpp:214-270): neighbour lists once on the device (K1 with
//    per-query self exclusion), then the reference's bounded Nelder-Mead on
//    the host, each loss evaluation a device LOOCV pass that moves only the
//    kernel parameters in and b predictions out;
//  * muygps_predict (muygps.cpp:272-295): K1 kNN of each test point, K2 on
//    those neighbourhoods, cross dot, + mean offset.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "capi_common.h"
#include "fmgp_internal.h"

using namespace fmgp_capi;

namespace fmgp {
namespace {

constexpr int kDotWarps = 8;

// out[r] = add + sum_t kernel(dist_rt) * C[r, t] (warp per row; the sum runs
// in t order through a shuffle chain). dist_is_sq: dist holds squared
// distances (sqrt taken here, as NeighborList.distances = sqrt(dist_sq)).
__global__ void __launch_bounds__(kDotWarps * kWarp)
cross_dot_kernel(const double* __restrict__ dist, int dist_is_sq, const double* __restrict__ C, int64_t rows, int k,
                 KParams kp, double add, double* __restrict__ out) {
  const int lane = threadIdx.x % kWarp;
  const int64_t w0 = static_cast<int64_t>(blockIdx.x) * kDotWarps + threadIdx.x / kWarp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kDotWarps;
  for (int64_t r = w0; r < rows; r += nw) {
    double acc = 0.0;
    for (int t0 = 0; t0 < k; t0 += kWarp) {
      const int t = t0 + lane;
      double prod = 0.0;
      if (t < k) {
        const double dv = dist[r * k + t];
        prod = __dmul_rn(kernel_eval(dist_is_sq ? sqrt(dv) : dv, kp), C[r * k + t]);
      }
      const int cnt = min(kWarp, k - t0);
      for (int s = 0; s < cnt; ++s) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, prod, s));
    }
    if (lane == 0) out[r] = __dadd_rn(acc, add);
  }
}

__global__ void gather_rows_d(const double* __restrict__ X, int d, const int32_t* __restrict__ idx, int64_t cnt,
                              double* __restrict__ out) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < cnt * d;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / d;
    out[e] = X[static_cast<int64_t>(idx[r]) * d + (e - r * d)];
  }
}

unsigned grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16)));
}

}  // namespace

cudaError_t cross_dot(const double* dist, int dist_is_sq, const double* C, int64_t rows, int k, const KParams& kp,
                      double add, double* out, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  cross_dot_kernel<<<grid_for(rows, kDotWarps), kDotWarps * kWarp, 0, s>>>(dist, dist_is_sq, C, rows, k, kp, add,
                                                                           out);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t gather_rows(const double* X, int d, const int32_t* idx, int64_t cnt, double* out, cudaStream_t s) {
  if (cnt <= 0) return cudaSuccess;
  gather_rows_d<<<grid_for(cnt * d, 256), 256, 0, s>>>(X, d, idx, cnt, out);
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace fmgp

// --------------------------------------------------------------- LOOCV session

struct fmgp_loocv {
  int64_t n = 0, b = 0;
  int32_t d = 0, k = 0;
  cudaStream_t s = nullptr;
  double *X = nullptr, *Y = nullptr, *dist = nullptr, *C = nullptr, *preds = nullptr;
  int32_t* nbr = nullptr;
  unsigned long long* fmin = nullptr;
  std::vector<int32_t> batch;   // host copy (error messages, residuals)
  std::vector<double> ybatch;   // Y[batch[t]]
  int64_t first_bad = -1;       // first entry failing validation (reported after the entries before it)
  int bad_code = FMGP_OK;
  std::string bad_msg;
  ~fmgp_loocv() {
    for (void* p : {static_cast<void*>(X), static_cast<void*>(Y), static_cast<void*>(dist), static_cast<void*>(C),
                    static_cast<void*>(preds), static_cast<void*>(nbr), static_cast<void*>(fmin)})
      if (p) cudaFree(p);
    if (s) cudaStreamDestroy(s);
  }
};

namespace {

// local_prediction's own checks (muygps.cpp:35-48) for every entry; the
// first failing entry is remembered so that the entries before it are still
// evaluated first, as the reference's sequential loop would.
void validate_entries(fmgp_loocv* h, const int32_t* batch_idx, const int32_t* nbr, const double* dist) {
  for (int64_t t = 0; t < h->b && h->first_bad < 0; ++t) {
    const int32_t i = batch_idx[t];
    std::string msg;
    if (h->k < 1) {
      msg = "local_prediction: empty neighbor list";
    } else if (i < 0 || i >= h->n) {
      msg = "local_prediction: index out of range";
    } else {
      for (int32_t j = 0; j < h->k && msg.empty(); ++j)
        if (nbr[t * h->k + j] == i)
          msg = "local_prediction: point " + std::to_string(i) + " appears in its own neighbor list";
      for (int32_t j = 0; j < h->k && msg.empty(); ++j) {
        const int32_t v = nbr[t * h->k + j];
        if (v < 0 || v >= h->n) msg = "local_prediction: neighbor index out of range";
        else if (dist != nullptr && !(std::isfinite(dist[t * h->k + j]) && dist[t * h->k + j] >= 0.0))
          msg = "kernel distance must be finite and non-negative";  // check_distance, kernel.cpp:32-36
      }
    }
    if (!msg.empty()) {
      h->first_bad = t;
      h->bad_code = FMGP_EINVAL;
      h->bad_msg = msg;
    }
  }
}

int loocv_alloc(fmgp_loocv* h) {
  FMGP_CUDA(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
  FMGP_CUDA(cudaMalloc(&h->X, sizeof(double) * h->n * h->d));
  FMGP_CUDA(cudaMalloc(&h->Y, sizeof(double) * h->n));
  FMGP_CUDA(cudaMalloc(&h->dist, sizeof(double) * std::max<int64_t>(1, h->b * h->k)));
  FMGP_CUDA(cudaMalloc(&h->C, sizeof(double) * std::max<int64_t>(1, h->b * h->k)));
  FMGP_CUDA(cudaMalloc(&h->preds, sizeof(double) * std::max<int64_t>(1, h->b)));
  FMGP_CUDA(cudaMalloc(&h->nbr, sizeof(int32_t) * std::max<int64_t>(1, h->b * h->k)));
  FMGP_CUDA(cudaMalloc(&h->fmin, sizeof(unsigned long long)));
  return FMGP_OK;
}

// Predictions of entries [0, rows) into preds_host; numeric failure names the
// lowest failing entry.
int loocv_run(fmgp_loocv* h, const fmgp::KParams& kp, int64_t rows, double* preds_host, int64_t* failed_entry) {
  if (failed_entry) *failed_entry = -1;
  if (rows <= 0) return FMGP_OK;
  const int sms = num_sms_current();
  FMGP_CUDA(cudaMemsetAsync(h->fmin, 0xFF, sizeof(unsigned long long), h->s));
  FMGP_CUDA(fmgp::fused_solve(h->X, h->Y, h->d, 1, h->nbr, rows, 0, h->k, kp, h->C, nullptr, h->fmin, sms, h->s));
  FMGP_CUDA(fmgp::cross_dot(h->dist, 0, h->C, rows, h->k, kp, 0.0, h->preds, h->s));
  unsigned long long fm = ~0ull;
  FMGP_CUDA(cudaMemcpyAsync(&fm, h->fmin, sizeof(fm), cudaMemcpyDeviceToHost, h->s));
  FMGP_CUDA(cudaMemcpyAsync(preds_host, h->preds, sizeof(double) * rows, cudaMemcpyDeviceToHost, h->s));
  FMGP_CUDA(cudaStreamSynchronize(h->s));
  if (fm != ~0ull) {
    if (failed_entry) *failed_entry = static_cast<int64_t>(fm);
    return fail(FMGP_ENUMERIC, "Cholesky factorization failed in local_prediction at index " +
                                   std::to_string(h->batch[fm]) + " after jitter escalation up to 1e-6");
  }
  return FMGP_OK;
}

int loocv_setup(const double* X, const double* Y, int64_t n, int32_t d, const int32_t* batch_idx, const int32_t* nbr,
                const double* dist, int64_t b, int32_t k, bool dist_on_device, fmgp_loocv* h) {
  h->n = n;
  h->d = d;
  h->b = b;
  h->k = k;
  h->batch.assign(batch_idx, batch_idx + b);
  validate_entries(h, batch_idx, nbr, dist_on_device ? nullptr : dist);
  h->ybatch.resize(b);
  for (int64_t t = 0; t < b; ++t) {
    const int32_t i = batch_idx[t];
    h->ybatch[t] = (i >= 0 && i < n) ? Y[i] : 0.0;
  }
  int rc;
  if ((rc = loocv_alloc(h)) != FMGP_OK) return rc;
  FMGP_CUDA(cudaMemcpyAsync(h->X, X, sizeof(double) * n * d, cudaMemcpyHostToDevice, h->s));
  FMGP_CUDA(cudaMemcpyAsync(h->Y, Y, sizeof(double) * n, cudaMemcpyHostToDevice, h->s));
  if (nbr != nullptr && b * k > 0)
    FMGP_CUDA(cudaMemcpyAsync(h->nbr, nbr, sizeof(int32_t) * b * k, cudaMemcpyHostToDevice, h->s));
  if (!dist_on_device && b * k > 0)
    FMGP_CUDA(cudaMemcpyAsync(h->dist, dist, sizeof(double) * b * k, cudaMemcpyHostToDevice, h->s));
  FMGP_CUDA(cudaStreamSynchronize(h->s));
  return FMGP_OK;
}

int loocv_loss_impl(fmgp_loocv* h, const fmgp::KParams& kp, double* loss_out, double* preds_out,
                    int64_t* failed_entry) {
  const int64_t rows = h->first_bad >= 0 ? h->first_bad : h->b;
  std::vector<double> preds(static_cast<size_t>(std::max<int64_t>(1, h->b)), 0.0);
  int rc = loocv_run(h, kp, rows, preds.data(), failed_entry);
  if (rc != FMGP_OK) return rc;
  if (h->first_bad >= 0) return fail(h->bad_code, h->bad_msg);
  double sum = 0.0;  // muygps.cpp:70-77: sequential over the batch
  for (int64_t t = 0; t < h->b; ++t) {
    const double r = h->ybatch[t] - preds[t];
    sum += r * r;
  }
  if (loss_out) *loss_out = sum / static_cast<double>(h->b);
  if (preds_out) std::copy(preds.begin(), preds.begin() + h->b, preds_out);
  return FMGP_OK;
}

int check_common(const double* X, const double* Y, int64_t n, int32_t d) {
  int rc;
  if ((rc = check_points(X, n, d)) != FMGP_OK) return rc;
  if (Y == nullptr) return fail(FMGP_EINVAL, "training responses must not be null");
  return require_device();
}

// ---- bounded Nelder-Mead (muygps.cpp:82-210), restated --------------------

enum class Coord { Rho, Nu, Tau };
struct Free {
  Coord which;
  double lo, hi;  // transformed (rho in log10)
  double to_param(double x) const { return which == Coord::Rho ? std::pow(10.0, x) : x; }
  double from_param(double v) const { return which == Coord::Rho ? std::log10(v) : v; }
};

fmgp_kernel_params with_coords(const fmgp_kernel_params& base, const std::vector<Free>& fr,
                               const std::vector<double>& x) {
  fmgp_kernel_params p = base;
  for (size_t j = 0; j < fr.size(); ++j) {
    const double v = fr[j].to_param(x[j]);
    if (fr[j].which == Coord::Rho) p.rho = v;
    else if (fr[j].which == Coord::Nu) p.nu = v;
    else p.tau = v;
  }
  return p;
}

struct Simplex {
  std::vector<double> best_x;
  double best_f;
  int evals;
};

// Objective returns FMGP_OK and the value, or an error code that aborts the search.
template <typename F>
int nelder_mead(F&& f, std::vector<double> x0, const std::vector<Free>& fr, int max_evals, double tol, Simplex* out) {
  const size_t dim = x0.size();
  auto clamp = [&](std::vector<double>& x) {
    for (size_t j = 0; j < dim; ++j) x[j] = std::clamp(x[j], fr[j].lo, fr[j].hi);
  };
  clamp(x0);
  int evals = 0;
  std::vector<double> best_x = x0;
  double best_f = std::numeric_limits<double>::infinity();
  int rc = FMGP_OK;
  auto eval = [&](const std::vector<double>& x) -> double {
    double v = 0.0;
    if (rc == FMGP_OK) rc = f(x, &v);
    ++evals;
    if (v < best_f) {
      best_f = v;
      best_x = x;
    }
    return v;
  };
  std::vector<std::vector<double>> pts(dim + 1, x0);
  for (size_t j = 0; j < dim; ++j) {
    const double step = 0.25 * (fr[j].hi - fr[j].lo);
    pts[j + 1][j] += (x0[j] + step <= fr[j].hi) ? step : -step;
  }
  std::vector<double> fv(dim + 1, 0.0);
  for (size_t v = 0; v <= dim && evals < max_evals; ++v) {
    fv[v] = eval(pts[v]);
    if (rc != FMGP_OK) return rc;
  }
  while (evals < max_evals) {
    std::vector<size_t> order(dim + 1);
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return fv[a] < fv[b]; });
    if (fv[order[dim]] - fv[order[0]] < tol) break;
    const size_t worst = order[dim];
    std::vector<double> cen(dim, 0.0);
    for (size_t v = 0; v <= dim; ++v) {
      if (v == worst) continue;
      for (size_t j = 0; j < dim; ++j) cen[j] += pts[v][j];
    }
    for (double& c : cen) c /= static_cast<double>(dim);
    auto blend = [&](double coef) {
      std::vector<double> x(dim);
      for (size_t j = 0; j < dim; ++j) x[j] = cen[j] + coef * (cen[j] - pts[worst][j]);
      clamp(x);
      return x;
    };
    const std::vector<double> xr = blend(1.0);
    const double fr_ = eval(xr);
    if (rc != FMGP_OK) return rc;
    if (fr_ < fv[order[0]] && evals < max_evals) {
      const std::vector<double> xe = blend(2.0);
      const double fe = eval(xe);
      if (rc != FMGP_OK) return rc;
      if (fe < fr_) {
        pts[worst] = xe;
        fv[worst] = fe;
      } else {
        pts[worst] = xr;
        fv[worst] = fr_;
      }
    } else if (fr_ < fv[order[dim - 1]]) {
      pts[worst] = xr;
      fv[worst] = fr_;
    } else if (evals < max_evals) {
      const std::vector<double> xc = blend(-0.5);
      const double fc = eval(xc);
      if (rc != FMGP_OK) return rc;
      if (fc < fv[worst]) {
        pts[worst] = xc;
        fv[worst] = fc;
      } else {  // shrink toward the best vertex
        for (size_t v = 0; v <= dim; ++v) {
          if (v == order[0]) continue;
          for (size_t j = 0; j < dim; ++j) pts[v][j] = 0.5 * (pts[v][j] + pts[order[0]][j]);
          if (evals >= max_evals) break;
          fv[v] = eval(pts[v]);
          if (rc != FMGP_OK) return rc;
        }
      }
    }
  }
  out->best_x = best_x;
  out->best_f = best_f;
  out->evals = evals;
  return FMGP_OK;
}

}  // namespace

extern "C" {

int fmgp_local_predictions(const double* X, const double* Y, int64_t n, int32_t d, const int32_t* batch_idx,
                           const int32_t* nbr, const double* dist, int64_t b, int32_t k,
                           const fmgp_kernel_params* params, double* preds_out, int64_t* failed_entry) {
  if (failed_entry) *failed_entry = -1;
  fmgp::KParams kp;
  int rc;
  if ((rc = make_kparams(params, &kp)) != FMGP_OK) return rc;
  if ((rc = check_common(X, Y, n, d)) != FMGP_OK) return rc;
  if (b < 0) return fail(FMGP_EINVAL, "local_predictions: negative batch size");
  if (b == 0) return FMGP_OK;
  fmgp_loocv h;
  if ((rc = loocv_setup(X, Y, n, d, batch_idx, nbr, dist, b, k, false, &h)) != FMGP_OK) return rc;
  const int64_t rows = h.first_bad >= 0 ? h.first_bad : b;
  if ((rc = loocv_run(&h, kp, rows, preds_out, failed_entry)) != FMGP_OK) return rc;
  if (h.first_bad >= 0) return fail(h.bad_code, h.bad_msg);
  return FMGP_OK;
}

int fmgp_loocv_create(const double* X, const double* Y, int64_t n, int32_t d, const int32_t* batch_idx,
                      const int32_t* nbr, const double* dist, int64_t b, int32_t k, fmgp_loocv** out) {
  if (out == nullptr) return fail(FMGP_EINVAL, "loocv session output must not be null");
  *out = nullptr;
  int rc;
  if ((rc = check_common(X, Y, n, d)) != FMGP_OK) return rc;
  if (b < 1) return fail(FMGP_EINVAL, "loocv_loss: batch and neighbor lists disagree");
  auto* h = new fmgp_loocv();
  if ((rc = loocv_setup(X, Y, n, d, batch_idx, nbr, dist, b, k, false, h)) != FMGP_OK) {
    delete h;
    return rc;
  }
  *out = h;
  return FMGP_OK;
}

int fmgp_loocv_eval(fmgp_loocv* h, const fmgp_kernel_params* params, double* loss_out, double* preds_out,
                    int64_t* failed_entry) {
  if (failed_entry) *failed_entry = -1;
  if (h == nullptr) return fail(FMGP_EINVAL, "null loocv session");
  fmgp::KParams kp;
  int rc;
  if ((rc = make_kparams(params, &kp)) != FMGP_OK) return rc;
  return loocv_loss_impl(h, kp, loss_out, preds_out, failed_entry);
}

void fmgp_loocv_destroy(fmgp_loocv* h) { delete h; }

int fmgp_train(const double* X, const double* Y, int64_t n, int32_t d, const int32_t* batch_idx, int64_t b,
               const fmgp_kernel_params* initial, const fmgp_train_config* cfg, fmgp_kernel_params* theta_out,
               double* final_loss, int32_t* evaluations, int32_t* improved) {
  if (initial == nullptr || cfg == nullptr) return fail(FMGP_EINVAL, "train: null argument");
  fmgp::KParams kp0;
  int rc;
  if ((rc = make_kparams(initial, &kp0)) != FMGP_OK) return rc;
  if (cfg->k < 2) return fail(FMGP_EINVAL, "train: k must be at least 2");
  if ((rc = check_common(X, Y, n, d)) != FMGP_OK) return rc;
  if (b < 1) return fail(FMGP_EINVAL, "loocv_loss: batch and neighbor lists disagree");
  for (int64_t t = 0; t < b; ++t)
    if (batch_idx[t] < 0 || batch_idx[t] >= n) return fail(FMGP_EINVAL, "train: batch index out of range");
  if (cfg->k > n - 1) return fail(FMGP_EINVAL, "query_knn: k out of range");
  // Neighbour lists (muygps.cpp:225-230): k exact neighbours of x_i, self excluded.
  auto* h = new fmgp_loocv();
  struct Guard {
    fmgp_loocv* h;
    ~Guard() { delete h; }
  } guard{h};
  h->n = n;
  h->d = d;
  h->b = b;
  h->k = cfg->k;
  h->batch.assign(batch_idx, batch_idx + b);
  h->ybatch.resize(b);
  for (int64_t t = 0; t < b; ++t) h->ybatch[t] = Y[batch_idx[t]];
  if ((rc = loocv_alloc(h)) != FMGP_OK) return rc;
  FMGP_CUDA(cudaMemcpyAsync(h->X, X, sizeof(double) * n * d, cudaMemcpyHostToDevice, h->s));
  FMGP_CUDA(cudaMemcpyAsync(h->Y, Y, sizeof(double) * n, cudaMemcpyHostToDevice, h->s));
  {
    DevBuf<int32_t> dB;
    DevBuf<double> dQ;
    FMGP_CUDA(dB.alloc(static_cast<size_t>(b), h->s));
    FMGP_CUDA(dQ.alloc(static_cast<size_t>(b) * d, h->s));
    FMGP_CUDA(cudaMemcpyAsync(dB.p, batch_idx, sizeof(int32_t) * b, cudaMemcpyHostToDevice, h->s));
    FMGP_CUDA(fmgp::gather_rows(h->X, d, dB.p, b, dQ.p, h->s));
    FMGP_CUDA(fmgp::knn_exact(dQ.p, b, h->X, n, d, cfg->k, -1, dB.p, 0, h->nbr, h->dist, num_sms_current(), h->s));
    FMGP_CUDA(fmgp::sqrt_inplace_launch(h->dist, b * cfg->k, h->s));
    FMGP_CUDA(cudaStreamSynchronize(h->s));
  }
  // Free coordinates (muygps.cpp:232-245), checked in rho, nu, tau order.
  std::vector<Free> fr;
  auto add = [&](Coord which, int32_t has, double lo, double hi, bool log_space) -> int {
    if (!has) return FMGP_OK;
    if (!(lo < hi) || !std::isfinite(lo) || !std::isfinite(hi)) return fail(FMGP_EINVAL, "train: invalid bounds");
    fr.push_back({which, log_space ? std::log10(lo) : lo, log_space ? std::log10(hi) : hi});
    return FMGP_OK;
  };
  if ((rc = add(Coord::Rho, cfg->has_rho, cfg->rho_lo, cfg->rho_hi, true)) != FMGP_OK) return rc;
  if ((rc = add(Coord::Nu, cfg->has_nu, cfg->nu_lo, cfg->nu_hi, false)) != FMGP_OK) return rc;
  if ((rc = add(Coord::Tau, cfg->has_tau, cfg->tau_lo, cfg->tau_hi, false)) != FMGP_OK) return rc;

  fmgp_kernel_params base = *initial;
  base.kind = cfg->kind;
  fmgp::KParams kpb;
  if ((rc = make_kparams(&base, &kpb)) != FMGP_OK) return rc;
  double q0 = 0.0;
  if ((rc = loocv_loss_impl(h, kpb, &q0, nullptr, nullptr)) != FMGP_OK) return rc;
  auto finish = [&](const fmgp_kernel_params& th, double loss, int ev, bool imp) {
    if (theta_out) *theta_out = th;
    if (final_loss) *final_loss = loss;
    if (evaluations) *evaluations = ev;
    if (improved) *improved = imp ? 1 : 0;
    return FMGP_OK;
  };
  if (fr.empty()) return finish(base, q0, 1, false);
  std::vector<double> x0;
  for (const Free& c : fr) {
    const double v = c.which == Coord::Rho ? base.rho : (c.which == Coord::Nu ? base.nu : base.tau);
    x0.push_back(std::clamp(c.from_param(v), c.lo, c.hi));
  }
  auto objective = [&](const std::vector<double>& x, double* val) -> int {
    const fmgp_kernel_params p = with_coords(base, fr, x);
    fmgp::KParams kp;
    int r = make_kparams(&p, &kp);
    if (r != FMGP_OK) return r;
    return loocv_loss_impl(h, kp, val, nullptr, nullptr);
  };
  Simplex res;
  if ((rc = nelder_mead(objective, x0, fr, cfg->max_evals, cfg->tol, &res)) != FMGP_OK) return rc;
  if (res.best_f >= q0) return finish(base, q0, res.evals, false);
  return finish(with_coords(base, fr, res.best_x), res.best_f, res.evals, true);
}

int fmgp_muygps_predict(const double* X, const double* Y, int64_t n, int32_t d, const double* Z, int64_t nz,
                        int32_t k, const fmgp_kernel_params* params, double mean_offset, double* out,
                        int64_t* failed_row) {
  if (failed_row) *failed_row = -1;
  fmgp::KParams kp;
  int rc;
  if ((rc = make_kparams(params, &kp)) != FMGP_OK) return rc;
  if ((rc = check_common(X, Y, n, d)) != FMGP_OK) return rc;
  if (nz <= 0) return FMGP_OK;
  for (int64_t e = 0; e < nz * d; ++e)
    if (!std::isfinite(Z[e])) return fail(FMGP_EINVAL, "query_knn: non-finite query");
  if (k < 1 || k > n) return fail(FMGP_EINVAL, "query_knn: k out of range");
  Stream st;
  FMGP_CUDA(st.create());
  DevBuf<double> dX, dY, dZ, dD, dC, dO;
  DevBuf<int32_t> dS;
  DevBuf<unsigned long long> fmin;
  FMGP_CUDA(dX.alloc(static_cast<size_t>(n) * d, st.s));
  FMGP_CUDA(dY.alloc(static_cast<size_t>(n), st.s));
  FMGP_CUDA(dZ.alloc(static_cast<size_t>(nz) * d, st.s));
  FMGP_CUDA(dD.alloc(static_cast<size_t>(nz) * k, st.s));
  FMGP_CUDA(dC.alloc(static_cast<size_t>(nz) * k, st.s));
  FMGP_CUDA(dO.alloc(static_cast<size_t>(nz), st.s));
  FMGP_CUDA(dS.alloc(static_cast<size_t>(nz) * k, st.s));
  FMGP_CUDA(fmin.alloc(1, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dX.p, X, sizeof(double) * n * d, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dY.p, Y, sizeof(double) * n, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dZ.p, Z, sizeof(double) * nz * d, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(cudaMemsetAsync(fmin.p, 0xFF, sizeof(unsigned long long), st.s));
  const int sms = num_sms_current();
  FMGP_CUDA(fmgp::knn_exact(dZ.p, nz, dX.p, n, d, k, -1, nullptr, 0, dS.p, dD.p, sms, st.s));
  FMGP_CUDA(fmgp::fused_solve(dX.p, dY.p, d, 1, dS.p, nz, 0, k, kp, dC.p, nullptr, fmin.p, sms, st.s));
  FMGP_CUDA(fmgp::cross_dot(dD.p, 1, dC.p, nz, k, kp, mean_offset, dO.p, st.s));
  unsigned long long fm = ~0ull;
  FMGP_CUDA(cudaMemcpyAsync(&fm, fmin.p, sizeof(fm), cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaMemcpyAsync(out, dO.p, sizeof(double) * nz, cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaStreamSynchronize(st.s));
  if (fm != ~0ull) {
    if (failed_row) *failed_row = static_cast<int64_t>(fm);
    return fail(FMGP_ENUMERIC, "Cholesky factorization failed in muygps_predict after jitter escalation up to 1e-6");
  }
  return FMGP_OK;
}

}  // extern "C"
