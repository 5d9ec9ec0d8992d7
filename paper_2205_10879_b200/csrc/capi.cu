#include <chrono>
// The C ABI (include/fmgp_b200.h): argument checks with the reference's
// error conventions, device memory and streams, and the stage launchers.
// There is no CPU compute path: without a usable CUDA device every compute
// entry point returns FMGP_ECUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fmgp_b200.h"
#include "fmgp_common.cuh"
#include "fmgp_internal.h"

#include "capi_common.h"
#include "capi_model.h"

using namespace fmgp_capi;

namespace {

// Opt-in stage timing (fmgp_set_stage_timing): CUDA events recorded on the
// launching stream around the kNN and fused-solve launches of each
// precompute call, resolved after the caller's timed region.
std::atomic<int> g_stage_timing{0};
std::mutex g_stage_mu;
struct StageEvents {
  cudaEvent_t e[3];
};
std::vector<StageEvents> g_stage_events;

int precompute_device_impl(const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                           const fmgp::KParams& kp, int32_t k, int64_t row_begin, int64_t row_end, int32_t* S_out,
                           double* C_out, int64_t* failed_row, cudaStream_t stream) {
  const int64_t nrows = row_end - row_begin;
  if (failed_row) *failed_row = -1;
  if (nrows <= 0) return FMGP_OK;
  const int sms = num_sms_current();
  StageEvents ev{};
  const bool timing = g_stage_timing.load(std::memory_order_relaxed) != 0;
  if (timing) {
    for (auto& e : ev.e) FMGP_CUDA(cudaEventCreate(&e));
    FMGP_CUDA(cudaEventRecord(ev.e[0], stream));
  }
  if (k > 1) {
    FMGP_CUDA(fmgp::knn_exact(X + row_begin * d, nrows, X, n, d, k - 1, row_begin, nullptr, 1, S_out, nullptr,
                                   sms, stream));
  } else {
    FMGP_CUDA(fmgp::self_rows_launch(S_out, nrows, row_begin, stream));
  }
  DevBuf<unsigned long long> fmin;
  FMGP_CUDA(fmin.alloc(1, stream));
  FMGP_CUDA(cudaMemsetAsync(fmin.p, 0xFF, sizeof(unsigned long long), stream));
  if (timing) FMGP_CUDA(cudaEventRecord(ev.e[1], stream));
  FMGP_CUDA(fmgp::fused_solve(X, Y, d, m, S_out, nrows, row_begin, k, kp, C_out, nullptr, fmin.p, sms, stream));
  if (timing) {
    FMGP_CUDA(cudaEventRecord(ev.e[2], stream));
    std::lock_guard<std::mutex> lk(g_stage_mu);
    g_stage_events.push_back(ev);
  }
  unsigned long long host_min = ~0ull;
  FMGP_CUDA(cudaMemcpyAsync(&host_min, fmin.p, sizeof(host_min), cudaMemcpyDeviceToHost, stream));
  FMGP_CUDA(cudaStreamSynchronize(stream));
  if (host_min != ~0ull) {
    if (failed_row) *failed_row = static_cast<int64_t>(host_min);
    return fail(FMGP_ENUMERIC, "Cholesky factorization failed in precompute row " + std::to_string(host_min) +
                                   " after jitter escalation up to 1e-6");
  }
  return FMGP_OK;
}

int check_solve_shape(int32_t k, int32_t d, int32_t m) {
  (void)k;
  (void)d;
  if (m < 1) return fail(FMGP_EINVAL, "number of outputs m must be >= 1");
  return FMGP_OK;
}

bool knn_force_brute() {
  static const bool force_brute = [] {
    const char* e = std::getenv("FMGP_KNN");
    return e != nullptr && std::string(e) == "brute";
  }();
  return force_brute;
}

// `grid`: a model handle's prebuilt predict grid (d <= 3), or null to build one for this call.
int predict_device_impl(const double* X, const int32_t* S, const double* C, int64_t n, int32_t d, int32_t k,
                        int32_t m, const fmgp::KParams& kp, const double* mean_offset_dev, const double* Z,
                        int64_t nz, double* out, int32_t* nn_out, cudaStream_t stream, const void* grid = nullptr) {
  if (nz <= 0) return FMGP_OK;
  const int sms = num_sms_current();
  if (!knn_force_brute() && d <= 3) {
    if (grid != nullptr)
      FMGP_CUDA(fmgp::predict_grid_cached(grid, X, S, C, k, m, kp, mean_offset_dev, Z, nz, out, nn_out, sms, stream));
    else
      FMGP_CUDA(fmgp::predict_grid(X, n, d, S, C, k, m, kp, mean_offset_dev, Z, nz, out, nn_out, sms, stream));
    return FMGP_OK;
  }
  DevBuf<int32_t> nn_tmp;
  int32_t* nn = nn_out;
  if (nn == nullptr) {
    FMGP_CUDA(nn_tmp.alloc(static_cast<size_t>(nz), stream));
    nn = nn_tmp.p;
  }
  FMGP_CUDA(fmgp::knn_exact(Z, nz, X, n, d, 1, -1, nullptr, 0, nn, nullptr, sms, stream));
  FMGP_CUDA(fmgp::predict_gather(X, S, C, d, k, m, kp, mean_offset_dev, Z, nz, nn, out, sms, stream));
  return FMGP_OK;
}

// Host-buffer batches that take the chunked, device-checked path of replica_predict_host:
// the cell-grid predict (d <= 3) from 65536 test points up.
bool predict_pipelined(const fmgp_model* mdl, int64_t nz) {
  return mdl->d <= 3 && nz >= 65536 && !knn_force_brute();
}

// One replica's share of a host-buffer predict: H2D of the test points, the
// walk / 1-NN + gather-kernel-dot, D2H of the means (and 1-NN indices).
int replica_predict_host(const fmgp_model* mdl, const fmgp_model_replica& r, const double* Z, int64_t nz, double* out,
                         int32_t* nn_out) {
  if (nz <= 0) return FMGP_OK;
  FMGP_CUDA(cudaSetDevice(r.device));
  if (predict_pipelined(mdl, nz)) {
    // Large low-d batches go through in chunks on three streams: the H2D copy of chunk i + 1 and
    // the D2H copy of chunk i - 1 overlap chunk i's kernels. The finiteness check of Z (done by the
    // caller on the host for small batches) runs on the device copy instead of a host scan of the
    // whole batch: non-finite coordinates are counted and zeroed in the device copy (so the cell
    // sort and the walk run on valid points), and a non-zero count becomes the error return after
    // the final synchronise. Per-point results do not depend on the chunking.
    constexpr int kStreams = 3;
    // chunks per call: 4 (cfg5, 8e6 points: 7.19 ms; 8 chunks 7.47 ms, 16 chunks 8.13 ms, 3 chunks 7.43 ms —
    // each chunk pays its own cell sort and launch train; fewer chunks expose more of the first copy)
    const char* pce = std::getenv("FMGP_PREDICT_CHUNKS");
    const int64_t want = pce != nullptr && std::atoi(pce) > 0 ? std::atoi(pce) : 4;
    const int64_t chunk = std::max<int64_t>(262144, (nz + want - 1) / want);
    const int nchunks = static_cast<int>((nz + chunk - 1) / chunk);
    Stream st[kStreams];
    for (auto& q : st) FMGP_CUDA(q.create());
    DevBuf<double> dZ, dO;
    DevBuf<int32_t> dN;
    DevBuf<unsigned int> bad;
    FMGP_CUDA(dZ.alloc(static_cast<size_t>(nz) * mdl->d, st[0].s));
    FMGP_CUDA(dO.alloc(static_cast<size_t>(nz) * mdl->m, st[0].s));
    if (nn_out) FMGP_CUDA(dN.alloc(static_cast<size_t>(nz), st[0].s));
    FMGP_CUDA(bad.alloc(static_cast<size_t>(nchunks), st[0].s));
    cudaEvent_t ready = nullptr;
    FMGP_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    FMGP_CUDA(cudaEventRecord(ready, st[0].s));
    for (int q = 1; q < kStreams; ++q) FMGP_CUDA(cudaStreamWaitEvent(st[q].s, ready, 0));
    const int sms = num_sms_current();
    int rc = FMGP_OK;
    for (int c = 0; c < nchunks && rc == FMGP_OK; ++c) {
      cudaStream_t q = st[c % kStreams].s;
      const int64_t b = c * chunk, e = std::min<int64_t>(nz, b + chunk);
      double* z = dZ.p + b * mdl->d;
      cudaError_t ce = cudaMemcpyAsync(z, Z + b * mdl->d, sizeof(double) * (e - b) * mdl->d, cudaMemcpyHostToDevice, q);
      if (ce == cudaSuccess) ce = fmgp::nonfinite_zero_launch(z, (e - b) * mdl->d, bad.p + c, sms, q);
      if (ce != cudaSuccess) {
        rc = cuda_fail(ce, "fmgp_model_predict");
        break;
      }
      rc = predict_device_impl(r.X, r.S, r.C, mdl->n, mdl->d, mdl->k, mdl->m, mdl->kp, r.mo, z, e - b,
                               dO.p + b * mdl->m, nn_out ? dN.p + b : nullptr, q, r.grid);
      if (rc != FMGP_OK) break;
      ce = cudaMemcpyAsync(out + b * mdl->m, dO.p + b * mdl->m, sizeof(double) * (e - b) * mdl->m,
                           cudaMemcpyDeviceToHost, q);
      if (ce == cudaSuccess && nn_out)
        ce = cudaMemcpyAsync(nn_out + b, dN.p + b, sizeof(int32_t) * (e - b), cudaMemcpyDeviceToHost, q);
      if (ce != cudaSuccess) rc = cuda_fail(ce, "fmgp_model_predict");
    }
    std::vector<unsigned int> hbad(static_cast<size_t>(nchunks), 0u);
    for (auto& q : st) {
      const cudaError_t ce = cudaStreamSynchronize(q.s);
      if (ce != cudaSuccess && rc == FMGP_OK) rc = cuda_fail(ce, "fmgp_model_predict");
    }
    cudaEventDestroy(ready);
    if (rc != FMGP_OK) return rc;
    FMGP_CUDA(cudaMemcpy(hbad.data(), bad.p, sizeof(unsigned int) * nchunks, cudaMemcpyDeviceToHost));
    for (unsigned int v : hbad)
      if (v != 0) return fail(FMGP_EINVAL, "fast_predict: non-finite test point");
    return FMGP_OK;
  }
  Stream st;
  FMGP_CUDA(st.create());
  DevBuf<double> dZ, dO;
  DevBuf<int32_t> dN;
  FMGP_CUDA(dZ.alloc(static_cast<size_t>(nz) * mdl->d, st.s));
  FMGP_CUDA(dO.alloc(static_cast<size_t>(nz) * mdl->m, st.s));
  if (nn_out) FMGP_CUDA(dN.alloc(static_cast<size_t>(nz), st.s));
  FMGP_CUDA(cudaMemcpyAsync(dZ.p, Z, sizeof(double) * nz * mdl->d, cudaMemcpyHostToDevice, st.s));
  int rc = predict_device_impl(r.X, r.S, r.C, mdl->n, mdl->d, mdl->k, mdl->m, mdl->kp, r.mo, dZ.p, nz, dO.p,
                               nn_out ? dN.p : nullptr, st.s, r.grid);
  if (rc != FMGP_OK) return rc;
  FMGP_CUDA(cudaMemcpyAsync(out, dO.p, sizeof(double) * nz * mdl->m, cudaMemcpyDeviceToHost, st.s));
  if (nn_out) FMGP_CUDA(cudaMemcpyAsync(nn_out, dN.p, sizeof(int32_t) * nz, cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaStreamSynchronize(st.s));
  return FMGP_OK;
}

}  // namespace

namespace fmgp_capi {

bool stage_timing_on() { return g_stage_timing.load(std::memory_order_relaxed) != 0; }

void stage_push(cudaEvent_t knn_begin, cudaEvent_t knn_end, cudaEvent_t solve_end) {
  StageEvents ev{};
  ev.e[0] = knn_begin;
  ev.e[1] = knn_end;
  ev.e[2] = solve_end;
  std::lock_guard<std::mutex> lk(g_stage_mu);
  g_stage_events.push_back(ev);
}

cudaError_t replica_finish(fmgp_model_replica& r, int64_t n, int32_t d, int32_t k, int32_t m, const double* mean_offset_host) {
  cudaError_t e = cudaMalloc(&r.mo, sizeof(double) * m);
  if (e == cudaSuccess) e = cudaMemcpy(r.mo, mean_offset_host, sizeof(double) * m, cudaMemcpyHostToDevice);
  // the reference's model owns its NeighborIndex (fast_predict.cpp:127-129);
  // here that is the predict walk's cell grid of X, built once per replica
  if (e == cudaSuccess && d <= 3 && !knn_force_brute()) r.grid = fmgp::predict_grid_cache_build(r.X, n, d, 0, &e);
  // and a cell-ordered copy of the model rows, so predict reads them (and the
  // neighbours' coordinates) with the locality of the cell-sorted test points
  if (e == cudaSuccess && r.grid != nullptr) e = fmgp::predict_grid_cache_attach(r.grid, r.S, r.C, k, m, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return e;
}

void replica_release(fmgp_model_replica& r) {
  cudaSetDevice(r.device);
  if (r.grid) fmgp::predict_grid_cache_free(r.grid);
  if (r.owns) {
    if (r.X) cudaFree(r.X);
    if (r.S) cudaFree(r.S);
    if (r.C) cudaFree(r.C);
  }
  if (r.mo) cudaFree(r.mo);
  r = fmgp_model_replica{};
}

}  // namespace fmgp_capi

namespace fmgp {
static std::atomic<int64_t> g_launches{0};
void note_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace fmgp


// Host-buffer precompute of rows [row_begin, row_end) (X, Y full; S_out and
// C_out hold the shard's rows). K1 for the shard, then K2 in row chunks; a
// second stream reads S back as soon as K1 is done and each chunk's C rows as
// soon as that chunk is solved, so the host read-back (the largest transfer:
// rows*k*m doubles) overlaps the solve.
static int precompute_host_rows(const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                                const fmgp_kernel_params* params, int32_t k, int64_t row_begin, int64_t row_end,
                                int32_t* S_out, double* C_out, int64_t* failed_row) {
  if (failed_row) *failed_row = -1;
  fmgp::KParams kp;
  int rc;
  if ((rc = make_kparams(params, &kp)) != FMGP_OK) return rc;
  if (k < 1 || k > n) return fail(FMGP_EINVAL, "precompute: k out of range");
  // shape checks now; the finiteness scan of X runs below, while X and Y copy
  if ((rc = check_points(nullptr, n, d)) != FMGP_OK) return rc;
  if ((rc = check_solve_shape(k, d, m)) != FMGP_OK) return rc;
  if (row_begin < 0 || row_end > n || row_begin > row_end) return fail(FMGP_EINVAL, "precompute: bad row range");
  if ((rc = require_device()) != FMGP_OK) {  // argument errors still take precedence
    if (!all_finite(X, n * d)) return fail(FMGP_EINVAL, "NeighborIndex: non-finite coordinates");
    return rc;
  }
  const int64_t rows = row_end - row_begin;
  if (rows == 0) return all_finite(X, n * d) ? FMGP_OK : fail(FMGP_EINVAL, "NeighborIndex: non-finite coordinates");
  Stream st;
  FMGP_CUDA(st.create());
  // FMGP_TRACE=1: stage timeline of this call on stderr (CUDA events on the
  // work and read-back streams, host issue time), for the e2e breakdown
  static const bool trace = [] {
    const char* e = std::getenv("FMGP_TRACE");
    return e != nullptr && e[0] == '1';
  }();
  const auto host_t0 = std::chrono::steady_clock::now();
  cudaEvent_t tev[6] = {};
  if (trace)
    for (auto& e : tev) cudaEventCreate(&e);
  auto mark = [&](int i, cudaStream_t s) {
    if (trace) cudaEventRecord(tev[i], s);
  };
  mark(0, st.s);
  DevBuf<double> dX, dY, dC;
  DevBuf<int32_t> dS;
  FMGP_CUDA(dX.alloc(static_cast<size_t>(n) * d, st.s));
  FMGP_CUDA(dY.alloc(static_cast<size_t>(n) * m, st.s));
  FMGP_CUDA(dS.alloc(static_cast<size_t>(rows) * k, st.s));
  FMGP_CUDA(dC.alloc(static_cast<size_t>(rows) * k * m, st.s));
  // X goes first on the work stream (the kNN needs it); Y only feeds the solve,
  // so it is copied on the read-back stream while the kNN runs
  Stream rb_st;
  FMGP_CUDA(rb_st.create());
  FMGP_CUDA(cudaMemcpyAsync(dX.p, X, sizeof(double) * n * d, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dY.p, Y, sizeof(double) * n * m, cudaMemcpyHostToDevice, rb_st.s));
  cudaEvent_t y_ready;
  FMGP_CUDA(cudaEventCreateWithFlags(&y_ready, cudaEventDisableTiming));
  struct EvOne {
    cudaEvent_t e;
    ~EvOne() { cudaEventDestroy(e); }
  } y_guard{y_ready};
  FMGP_CUDA(cudaEventRecord(y_ready, rb_st.s));
  const int sms = num_sms_current();
  {  // NeighborIndex::build's finiteness check, on the device copy of X (a 16 MB
     // host scan costs ~1 ms of host time the kNN launch would wait for)
    DevBuf<unsigned int> nbad;
    FMGP_CUDA(nbad.alloc(1, st.s));
    FMGP_CUDA(fmgp::nonfinite_count_launch(dX.p, n * d, nbad.p, sms, st.s));
    unsigned int host_bad = 0;
    FMGP_CUDA(cudaMemcpyAsync(&host_bad, nbad.p, sizeof(host_bad), cudaMemcpyDeviceToHost, st.s));
    FMGP_CUDA(cudaStreamSynchronize(st.s));
    if (host_bad != 0) {
      cudaStreamSynchronize(rb_st.s);
      return fail(FMGP_EINVAL, "NeighborIndex: non-finite coordinates");
    }
  }
  mark(1, st.s);
  if (k > 1) {
    FMGP_CUDA(fmgp::knn_exact(dX.p + static_cast<size_t>(row_begin) * d, rows, dX.p, n, d, k - 1, row_begin, nullptr,
                              1, dS.p, nullptr, sms, st.s));
  } else {
    FMGP_CUDA(fmgp::self_rows_launch(dS.p, rows, row_begin, st.s));
  }
  mark(2, st.s);
  FMGP_CUDA(cudaStreamWaitEvent(st.s, y_ready, 0));  // the solve reads Y
  std::vector<cudaEvent_t> evs;
  struct EvGuard {
    std::vector<cudaEvent_t>& v;
    ~EvGuard() {
      for (auto e : v) cudaEventDestroy(e);
    }
  } evg{evs};
  auto handoff = [&]() -> cudaError_t {  // rb_st waits for everything issued on st so far
    cudaEvent_t e;
    cudaError_t err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (err != cudaSuccess) return err;
    evs.push_back(e);
    err = cudaEventRecord(e, st.s);
    return err == cudaSuccess ? cudaStreamWaitEvent(rb_st.s, e, 0) : err;
  };
  FMGP_CUDA(handoff());
  FMGP_CUDA(cudaMemcpyAsync(S_out, dS.p, sizeof(int32_t) * rows * k, cudaMemcpyDeviceToHost, rb_st.s));
  DevBuf<unsigned long long> fmin;
  FMGP_CUDA(fmin.alloc(1, st.s));
  FMGP_CUDA(cudaMemsetAsync(fmin.p, 0xFF, sizeof(unsigned long long), st.s));
  // chunks of rows/16, halving once fewer than two remain (down to 8192
  // rows), so the read-back of the last chunk, which nothing hides, is short
  const int64_t base = std::max<int64_t>(int64_t(1) << 15, (rows + 15) / 16);
  for (int64_t rb = 0; rb < rows;) {
    const int64_t left = rows - rb;
    const int64_t chunk = left <= 8192 ? left : std::max<int64_t>(8192, std::min(base, (left + 1) / 2));
    const int64_t re = rb + chunk;
    const size_t c0 = static_cast<size_t>(rb) * k * m, cn = static_cast<size_t>(re - rb) * k * m;
    FMGP_CUDA(fmgp::fused_solve(dX.p, dY.p, d, m, dS.p + static_cast<size_t>(rb) * k, re - rb, row_begin + rb, k, kp,
                                dC.p + c0, nullptr, fmin.p, sms, st.s));
    FMGP_CUDA(handoff());
    FMGP_CUDA(cudaMemcpyAsync(C_out + c0, dC.p + c0, sizeof(double) * cn, cudaMemcpyDeviceToHost, rb_st.s));
    rb = re;
  }
  mark(3, st.s);
  mark(4, rb_st.s);
  const double host_issue_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
  unsigned long long host_min = ~0ull;
  FMGP_CUDA(cudaMemcpyAsync(&host_min, fmin.p, sizeof(host_min), cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaStreamSynchronize(st.s));
  FMGP_CUDA(cudaStreamSynchronize(rb_st.s));
  if (trace) {
    float t[5] = {};
    for (int i = 1; i < 5; ++i) cudaEventElapsedTime(&t[i], tev[0], tev[i]);
    const double host_total_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
    std::fprintf(stderr,
                 "[fmgp trace] precompute rows %lld: h2d done %.3f ms, kNN done %.3f, solve done %.3f, "
                 "read-back done %.3f (device, from call start); host issue %.3f ms, host total %.3f ms\n",
                 static_cast<long long>(rows), t[1], t[2], t[3], t[4], host_issue_ms, host_total_ms);
    for (auto e : tev) cudaEventDestroy(e);
  }
  if (host_min != ~0ull) {
    if (failed_row) *failed_row = static_cast<int64_t>(host_min);
    return fail(FMGP_ENUMERIC, "Cholesky factorization failed in precompute row " + std::to_string(host_min) +
                                   " after jitter escalation up to 1e-6");
  }
  return FMGP_OK;
}

extern "C" {

int fmgp_abi_version(void) { return FMGP_ABI_VERSION; }

void fmgp_set_stage_timing(int on) { g_stage_timing.store(on ? 1 : 0); }

int fmgp_stage_times(double* knn_ms, double* solve_ms, int64_t* calls) {
  std::vector<StageEvents> evs;
  {
    std::lock_guard<std::mutex> lk(g_stage_mu);
    evs.swap(g_stage_events);
  }
  double a = 0.0, b = 0.0;
  int rc = FMGP_OK;
  for (auto& ev : evs) {
    float t01 = 0.f, t12 = 0.f;
    if (rc == FMGP_OK) {
      cudaError_t e = cudaEventSynchronize(ev.e[2]);
      if (e == cudaSuccess) e = cudaEventElapsedTime(&t01, ev.e[0], ev.e[1]);
      if (e == cudaSuccess) e = cudaEventElapsedTime(&t12, ev.e[1], ev.e[2]);
      if (e != cudaSuccess) rc = cuda_fail(e, "fmgp_stage_times");
    }
    a += t01;
    b += t12;
    for (auto& x : ev.e) cudaEventDestroy(x);
  }
  if (knn_ms) *knn_ms = a;
  if (solve_ms) *solve_ms = b;
  if (calls) *calls = static_cast<int64_t>(evs.size());
  return rc;
}
const char* fmgp_last_error(void) { return g_err.c_str(); }
int64_t fmgp_launch_count(void) { return fmgp::g_launches.load(); }

int fmgp_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

int fmgp_validate_kernel(const fmgp_kernel_params* p) {
  fmgp::KParams kp;
  return make_kparams(p, &kp);
}

int fmgp_precompute(const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                    const fmgp_kernel_params* params, int32_t k, int32_t* S_out, double* C_out,
                    int64_t* failed_row) {
  // FMGP_DEVICES="0,1,..." (several entries): rows split contiguously over the
  // listed devices, one host thread per device running the shard path into
  // the caller's buffers. Rows are independent, so S and C are identical for
  // any device list; a failure reports the lowest failing row over all shards.
  DeviceGuard dg;
  std::vector<int> devs;
  if (const char* e = std::getenv("FMGP_DEVICES")) {
    for (const char* p = e; *p;) {
      char* end = nullptr;
      const long v = std::strtol(p, &end, 10);
      if (end == p) break;
      devs.push_back(static_cast<int>(v));
      p = (*end == ',') ? end + 1 : end;
    }
  }
  if (devs.size() <= 1) {
    if (devs.size() == 1 && cudaSetDevice(devs[0]) != cudaSuccess)
      return fail(FMGP_ECUDA, "FMGP_DEVICES names an unusable device");
    return precompute_host_rows(X, Y, n, d, m, params, k, 0, n, S_out, C_out, failed_row);
  }
  if (failed_row) *failed_row = -1;
  int caller_dev = 0;
  cudaGetDevice(&caller_dev);
  const int g = static_cast<int>(devs.size());
  const int64_t per = (n + g - 1) / g;
  std::vector<int> rcs(g, FMGP_OK);
  std::vector<int64_t> fails(g, -1);
  std::vector<std::string> msgs(g);
  std::vector<std::thread> th;
  for (int r = 0; r < g; ++r) {
    th.emplace_back([&, r] {
      const int64_t b = std::min<int64_t>(n, r * per), e = std::min<int64_t>(n, b + per);
      if (cudaSetDevice(devs[r]) != cudaSuccess) {
        rcs[r] = FMGP_ECUDA;
        msgs[r] = "FMGP_DEVICES names an unusable device";
        return;
      }
      rcs[r] = precompute_host_rows(X, Y, n, d, m, params, k, b, e, S_out + static_cast<size_t>(b) * k,
                                    C_out + static_cast<size_t>(b) * k * m, &fails[r]);
      if (rcs[r] != FMGP_OK) msgs[r] = g_err;  // thread-local error text of this worker
    });
  }
  for (auto& t : th) t.join();
  cudaSetDevice(caller_dev);
  int worst = -1;
  for (int r = 0; r < g; ++r) {
    if (rcs[r] == FMGP_OK) continue;
    // argument errors are identical on every shard; numeric failures: the lowest row
    if (worst < 0 || (rcs[r] == FMGP_ENUMERIC && rcs[worst] == FMGP_ENUMERIC && fails[r] < fails[worst])) worst = r;
  }
  if (worst < 0) return FMGP_OK;
  if (failed_row) *failed_row = fails[worst];
  return fail(rcs[worst], msgs[worst]);
}

int fmgp_precompute_rows(const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                         const fmgp_kernel_params* params, int32_t k, int64_t row_begin, int64_t row_end,
                         int32_t* S_out, double* C_out, int64_t* failed_row) {
  return precompute_host_rows(X, Y, n, d, m, params, k, row_begin, row_end, S_out, C_out, failed_row);
}

int fmgp_precompute_device(const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                           const fmgp_kernel_params* params, int32_t k, int64_t row_begin, int64_t row_end,
                           int32_t* S_out, double* C_out, int64_t* failed_row, void* stream) {
  if (failed_row) *failed_row = -1;
  fmgp::KParams kp;
  int rc;
  if ((rc = make_kparams(params, &kp)) != FMGP_OK) return rc;
  if (k < 1 || k > n) return fail(FMGP_EINVAL, "precompute: k out of range");
  if ((rc = check_points(nullptr, n, d)) != FMGP_OK) return rc;
  if ((rc = check_solve_shape(k, d, m)) != FMGP_OK) return rc;
  if (row_begin < 0 || row_end > n || row_begin > row_end) return fail(FMGP_EINVAL, "precompute: bad row range");
  if ((rc = require_device()) != FMGP_OK) return rc;
  return precompute_device_impl(X, Y, n, d, m, kp, k, row_begin, row_end, S_out, C_out, failed_row,
                                static_cast<cudaStream_t>(stream));
}

int fmgp_knn_rows_device(const double* X, int64_t n, int32_t d, int32_t k, int64_t row_begin, int64_t row_end,
                         int32_t* S_out, void* stream) {
  int rc;
  if (k < 1 || k > n) return fail(FMGP_EINVAL, "precompute: k out of range");
  if ((rc = check_points(nullptr, n, d)) != FMGP_OK) return rc;
  if (row_begin < 0 || row_end > n || row_begin > row_end) return fail(FMGP_EINVAL, "precompute: bad row range");
  if ((rc = require_device()) != FMGP_OK) return rc;
  const int64_t rows = row_end - row_begin;
  if (rows == 0) return FMGP_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (k > 1) {
    FMGP_CUDA(fmgp::knn_exact(X + row_begin * d, rows, X, n, d, k - 1, row_begin, nullptr, 1, S_out, nullptr,
                              num_sms_current(), st));
  } else {
    FMGP_CUDA(fmgp::self_rows_launch(S_out, rows, row_begin, st));
  }
  return FMGP_OK;
}

int fmgp_solve_rows_device(const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                           const fmgp_kernel_params* params, int32_t k, const int32_t* S_rows, int64_t nrows,
                           int64_t row_begin, double* C_out, uint64_t* fail_dev, int64_t* failed_row,
                           void* stream) {
  if (failed_row) *failed_row = -1;
  fmgp::KParams kp;
  int rc;
  if ((rc = make_kparams(params, &kp)) != FMGP_OK) return rc;
  if (k < 1 || k > n) return fail(FMGP_EINVAL, "precompute: k out of range");
  if ((rc = check_points(nullptr, n, d)) != FMGP_OK) return rc;
  if ((rc = check_solve_shape(k, d, m)) != FMGP_OK) return rc;
  if (nrows < 0 || row_begin < 0) return fail(FMGP_EINVAL, "precompute: bad row range");
  if ((rc = require_device()) != FMGP_OK) return rc;
  if (nrows == 0) return FMGP_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (fail_dev != nullptr) {  // asynchronous: the caller min-combines and checks the word later
    FMGP_CUDA(fmgp::fused_solve(X, Y, d, m, S_rows, nrows, row_begin, k, kp, C_out, nullptr,
                                reinterpret_cast<unsigned long long*>(fail_dev), num_sms_current(), st));
    return FMGP_OK;
  }
  DevBuf<unsigned long long> fmin;
  FMGP_CUDA(fmin.alloc(1, st));
  FMGP_CUDA(cudaMemsetAsync(fmin.p, 0xFF, sizeof(unsigned long long), st));
  FMGP_CUDA(fmgp::fused_solve(X, Y, d, m, S_rows, nrows, row_begin, k, kp, C_out, nullptr, fmin.p,
                              num_sms_current(), st));
  unsigned long long host_min = ~0ull;
  FMGP_CUDA(cudaMemcpyAsync(&host_min, fmin.p, sizeof(host_min), cudaMemcpyDeviceToHost, st));
  FMGP_CUDA(cudaStreamSynchronize(st));
  if (host_min != ~0ull) {
    if (failed_row) *failed_row = static_cast<int64_t>(host_min);
    return fail(FMGP_ENUMERIC, "Cholesky factorization failed in precompute row " + std::to_string(host_min) +
                                   " after jitter escalation up to 1e-6");
  }
  return FMGP_OK;
}

int fmgp_query_knn_device(const double* P, int64_t np, int32_t d, const double* Q, int64_t nq, int32_t k,
                          int64_t self_offset, int32_t* idx_out, double* dist_sq_out, void* stream) {
  int rc;
  if ((rc = check_points(nullptr, np, d)) != FMGP_OK) return rc;
  if (k < 1 || k > np - (self_offset >= 0 ? 1 : 0)) return fail(FMGP_EINVAL, "query_knn: k out of range");
  if ((rc = require_device()) != FMGP_OK) return rc;
  FMGP_CUDA(fmgp::knn_exact(Q, nq, P, np, d, k, self_offset, nullptr, 0, idx_out, dist_sq_out,
                                 num_sms_current(), static_cast<cudaStream_t>(stream)));
  return FMGP_OK;
}

int fmgp_query_knn(const double* P, int64_t np, int32_t d, const double* Q, int64_t nq, int32_t k,
                   const int32_t* exclude, int32_t* idx_out, double* dist_out) {
  int rc;
  if ((rc = check_points(P, np, d)) != FMGP_OK) return rc;
  bool any_excl = false;
  if (exclude != nullptr)
    for (int64_t q = 0; q < nq; ++q) any_excl |= exclude[q] >= 0;
  if (k < 1 || k > np - (any_excl ? 1 : 0)) return fail(FMGP_EINVAL, "query_knn: k out of range");
  if (!all_finite(Q, nq * d)) return fail(FMGP_EINVAL, "query_knn: non-finite query");
  if ((rc = require_device()) != FMGP_OK) return rc;
  if (nq <= 0) return FMGP_OK;
  Stream st;
  FMGP_CUDA(st.create());
  DevBuf<double> dP, dQ, dD;
  DevBuf<int32_t> dI, dE;
  FMGP_CUDA(dP.alloc(static_cast<size_t>(np) * d, st.s));
  FMGP_CUDA(dQ.alloc(static_cast<size_t>(nq) * d, st.s));
  FMGP_CUDA(dI.alloc(static_cast<size_t>(nq) * k, st.s));
  FMGP_CUDA(dD.alloc(static_cast<size_t>(nq) * k, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dP.p, P, sizeof(double) * np * d, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dQ.p, Q, sizeof(double) * nq * d, cudaMemcpyHostToDevice, st.s));
  if (exclude != nullptr) {
    FMGP_CUDA(dE.alloc(static_cast<size_t>(nq), st.s));
    FMGP_CUDA(cudaMemcpyAsync(dE.p, exclude, sizeof(int32_t) * nq, cudaMemcpyHostToDevice, st.s));
  }
  FMGP_CUDA(fmgp::knn_exact(dQ.p, nq, dP.p, np, d, k, -1, dE.p, 0, dI.p, dD.p, num_sms_current(), st.s));
  FMGP_CUDA(fmgp::sqrt_inplace_launch(dD.p, nq * k, st.s));
  FMGP_CUDA(cudaMemcpyAsync(idx_out, dI.p, sizeof(int32_t) * nq * k, cudaMemcpyDeviceToHost, st.s));
  if (dist_out) FMGP_CUDA(cudaMemcpyAsync(dist_out, dD.p, sizeof(double) * nq * k, cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaStreamSynchronize(st.s));
  return FMGP_OK;
}

int fmgp_nearest_device(const double* P, int64_t np, int32_t d, const double* Q, int64_t nq, int32_t* idx_out,
                        void* stream) {
  int rc;
  if ((rc = check_points(nullptr, np, d)) != FMGP_OK) return rc;
  if ((rc = require_device()) != FMGP_OK) return rc;
  FMGP_CUDA(fmgp::knn_exact(Q, nq, P, np, d, 1, -1, nullptr, 0, idx_out, nullptr, num_sms_current(),
                                 static_cast<cudaStream_t>(stream)));
  return FMGP_OK;
}

int fmgp_nearest(const double* P, int64_t np, int32_t d, const double* Q, int64_t nq, int32_t* idx_out) {
  int rc;
  if ((rc = check_points(P, np, d)) != FMGP_OK) return rc;
  if (!all_finite(Q, nq * d)) return fail(FMGP_EINVAL, "nearest_training_point: non-finite query");
  if ((rc = require_device()) != FMGP_OK) return rc;
  if (nq <= 0) return FMGP_OK;
  Stream st;
  FMGP_CUDA(st.create());
  DevBuf<double> dP, dQ;
  DevBuf<int32_t> dI;
  FMGP_CUDA(dP.alloc(static_cast<size_t>(np) * d, st.s));
  FMGP_CUDA(dQ.alloc(static_cast<size_t>(nq) * d, st.s));
  FMGP_CUDA(dI.alloc(static_cast<size_t>(nq), st.s));
  FMGP_CUDA(cudaMemcpyAsync(dP.p, P, sizeof(double) * np * d, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dQ.p, Q, sizeof(double) * nq * d, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(fmgp::knn_exact(dQ.p, nq, dP.p, np, d, 1, -1, nullptr, 0, dI.p, nullptr, num_sms_current(), st.s));
  FMGP_CUDA(cudaMemcpyAsync(idx_out, dI.p, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaStreamSynchronize(st.s));
  return FMGP_OK;
}

int fmgp_index_create(const double* P, int64_t np, int32_t d, int32_t device, fmgp_index** out) {
  if (out == nullptr) return fail(FMGP_EINVAL, "index output pointer is null");
  *out = nullptr;
  int rc;
  if ((rc = check_points(P, np, d)) != FMGP_OK) return rc;
  if ((rc = require_device()) != FMGP_OK) return rc;
  DeviceGuard dg;
  if (device < 0) FMGP_CUDA(cudaGetDevice(&device));  // -1: the calling thread's current device
  FMGP_CUDA(cudaSetDevice(device));
  auto* ix = new fmgp_index();
  ix->device = device;
  ix->n = np;
  ix->d = d;
  cudaError_t e = cudaMalloc(&ix->P, sizeof(double) * np * d);
  if (e == cudaSuccess) e = cudaMemcpy(ix->P, P, sizeof(double) * np * d, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && d <= 3 && !knn_force_brute()) ix->grid = fmgp::predict_grid_cache_build(ix->P, np, d, 0, &e);
  if (e != cudaSuccess) {
    fmgp_index_destroy(ix);
    return cuda_fail(e, "fmgp_index_create");
  }
  *out = ix;
  return FMGP_OK;
}

void fmgp_index_destroy(fmgp_index* ix) {
  if (ix == nullptr) return;
  DeviceGuard dg;
  cudaSetDevice(ix->device);
  if (ix->grid) fmgp::predict_grid_cache_free(ix->grid);
  if (ix->P) cudaFree(ix->P);
  delete ix;
}

int fmgp_index_query_knn(const fmgp_index* ix, const double* Q, int64_t nq, int32_t k, const int32_t* exclude,
                         int32_t* idx_out, double* dist_out) {
  if (ix == nullptr) return fail(FMGP_EINVAL, "null index");
  bool any_excl = false;
  if (exclude != nullptr)
    for (int64_t q = 0; q < nq; ++q) any_excl |= exclude[q] >= 0;
  if (k < 1 || k > ix->n - (any_excl ? 1 : 0)) return fail(FMGP_EINVAL, "query_knn: k out of range");
  if (nq <= 0) return FMGP_OK;
  if (!all_finite(Q, nq * ix->d)) return fail(FMGP_EINVAL, "query_knn: non-finite query");
  DeviceGuard dg;
  FMGP_CUDA(cudaSetDevice(ix->device));
  Stream st;
  FMGP_CUDA(st.create());
  DevBuf<double> dQ, dD;
  DevBuf<int32_t> dI, dE;
  FMGP_CUDA(dQ.alloc(static_cast<size_t>(nq) * ix->d, st.s));
  FMGP_CUDA(dI.alloc(static_cast<size_t>(nq) * k, st.s));
  FMGP_CUDA(dD.alloc(static_cast<size_t>(nq) * k, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dQ.p, Q, sizeof(double) * nq * ix->d, cudaMemcpyHostToDevice, st.s));
  if (any_excl) {
    FMGP_CUDA(dE.alloc(static_cast<size_t>(nq), st.s));
    FMGP_CUDA(cudaMemcpyAsync(dE.p, exclude, sizeof(int32_t) * nq, cudaMemcpyHostToDevice, st.s));
  }
  FMGP_CUDA(fmgp::knn_exact(dQ.p, nq, ix->P, ix->n, ix->d, k, -1, dE.p, 0, dI.p, dD.p, num_sms_current(), st.s));
  FMGP_CUDA(fmgp::sqrt_inplace_launch(dD.p, nq * k, st.s));
  FMGP_CUDA(cudaMemcpyAsync(idx_out, dI.p, sizeof(int32_t) * nq * k, cudaMemcpyDeviceToHost, st.s));
  if (dist_out) FMGP_CUDA(cudaMemcpyAsync(dist_out, dD.p, sizeof(double) * nq * k, cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaStreamSynchronize(st.s));
  return FMGP_OK;
}

int fmgp_index_nearest(const fmgp_index* ix, const double* Q, int64_t nq, int32_t* idx_out) {
  if (ix == nullptr) return fail(FMGP_EINVAL, "null index");
  if (nq <= 0) return FMGP_OK;
  // the reference returns -1 for a NaN query and its caller indexes with it
  if (!all_finite(Q, nq * ix->d)) return fail(FMGP_EINVAL, "nearest_training_point: non-finite query");
  DeviceGuard dg;
  FMGP_CUDA(cudaSetDevice(ix->device));
  Stream st;
  FMGP_CUDA(st.create());
  DevBuf<double> dQ;
  DevBuf<int32_t> dI;
  FMGP_CUDA(dQ.alloc(static_cast<size_t>(nq) * ix->d, st.s));
  FMGP_CUDA(dI.alloc(static_cast<size_t>(nq), st.s));
  FMGP_CUDA(cudaMemcpyAsync(dQ.p, Q, sizeof(double) * nq * ix->d, cudaMemcpyHostToDevice, st.s));
  if (ix->grid != nullptr) {  // the cached walk grid, nearest only (no gather)
    fmgp::KParams none{};
    none.kind = 1;
    FMGP_CUDA(fmgp::predict_grid_cached(ix->grid, ix->P, nullptr, nullptr, 1, 1, none, nullptr, dQ.p, nq, nullptr,
                                        dI.p, num_sms_current(), st.s));
  } else {
    FMGP_CUDA(fmgp::knn_exact(dQ.p, nq, ix->P, ix->n, ix->d, 1, -1, nullptr, 0, dI.p, nullptr, num_sms_current(),
                              st.s));
  }
  FMGP_CUDA(cudaMemcpyAsync(idx_out, dI.p, sizeof(int32_t) * nq, cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaStreamSynchronize(st.s));
  return FMGP_OK;
}

int fmgp_index_distances(const fmgp_index* ix, const double* q, const int32_t* idx, int64_t cnt, double* out) {
  if (ix == nullptr) return fail(FMGP_EINVAL, "null index");
  for (int64_t e = 0; e < cnt; ++e)
    if (idx[e] < 0 || idx[e] >= ix->n) return fail(FMGP_EINVAL, "distance_to: bad query or index");
  if (cnt <= 0) return FMGP_OK;
  DeviceGuard dg;
  FMGP_CUDA(cudaSetDevice(ix->device));
  Stream st;
  FMGP_CUDA(st.create());
  DevBuf<double> dq, dO;
  DevBuf<int32_t> dI;
  FMGP_CUDA(dq.alloc(static_cast<size_t>(ix->d), st.s));
  FMGP_CUDA(dI.alloc(static_cast<size_t>(cnt), st.s));
  FMGP_CUDA(dO.alloc(static_cast<size_t>(cnt), st.s));
  FMGP_CUDA(cudaMemcpyAsync(dq.p, q, sizeof(double) * ix->d, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dI.p, idx, sizeof(int32_t) * cnt, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(fmgp::distances_launch(ix->P, ix->d, dq.p, dI.p, cnt, dO.p, st.s));
  FMGP_CUDA(cudaMemcpyAsync(out, dO.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaStreamSynchronize(st.s));
  return FMGP_OK;
}

int fmgp_predict_device(const double* X, const int32_t* S, const double* C, int64_t n, int32_t d, int32_t k,
                        int32_t m, const fmgp_kernel_params* params, const double* mean_offset, const double* Z,
                        int64_t nz, double* out, int32_t* nn_out, void* stream) {
  fmgp::KParams kp;
  int rc;
  if ((rc = make_kparams(params, &kp)) != FMGP_OK) return rc;
  if ((rc = check_points(nullptr, n, d)) != FMGP_OK) return rc;
  if (k < 1 || k > n || m < 1) return fail(FMGP_EINVAL, "predict: bad k or m");
  if ((rc = require_device()) != FMGP_OK) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  DevBuf<double> mo;
  FMGP_CUDA(mo.alloc(static_cast<size_t>(m), s));
  FMGP_CUDA(cudaMemcpyAsync(mo.p, mean_offset, sizeof(double) * m, cudaMemcpyHostToDevice, s));
  rc = predict_device_impl(X, S, C, n, d, k, m, kp, mo.p, Z, nz, out, nn_out, s);
  if (rc != FMGP_OK) return rc;
  // mean_offset may be a pageable stack array: make sure the copy finished.
  FMGP_CUDA(cudaStreamSynchronize(s));
  return FMGP_OK;
}

int fmgp_model_create(const double* X, const int32_t* S, const double* C, int64_t n, int32_t d, int32_t k,
                      int32_t m, const fmgp_kernel_params* params, const double* mean_offset, int32_t device,
                      fmgp_model** out) {
  if (out == nullptr) return fail(FMGP_EINVAL, "model output pointer is null");
  *out = nullptr;
  fmgp::KParams kp;
  int rc;
  if ((rc = make_kparams(params, &kp)) != FMGP_OK) return rc;
  if ((rc = check_points(X, n, d)) != FMGP_OK) return rc;
  if (k < 1 || k > n || m < 1) return fail(FMGP_EINVAL, "model: bad k or m");
  for (int64_t i = 0; i < n; ++i)
    if (S[i * k] != static_cast<int32_t>(i))
      return fail(FMGP_EINVAL, "neighbor table row does not start with its own index");
  if ((rc = require_device()) != FMGP_OK) return rc;
  DeviceGuard dg;
  if (device < 0) FMGP_CUDA(cudaGetDevice(&device));  // -1: the calling thread's current device
  FMGP_CUDA(cudaSetDevice(device));
  auto* mdl = new fmgp_model();
  mdl->n = n;
  mdl->d = d;
  mdl->k = k;
  mdl->m = m;
  mdl->kp = kp;
  mdl->reps.emplace_back();
  fmgp_model_replica& r = mdl->reps.back();
  r.device = device;
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = cudaMalloc(&r.X, sizeof(double) * n * d);
  if (e == cudaSuccess) e = cudaMalloc(&r.S, sizeof(int32_t) * n * k);
  if (e == cudaSuccess) e = cudaMalloc(&r.C, sizeof(double) * n * k * m);
  if (e == cudaSuccess) e = cudaMemcpy(r.X, X, sizeof(double) * n * d, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(r.S, S, sizeof(int32_t) * n * k, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(r.C, C, sizeof(double) * n * k * m, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = replica_finish(r, n, d, k, m, mean_offset);
  if (e != cudaSuccess) {
    fmgp_model_destroy(mdl);
    return cuda_fail(e, "fmgp_model_create");
  }
  *out = mdl;
  return FMGP_OK;
}

int fmgp_model_wrap_device(const double* X, const int32_t* S, const double* C, int64_t n, int32_t d, int32_t k,
                           int32_t m, const fmgp_kernel_params* params, const double* mean_offset, fmgp_model** out) {
  if (out == nullptr) return fail(FMGP_EINVAL, "model output pointer is null");
  *out = nullptr;
  fmgp::KParams kp;
  int rc;
  if ((rc = make_kparams(params, &kp)) != FMGP_OK) return rc;
  if ((rc = check_points(nullptr, n, d)) != FMGP_OK) return rc;
  if (k < 1 || k > n || m < 1) return fail(FMGP_EINVAL, "model: bad k or m");
  if ((rc = require_device()) != FMGP_OK) return rc;
  int dev = 0;
  FMGP_CUDA(cudaGetDevice(&dev));
  auto* mdl = new fmgp_model();
  mdl->n = n;
  mdl->d = d;
  mdl->k = k;
  mdl->m = m;
  mdl->kp = kp;
  mdl->reps.emplace_back();
  fmgp_model_replica& r = mdl->reps.back();
  r.device = dev;
  r.owns = false;
  r.X = const_cast<double*>(X);
  r.S = const_cast<int32_t*>(S);
  r.C = const_cast<double*>(C);
  cudaError_t e = replica_finish(r, n, d, k, m, mean_offset);
  if (e != cudaSuccess) {
    fmgp_model_destroy(mdl);
    return cuda_fail(e, "fmgp_model_wrap_device");
  }
  *out = mdl;
  return FMGP_OK;
}

int fmgp_model_replicas(const fmgp_model* mdl) { return mdl == nullptr ? 0 : static_cast<int>(mdl->reps.size()); }

int fmgp_model_predict(const fmgp_model* mdl, const double* Z, int64_t nz, double* out, int32_t* nn_out) {
  if (mdl == nullptr) return fail(FMGP_EINVAL, "null model");
  if (nz <= 0) return FMGP_OK;
  // a test point must have a nearest training point (the reference returns -1
  // from nearest_training_point for a NaN query and indexes with it)
  const int g = static_cast<int>(mdl->reps.size());
  const int64_t per_rep = (g == 1 || nz < 4096) ? nz : (nz + g - 1) / g;
  if (!predict_pipelined(mdl, per_rep) && !all_finite(Z, nz * mdl->d))  // else: checked on the device copy
    return fail(FMGP_EINVAL, "fast_predict: non-finite test point");
  DeviceGuard dg;
  // small batches (e.g. fast_predict_one) stay on one replica
  if (g == 1 || nz < 4096) return replica_predict_host(mdl, mdl->reps[0], Z, nz, out, nn_out);
  // test points split contiguously over the replicas (one host thread each)
  const int64_t per = (nz + g - 1) / g;
  std::vector<int> rcs(g, FMGP_OK);
  std::vector<std::string> msgs(g);
  std::vector<std::thread> th;
  for (int r = 0; r < g; ++r) {
    const int64_t b = std::min<int64_t>(nz, r * per), e = std::min<int64_t>(nz, b + per);
    th.emplace_back([&, r, b, e] {
      rcs[r] = replica_predict_host(mdl, mdl->reps[r], Z + b * mdl->d, e - b, out + b * mdl->m,
                                    nn_out ? nn_out + b : nullptr);
      if (rcs[r] != FMGP_OK) msgs[r] = g_err;
    });
  }
  for (auto& t : th) t.join();
  for (int r = 0; r < g; ++r)
    if (rcs[r] != FMGP_OK) return fail(rcs[r], msgs[r]);
  return FMGP_OK;
}

int fmgp_model_predict_device(const fmgp_model* mdl, const double* Z, int64_t nz, double* out, int32_t* nn_out,
                              void* stream) {
  if (mdl == nullptr) return fail(FMGP_EINVAL, "null model");
  if (nz <= 0) return FMGP_OK;
  int dev = 0;
  FMGP_CUDA(cudaGetDevice(&dev));
  for (const auto& r : mdl->reps)
    if (r.device == dev)
      return predict_device_impl(r.X, r.S, r.C, mdl->n, mdl->d, mdl->k, mdl->m, mdl->kp, r.mo, Z, nz, out, nn_out,
                                 static_cast<cudaStream_t>(stream), r.grid);
  return fail(FMGP_EINVAL, "model has no replica on the current device");
}

void fmgp_model_destroy(fmgp_model* mdl) {
  if (mdl == nullptr) return;
  DeviceGuard dg;
  for (auto& r : mdl->reps) replica_release(r);
  delete mdl;
}

int fmgp_predict(const double* X, const int32_t* S, const double* C, int64_t n, int32_t d, int32_t k, int32_t m,
                 const fmgp_kernel_params* params, const double* mean_offset, const double* Z, int64_t nz,
                 double* out, int32_t* nn_out) {
  int dev = 0;
  if (require_device() != FMGP_OK) return FMGP_ECUDA;
  FMGP_CUDA(cudaGetDevice(&dev));
  fmgp_model* mdl = nullptr;
  int rc = fmgp_model_create(X, S, C, n, d, k, m, params, mean_offset, dev, &mdl);
  if (rc != FMGP_OK) return rc;
  rc = fmgp_model_predict(mdl, Z, nz, out, nn_out);
  fmgp_model_destroy(mdl);
  return rc;
}

int fmgp_cov_matrix(const double* A, int64_t na, const double* B, int64_t nb, int32_t d,
                    const fmgp_kernel_params* params, double* K_out) {
  fmgp::KParams kp;
  int rc;
  if ((rc = make_kparams(params, &kp)) != FMGP_OK) return rc;
  if (d < 1) return fail(FMGP_EINVAL, "cov_matrix: point sets have mismatched dimension");
  if ((rc = require_device()) != FMGP_OK) return rc;
  if (B == nullptr) nb = na;
  if (na * nb == 0) return FMGP_OK;
  Stream st;
  FMGP_CUDA(st.create());
  DevBuf<double> dA, dB, dK;
  FMGP_CUDA(dA.alloc(static_cast<size_t>(na) * d, st.s));
  FMGP_CUDA(dK.alloc(static_cast<size_t>(na) * nb, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dA.p, A, sizeof(double) * na * d, cudaMemcpyHostToDevice, st.s));
  if (B != nullptr) {
    FMGP_CUDA(dB.alloc(static_cast<size_t>(nb) * d, st.s));
    FMGP_CUDA(cudaMemcpyAsync(dB.p, B, sizeof(double) * nb * d, cudaMemcpyHostToDevice, st.s));
  }
  FMGP_CUDA(fmgp::cov_matrix_launch(dA.p, na, B ? dB.p : nullptr, nb, d, kp, dK.p, st.s));
  FMGP_CUDA(cudaMemcpyAsync(K_out, dK.p, sizeof(double) * na * nb, cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaStreamSynchronize(st.s));
  return FMGP_OK;
}

int fmgp_kernel_values(const double* dist, int64_t ndist, const fmgp_kernel_params* params, double* out) {
  fmgp::KParams kp;
  int rc;
  if ((rc = make_kparams(params, &kp)) != FMGP_OK) return rc;
  for (int64_t i = 0; i < ndist; ++i)
    if (!(std::isfinite(dist[i]) && dist[i] >= 0.0))
      return fail(FMGP_EINVAL, "kernel distance must be finite and non-negative");
  if ((rc = require_device()) != FMGP_OK) return rc;
  if (ndist <= 0) return FMGP_OK;
  Stream st;
  FMGP_CUDA(st.create());
  DevBuf<double> dD, dO;
  FMGP_CUDA(dD.alloc(static_cast<size_t>(ndist), st.s));
  FMGP_CUDA(dO.alloc(static_cast<size_t>(ndist), st.s));
  FMGP_CUDA(cudaMemcpyAsync(dD.p, dist, sizeof(double) * ndist, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(fmgp::kernel_values_launch(dD.p, ndist, kp, dO.p, st.s));
  FMGP_CUDA(cudaMemcpyAsync(out, dO.p, sizeof(double) * ndist, cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaStreamSynchronize(st.s));
  return FMGP_OK;
}

int fmgp_solve_spd_batched(const double* K, const double* B, int64_t batch, int32_t k, int32_t m, double* X_out,
                           double* applied_jitter, int64_t* failed_index) {
  if (failed_index) *failed_index = -1;
  int rc;
  if (k < 1 || m < 1) return fail(FMGP_EINVAL, "solve_spd: empty system");
  if ((rc = check_solve_shape(k, 1, m)) != FMGP_OK) return rc;
  if ((rc = require_device()) != FMGP_OK) return rc;
  if (batch <= 0) return FMGP_OK;
  Stream st;
  FMGP_CUDA(st.create());
  DevBuf<double> dK, dB, dJ;
  DevBuf<unsigned long long> fmin;
  FMGP_CUDA(dK.alloc(static_cast<size_t>(batch) * k * k, st.s));
  FMGP_CUDA(dB.alloc(static_cast<size_t>(batch) * k * m, st.s));
  FMGP_CUDA(dJ.alloc(static_cast<size_t>(batch), st.s));
  FMGP_CUDA(fmin.alloc(1, st.s));
  FMGP_CUDA(cudaMemsetAsync(fmin.p, 0xFF, sizeof(unsigned long long), st.s));
  FMGP_CUDA(cudaMemcpyAsync(dK.p, K, sizeof(double) * batch * k * k, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dB.p, B, sizeof(double) * batch * k * m, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(fmgp::spd_solve_batched(dK.p, dB.p, batch, k, m, dB.p, dJ.p, fmin.p, num_sms_current(), st.s));
  unsigned long long host_min = ~0ull;
  FMGP_CUDA(cudaMemcpyAsync(&host_min, fmin.p, sizeof(host_min), cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaMemcpyAsync(X_out, dB.p, sizeof(double) * batch * k * m, cudaMemcpyDeviceToHost, st.s));
  if (applied_jitter)
    FMGP_CUDA(cudaMemcpyAsync(applied_jitter, dJ.p, sizeof(double) * batch, cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaStreamSynchronize(st.s));
  if (host_min != ~0ull) {
    if (failed_index) *failed_index = static_cast<int64_t>(host_min);
    return fail(FMGP_ENUMERIC, "Cholesky factorization failed after jitter escalation up to 1e-6 (matrix " +
                                   std::to_string(host_min) + ")");
  }
  return FMGP_OK;
}

int fmgp_debug_tc_tile(const double* Q, int64_t nq, const double* P, int64_t np, int32_t d, float* G_out) {
  int rc;
  if ((rc = check_points(P, np, d)) != FMGP_OK) return rc;
  if (d < 4) return fail(FMGP_EINVAL, "debug tc tile needs d >= 4");
  if ((rc = require_device()) != FMGP_OK) return rc;
  Stream st;
  FMGP_CUDA(st.create());
  DevBuf<double> dQ, dP;
  DevBuf<float> dG;
  DevBuf<int32_t> dO;
  FMGP_CUDA(dQ.alloc(static_cast<size_t>(nq) * d, st.s));
  FMGP_CUDA(dP.alloc(static_cast<size_t>(np) * d, st.s));
  FMGP_CUDA(dG.alloc(128 * 256, st.s));
  FMGP_CUDA(dO.alloc(static_cast<size_t>(nq), st.s));
  FMGP_CUDA(cudaMemsetAsync(dG.p, 0, sizeof(float) * 128 * 256, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dQ.p, Q, sizeof(double) * nq * d, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(cudaMemcpyAsync(dP.p, P, sizeof(double) * np * d, cudaMemcpyHostToDevice, st.s));
  FMGP_CUDA(fmgp::knn_tc(dQ.p, nq, dP.p, np, d, 1, -1, nullptr, 0, dO.p, nullptr, num_sms_current(), st.s, dG.p));
  FMGP_CUDA(cudaMemcpyAsync(G_out, dG.p, sizeof(float) * 128 * 256, cudaMemcpyDeviceToHost, st.s));
  FMGP_CUDA(cudaStreamSynchronize(st.s));
  return FMGP_OK;
}

}  // extern "C"
