/* fmgp_b200.h — the drop-in boundary: a C ABI over the B200 (sm_100a)
 * implementation of the FastMuyGPs posterior-mean path.
 *
 * The reference exposes this path only as a C++ API in namespace fastmuygps
 * (paths relative to /root/reference/proj):
 *   precompute            core/include/fastmuygps/fast_predict.hpp:38-41
 *   fast_predict_one      core/include/fastmuygps/fast_predict.hpp:45-46
 *   fast_predict_batch    core/include/fastmuygps/fast_predict.hpp:48-49
 *   NeighborIndex (Exact) core/include/fastmuygps/nn_index.hpp:34-51
 *   kernel_value / cov_matrix / cov_matrix_self  core/include/fastmuygps/kernel.hpp:39-55
 *   cholesky_with_jitter / solve_spd             core/include/fastmuygps/linalg.hpp:13-20
 * The C++ facade in paper_2205_10879_b200/cpp re-exports those exact headers
 * and calls the functions below; any other FFI (ctypes, cgo, JNI) binds them
 * directly — see INTEGRATION.md.
 *
 * Conventions
 *  - Plain pointers and sizes only. Matrices are ROW-MAJOR: X n*d, Y n*m,
 *    Z nz*d, S n*k int32 (the reference's NeighborTable layout,
 *    fast_predict.hpp:15-18), C n*k*m f64 (m = 1 is the reference's
 *    RowMajor n*k table, fast_predict.hpp:27).
 *  - Functions without `_device` take HOST buffers owned by the caller and
 *    do every host<->device copy internally (synchronous on return).
 *    Functions with `_device` take DEVICE pointers on the current CUDA device
 *    and a cudaStream_t passed as void*; they are stream-ordered and return
 *    after enqueueing, except where a status must be read back (noted).
 *  - No exceptions cross the ABI. Return codes map to the reference's
 *    exceptions (the facade re-throws them with the reference's messages):
 *      FMGP_OK        0
 *      FMGP_EINVAL    1  std::domain_error   (argument/precondition errors)
 *      FMGP_ENUMERIC  2  fastmuygps::NumericError (jitter ladder exhausted,
 *                        linalg.cpp:28-30; *failed_row = lowest failing row,
 *                        matching the reference run with threads = 1)
 *      FMGP_ECUDA     3  CUDA error or no usable device (never a CPU fallback)
 *    fmgp_last_error() returns the calling thread's last message.
 *  - Results do not depend on how rows are sharded (row_begin/row_end) or on
 *    the number of GPUs: every row is computed by the same arithmetic.
 */
#ifndef FMGP_B200_H
#define FMGP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMGP_ABI_VERSION 2

enum fmgp_status { FMGP_OK = 0, FMGP_EINVAL = 1, FMGP_ENUMERIC = 2, FMGP_ECUDA = 3 };

/* KernelKind (kernel.hpp:7); the numeric values are the model-file tag
 * (fast_predict.cpp:179). */
enum fmgp_kernel_kind { FMGP_MATERN = 0, FMGP_RBF = 1 };

/* KernelParams (kernel.hpp:12-33) + KernelKind. Validated like the
 * reference constructor (kernel.cpp:13-28): sigma, rho, nu > 0 and finite,
 * tau >= 0 and finite. The device path evaluates Matern for nu in
 * {0.5, 1.5, 2.5} (the closed forms of kernel.cpp:63-71) and RBF for any nu. */
typedef struct fmgp_kernel_params {
  int32_t kind;
  double sigma;
  double rho;
  double nu;
  double tau;
} fmgp_kernel_params;

int fmgp_abi_version(void);
const char* fmgp_last_error(void);
/* Diagnostics: number of CUDA kernels this library has launched (process-wide). */
int64_t fmgp_launch_count(void);
/* Number of visible CUDA devices (0 when none: every compute call then
 * returns FMGP_ECUDA). */
int fmgp_device_count(void);

/* KernelParams constructor checks (kernel.cpp:13-28) plus the device path's
 * nu support. */
int fmgp_validate_kernel(const fmgp_kernel_params* p);

/* ---- precompute (fast_predict.cpp:70-130) ---------------------------------
 * S_out[i,0] = i; S_out[i,1..k-1] = the k-1 nearest training points of x_i,
 * excluding i by index, ascending by (dist_sq, index) — bit-exact with the
 * reference's Exact NeighborIndex. C_out[i] = K(X_S_i, X_S_i)^-1 Y_S_i with
 * the nugget/jitter conventions of kernel.cpp:58-60 and linalg.cpp:10-31.
 * Errors: k not in [1, n] or n < 1 or d < 1 or m < 1 or non-finite X
 * (fast_predict.cpp:74-76, nn_index.cpp:56-62) -> FMGP_EINVAL.
 * Multi-GPU in one process (the reference's `threads` knob):
 * with FMGP_DEVICES="0,1,..." the rows are split contiguously over the listed
 * devices (one host thread each); S and C are identical for any device list
 * and a numeric failure names the lowest failing row over all shards. */
int fmgp_precompute(const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                    const fmgp_kernel_params* params, int32_t k, int32_t* S_out, double* C_out,
                    int64_t* failed_row);

/* Row shard [row_begin, row_end) of precompute with HOST buffers (one process
 * per GPU: each rank passes the full X, Y and receives its rows of S and C;
 * same semantics and failure rule as fmgp_precompute, row ids global). */
int fmgp_precompute_rows(const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                         const fmgp_kernel_params* params, int32_t k, int64_t row_begin, int64_t row_end,
                         int32_t* S_out, double* C_out, int64_t* failed_row);

/* The neighbour stage (K1) alone, device pointers: precompute's S rows
 * [row_begin, row_end) (S[i][0] = i, then the k-1 nearest, self excluded by
 * index), stream-ordered, no synchronisation. */
int fmgp_knn_rows_device(const double* X, int64_t n, int32_t d, int32_t k, int64_t row_begin, int64_t row_end,
                         int32_t* S_out, void* stream);

/* The fused solve (K2) alone, device pointers: rows [row_begin, row_begin +
 * nrows) of C from their given neighbour rows S_rows (nrows x k, S[i][0] = i
 * as precompute produces them). With fmgp_query_knn_device this lets a caller
 * run K1 once for a shard and K2 in chunks (e.g. to overlap a collective with
 * the next chunk). fail_dev == NULL: synchronises `stream` and reports a
 * failure as FMGP_ENUMERIC (*failed_row = lowest failing row); otherwise fully
 * asynchronous: the lowest failing row is min-combined into the device word
 * *fail_dev (initialise it to UINT64_MAX; it stays so when every row succeeds). */
int fmgp_solve_rows_device(const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                           const fmgp_kernel_params* params, int32_t k, const int32_t* S_rows, int64_t nrows,
                           int64_t row_begin, double* C_out, uint64_t* fail_dev, int64_t* failed_row,
                           void* stream);

/* Row shard [row_begin, row_end) of precompute with everything in HBM:
 * X (n*d) and Y (n*m) are the full, replicated training set; S_out and C_out
 * hold (row_end-row_begin) rows. Reads back one status word, so it returns
 * after the shard is finished. X is not re-validated here. */
int fmgp_precompute_device(const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                           const fmgp_kernel_params* params, int32_t k, int64_t row_begin,
                           int64_t row_end, int32_t* S_out, double* C_out, int64_t* failed_row,
                           void* stream);

/* ---- neighbour search (nn_index.cpp:254-287, :351-366) --------------------
 * For each of nq queries, the k nearest of the np points by (dist_sq, index);
 * exclude (nullable, nq entries) removes one point index per query (-1: none),
 * by index identity (nn_index.cpp:268). idx_out nq*k; dist_out (nullable)
 * nq*k receives sqrt(dist_sq) like NeighborList::distances (:337-340).
 * Errors: k < 1 or k > np - (exclude >= 0) -> FMGP_EINVAL (:260-263). */
int fmgp_query_knn(const double* P, int64_t np, int32_t d, const double* Q, int64_t nq, int32_t k,
                   const int32_t* exclude, int32_t* idx_out, double* dist_out);
int fmgp_query_knn_device(const double* P, int64_t np, int32_t d, const double* Q, int64_t nq,
                          int32_t k, int64_t self_offset, int32_t* idx_out, double* dist_sq_out,
                          void* stream);
/* nearest_training_point for nq queries: ties go to the lower index. */
int fmgp_nearest(const double* P, int64_t np, int32_t d, const double* Q, int64_t nq, int32_t* idx_out);
int fmgp_nearest_device(const double* P, int64_t np, int32_t d, const double* Q, int64_t nq,
                        int32_t* idx_out, void* stream);

/* ---- NeighborIndex handle (nn_index.hpp:33-60, Exact mode) ---------------
 * A device-resident copy of the points; queries upload only the query
 * points. Immutable; safe for concurrent queries (nn_index.hpp:28-31).
 * fmgp_index_distances: distance_to (nn_index.cpp:344-349) of one query q
 * to cnt stored points idx[], i.e. sqrt(dist_sq); idx out of range ->
 * FMGP_EINVAL ("distance_to: bad query or index"). */
typedef struct fmgp_index fmgp_index;
/* device < 0: the calling thread's current device (also for fmgp_model_create).
 * Entry points that switch devices restore the caller's current device. */
int fmgp_index_create(const double* P, int64_t np, int32_t d, int32_t device, fmgp_index** out);
int fmgp_index_query_knn(const fmgp_index* index, const double* Q, int64_t nq, int32_t k,
                         const int32_t* exclude, int32_t* idx_out, double* dist_out);
int fmgp_index_nearest(const fmgp_index* index, const double* Q, int64_t nq, int32_t* idx_out);
int fmgp_index_distances(const fmgp_index* index, const double* q, const int32_t* idx, int64_t cnt,
                         double* out);
void fmgp_index_destroy(fmgp_index* index);

/* ---- ApproxGraph index (IndexMode::ApproxGraph; nn_index.cpp:83-237, :288-341,
 * :351-366, :397-470) ------------------------------------------------------
 * A navigable-small-world graph over an index's points (the index must
 * outlive it). fmgp_graph_build: levels from the reference's seeded
 * generator (splitmix64 of seed ^ 0xa02bdbf7bb3c0a7, floor(-ln u / ln M)),
 * so layer sizes, maximum level and entry point are the reference's; each
 * layer links every node to its 2M (layer 0) / M (above) exact nearest
 * neighbours among the layer's nodes (one batched exact search per layer, in
 * place of the reference's sequential insertion; build_beam is recorded).
 * fmgp_graph_load: a serialized graph (the reference's blob after its mode
 * tag, parsed by the caller: levels[n]; counts[] node-major, layer 0 first;
 * ids[] concatenated). fmgp_graph_info / fmgp_graph_export give the same
 * arrays back for serialize(). Queries run the reference's search (greedy
 * descent on the upper layers, best-first beam search on layer 0 with beam
 * query_beam or max(64, 2k), nearest: query_beam or 64) one warp per query,
 * with the exact scan for any query that returns fewer than k results;
 * dist_evals (nullable) accumulates the distance evaluations, as the
 * reference's counter does. */
typedef struct fmgp_graph fmgp_graph;
int fmgp_graph_build(const fmgp_index* index, int32_t max_degree, int32_t build_beam, int32_t query_beam,
                     uint64_t seed, fmgp_graph** out);
int fmgp_graph_load(const fmgp_index* index, int32_t max_degree, int32_t build_beam, int32_t query_beam,
                    uint64_t seed, int32_t entry, int32_t max_level, const int32_t* levels,
                    const uint32_t* counts, const int32_t* ids, fmgp_graph** out);
int fmgp_graph_info(const fmgp_graph* graph, int32_t* entry, int32_t* max_level, int64_t* counts_total,
                    int64_t* ids_total);
int fmgp_graph_export(const fmgp_graph* graph, int32_t* levels, uint32_t* counts, int32_t* ids);
int fmgp_graph_query_knn(const fmgp_graph* graph, const double* Q, int64_t nq, int32_t k,
                         const int32_t* exclude, int32_t* idx_out, double* dist_out, uint64_t* dist_evals);
int fmgp_graph_nearest(const fmgp_graph* graph, const double* Q, int64_t nq, int32_t* idx_out,
                       uint64_t* dist_evals);
void fmgp_graph_destroy(fmgp_graph* graph);

/* ---- predict (fast_predict.cpp:132-156) -----------------------------------
 * out[t*m + c] = sum_s kernel(||z_t - x_{S[j,s]}||) C[j,s,c] + mean_offset[c],
 * j = nearest training point of z_t (nn_out, nullable, receives j). */
int fmgp_predict(const double* X, const int32_t* S, const double* C, int64_t n, int32_t d, int32_t k,
                 int32_t m, const fmgp_kernel_params* params, const double* mean_offset, const double* Z,
                 int64_t nz, double* out, int32_t* nn_out);
/* Same with X, S, C, Z, out, nn_out in HBM; mean_offset is a host array of m. */
int fmgp_predict_device(const double* X, const int32_t* S, const double* C, int64_t n, int32_t d,
                        int32_t k, int32_t m, const fmgp_kernel_params* params, const double* mean_offset,
                        const double* Z, int64_t nz, double* out, int32_t* nn_out, void* stream);

/* ---- PrecomputedModel handle (fast_predict.hpp:25-33) ---------------------
 * Device-resident, immutable copy of X, S, C, kernel and mean offsets on
 * `device`. fmgp_model_predict is safe to call concurrently from several host
 * threads on one handle (fast_predict.hpp:20-24). */
typedef struct fmgp_model fmgp_model;
int fmgp_model_create(const double* X, const int32_t* S, const double* C, int64_t n, int32_t d,
                      int32_t k, int32_t m, const fmgp_kernel_params* params, const double* mean_offset,
                      int32_t device, fmgp_model** out);
int fmgp_model_predict(const fmgp_model* model, const double* Z, int64_t nz, double* out,
                       int32_t* nn_out);
void fmgp_model_destroy(fmgp_model* model);
/* A model over caller-owned DEVICE buffers X (n*d), S (n*k), C (n*k*m) on the
 * current device (not copied; they must outlive the handle); mean_offset is a
 * host array of m. Builds the predict-walk grid once. */
int fmgp_model_wrap_device(const double* X, const int32_t* S, const double* C, int64_t n, int32_t d, int32_t k,
                           int32_t m, const fmgp_kernel_params* params, const double* mean_offset, fmgp_model** out);
/* Stream-ordered predict with Z, out, nn_out (nullable) in HBM on the current
 * device, through the handle's replica on that device and its cached grid. */
int fmgp_model_predict_device(const fmgp_model* model, const double* Z, int64_t nz, double* out, int32_t* nn_out,
                              void* stream);
/* Number of device replicas (1, or the members of the group that built it). */
int fmgp_model_replicas(const fmgp_model* model);

/* ---- device groups: multi-GPU precompute (the reference's
 * thread split, fast_predict.cpp:110-125) ------------------------------------
 * The training set is replicated on every member GPU; training rows are dealt
 * block-cyclically (fmgp_group_rows lists a member's [begin, end) blocks); S
 * and C are all-gathered in place over NVLink (NCCL, loaded at run time), each
 * round's exchange overlapped with the next round's solve. Results are
 * bit-identical to fmgp_precompute for any group.
 *  - rank group: one process per GPU. Rank 0 calls fmgp_group_unique_id and
 *    the caller distributes the 128 bytes (e.g. torch.distributed); every
 *    rank then calls fmgp_group_create_rank (collective).
 *  - device group: one process, several devices, one host thread each; NCCL
 *    when the devices are distinct, peer copies otherwise (a device may be
 *    listed twice to exercise the layout on one GPU). */
typedef struct fmgp_group fmgp_group;
int fmgp_group_unique_id(uint8_t* id_out /* 128 bytes */);
int fmgp_group_create_rank(const uint8_t* id, int32_t nranks, int32_t rank, int32_t device, fmgp_group** out);
int fmgp_group_create_devices(const int32_t* devices, int32_t ndev, fmgp_group** out);
/* backend: 0 none (one member), 1 NCCL, 2 peer copies */
int fmgp_group_info(const fmgp_group* group, int32_t* nranks, int32_t* local_members, int32_t* backend);
/* The row layout (no device needed): member `member` of `nranks` owns
 * *nblocks blocks, ranges[2*b], ranges[2*b+1] = [begin, end) (nullable).
 * Blocks of pc = ceil(n / (nranks * R)) rows, R = FMGP_GROUP_CHUNKS (4). */
int fmgp_group_rows(int64_t n, int32_t nranks, int32_t member, int64_t* nblocks, int64_t* ranges);
void fmgp_group_destroy(fmgp_group* group);
/* Host buffers: X (n*d), Y (n*m) in; S_out (n*k) and C_out (n*k*m) receive
 * the rows this process's members computed (every row for a device group,
 * the rank's blocks for a rank group). model_out (nullable; needs
 * mean_offset, m values): a model whose replicas are the members' full,
 * all-gathered device results (no copy). Collective over the group. */
int fmgp_group_precompute(fmgp_group* group, const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                          const fmgp_kernel_params* params, int32_t k, const double* mean_offset, int32_t* S_out,
                          double* C_out, int64_t* failed_row, fmgp_model** model_out);
/* Rank groups: X, Y full replicas in HBM; S_out (n*k) and C_out (n*k*m) are
 * full-size device buffers that end holding every row on every rank. Work is
 * issued on `stream`; returns after the failure word is read back. */
int fmgp_group_precompute_device(fmgp_group* group, const double* X, const double* Y, int64_t n, int32_t d,
                                 int32_t m, const fmgp_kernel_params* params, int32_t k, int32_t* S_out,
                                 double* C_out, int64_t* failed_row, void* stream);

/* ---- kernel arithmetic on device (kernel.cpp:88-119) ----------------------
 * K_out (na*nb row-major) = kernel(||A_i - B_j||); with B == NULL computes
 * cov_matrix_self(A) (exact symmetric fill, diagonal kernel(0)). */
int fmgp_cov_matrix(const double* A, int64_t na, const double* B, int64_t nb, int32_t d,
                    const fmgp_kernel_params* params, double* K_out);
/* kernel_value at ndist distances (check_distance, kernel.cpp:32-36:
 * negative or non-finite -> FMGP_EINVAL). */
int fmgp_kernel_values(const double* dist, int64_t ndist, const fmgp_kernel_params* params, double* out);

/* ---- batched SPD solve (linalg.cpp:10-36) ---------------------------------
 * For each of `batch` symmetric k*k matrices K (row-major, lower triangle
 * used), solve K X = B (B: k*m row-major) under the jitter ladder
 * {0, 1e-10, 1e-8, 1e-6}. X_out may alias B. applied_jitter (nullable,
 * batch) receives the rung that succeeded. On failure returns FMGP_ENUMERIC
 * with *failed_index = the lowest failing matrix. */
int fmgp_solve_spd_batched(const double* K, const double* B, int64_t batch, int32_t k, int32_t m,
                           double* X_out, double* applied_jitter, int64_t* failed_index);

/* ---- MuyGPs training and the localized baseline ---------
 * muygps.cpp:32-62 local_prediction for b batch entries at once: entry t
 * predicts Y[batch_idx[t]] from its neighbour list nbr[t*k .. t*k+k) (the
 * caller's NeighborList indices, which must not contain batch_idx[t]) and
 * the list's distances dist[t*k ..] (cross-covariance = kernel(distance), as
 * the reference uses NeighborList.distances):
 *   preds_out[t] = cross_t . K(X[nbr_t])^{-1} Y[nbr_t]   (Y: n values)
 * One fused gather -> K -> jitter-ladder Cholesky -> solve per entry, then a
 * cross-covariance dot. FMGP_ENUMERIC: *failed_entry = the lowest failing t
 * (the first entry the reference's sequential loop would throw on).
 * Replaces local_prediction (muygps.hpp:50-52, muygps.cpp:32-62). */
int fmgp_local_predictions(const double* X, const double* Y, int64_t n, int32_t d, const int32_t* batch_idx,
                           const int32_t* nbr, const double* dist, int64_t b, int32_t k,
                           const fmgp_kernel_params* params, double* preds_out, int64_t* failed_entry);

/* Device-resident leave-one-out session for the optimizer loop (muygps.cpp:
 * 64-78 loocv_loss, evaluated up to max_evals times by train): X, Y, the
 * batch, its neighbour lists and distances are uploaded once; each
 * evaluation uploads the kernel parameters only and reads back b
 * predictions. loss_out = sum_t (Y[i_t] - pred_t)^2 / b accumulated on the
 * host in batch order (the reference's bit-stable order). preds_out
 * (nullable, b). */
typedef struct fmgp_loocv fmgp_loocv;
int fmgp_loocv_create(const double* X, const double* Y, int64_t n, int32_t d, const int32_t* batch_idx,
                      const int32_t* nbr, const double* dist, int64_t b, int32_t k, fmgp_loocv** out);
int fmgp_loocv_eval(fmgp_loocv* session, const fmgp_kernel_params* params, double* loss_out, double* preds_out,
                    int64_t* failed_entry);
void fmgp_loocv_destroy(fmgp_loocv* session);

/* train (muygps.cpp:214-270): neighbour lists of the batch (k exact
 * neighbours, self excluded) computed once on the device, then a bounded
 * Nelder-Mead over log10(rho), nu, tau (each free when its has_* flag is
 * set) minimising the device LOOCV loss; never returns a loss above the
 * initial one. kind is fixed. Outputs the fitted parameters (theta_out),
 * the final loss, the number of loss evaluations and whether the initial
 * guess was improved. Errors: FMGP_EINVAL with the reference's messages
 * ("train: k must be at least 2", "train: invalid bounds", ...),
 * FMGP_ENUMERIC when a local solve fails ("local_prediction at index i"). */
typedef struct {
  int32_t k;
  int32_t kind;
  int32_t has_rho, has_nu, has_tau;
  double rho_lo, rho_hi, nu_lo, nu_hi, tau_lo, tau_hi;
  int32_t max_evals;
  double tol;
} fmgp_train_config;
int fmgp_train(const double* X, const double* Y, int64_t n, int32_t d, const int32_t* batch_idx, int64_t b,
               const fmgp_kernel_params* initial, const fmgp_train_config* config, fmgp_kernel_params* theta_out,
               double* final_loss, int32_t* evaluations, int32_t* improved);

/* muygps_predict (muygps.cpp:272-295), the localized baseline predictor:
 * each test point's own k exact neighbours (device kNN), one k x k solve,
 * cross-covariance dot, + mean_offset. FMGP_ENUMERIC names the lowest
 * failing test row in *failed_row ("muygps_predict" context). */
int fmgp_muygps_predict(const double* X, const double* Y, int64_t n, int32_t d, const double* Z, int64_t nz,
                        int32_t k, const fmgp_kernel_params* params, double mean_offset, double* out,
                        int64_t* failed_row);

/* ---- diagnostics ---------------------------------------------------------
 * Stage timing for benchmarks: while enabled, every precompute call records
 * CUDA events on its launch stream around the kNN stage (K1) and the fused
 * solve (K2); fmgp_stage_times synchronises those events and returns the
 * summed kernel-stage times (ms) and the number of calls since the last read. */
void fmgp_set_stage_timing(int on);
int fmgp_stage_times(double* knn_ms, double* solve_ms, int64_t* calls);

/* FP64 roofline denominators measured on the current device now: DFMA and
 * DMMA (m8n8k4) TFLOP/s over the whole chip (best of three ~1 ms runs). */
int fmgp_diag_fp64_peak(double* dfma_tflops, double* dmma_tflops);

/* ---- diagnostics (tensor-core kNN) ----------------------------------------
 * D~ (the tensor-core filter value n^_q + n^_p - 2 q^.p^ in the scaled fp16
 * space) of the first 128 x 256 (query, point) tile of the tcgen05 kNN, for
 * validating the GEMM plumbing. G_out: 128 x 256 fp32 (host). d >= 4. */
int fmgp_debug_tc_tile(const double* Q, int64_t nq, const double* P, int64_t np, int32_t d, float* G_out);

#ifdef __cplusplus
}
#endif
#endif /* FMGP_B200_H */
