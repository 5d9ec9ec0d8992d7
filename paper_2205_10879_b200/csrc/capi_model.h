// The model handle of the C ABI (fmgp_model, include/fmgp_b200.h), shared by
// capi.cu (single-device create/predict) and group.cu (multi-GPU precompute
// whose device results become the handle's replicas without a host trip).
//
// A handle holds one device-resident replica of the reference's
// PrecomputedModel (fast_predict.hpp:25-33: X, the neighbour table S, the
// coefficients C, kernel, mean offsets) per device it spans, plus the
// predict-walk cell grid of X (d <= 3) that stands in for the model's own
// NeighborIndex (fast_predict.cpp:127-129). Predict splits the test points
// contiguously over the replicas; every point's arithmetic is the same on any
// replica, so the result does not depend on the replica count.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "fmgp_common.cuh"

struct fmgp_model_replica {
  int device = 0;
  bool owns = true;  // false: X/S/C wrap caller-owned device buffers (fmgp_model_wrap_device)
  double* X = nullptr;
  int32_t* S = nullptr;
  double* C = nullptr;
  double* mo = nullptr;  // m mean offsets (always owned)
  void* grid = nullptr;  // predict-walk grid of X (d <= 3), always owned
};

struct fmgp_model {
  int64_t n = 0;
  int32_t d = 0, k = 0, m = 0;
  fmgp::KParams kp{};
  std::vector<fmgp_model_replica> reps;
};

// The device-resident point set of NeighborIndex (fmgp_index_create): a
// row-major device copy of the points; the ApproxGraph index (graph.cu)
// searches over it.
struct fmgp_index {
  int device = 0;
  int64_t n = 0;
  int32_t d = 0;
  double* P = nullptr;
  void* grid = nullptr;  // nearest-point walk grid of P (d <= 3), built once at create
};

namespace fmgp_capi {

// Finish a replica whose X/S/C are set on the current device: mean offsets
// (host array of m) and the predict grid. Synchronous.
cudaError_t replica_finish(fmgp_model_replica& r, int64_t n, int32_t d, int32_t k, int32_t m, const double* mean_offset_host);
void replica_release(fmgp_model_replica& r);

}  // namespace fmgp_capi
