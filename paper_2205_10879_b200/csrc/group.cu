// Multi-GPU precompute and model replicas through the C ABI (
// include/fmgp_b200.h "device groups"). The reference's analogue is the
// thread split of precompute (fast_predict.cpp:110-125): contiguous row
// chunks, one worker each, bit-stable results. Here a group member is one
// GPU; the training set is replicated on every member, the training rows
// (the kNN / solve queries) are dealt block-cyclically, and the neighbour
// table S and coefficient tensor C are all-gathered over NVLink so every
// member ends with the whole model, ready to predict its share of test points.
//
// Row layout: blocks of pc rows dealt round-robin, round c = rows
// [c*G*pc, (c+1)*G*pc): member r owns block c*G + r of every round. A round's
// blocks are contiguous in S and C, so its exchange is ONE in-place all-gather
// (ncclAllGather, sendbuff = recvbuff + r*count) with no staging copy, and
// round c's exchange runs on a side stream while round c+1 is solved. A short
// last round (n not a multiple of G*pc) is exchanged by grouped in-place
// broadcasts (one per member, its block's size).
//
// Two kinds of group:
//  * rank groups (one process per GPU, fmgp_group_create_rank): NCCL
//    communicator from a unique id the caller distributes;
//  * device groups (one process, several GPUs, fmgp_group_create_devices):
//    one host thread per member; NCCL (ncclCommInitAll) when the devices are
//    distinct, otherwise (a device listed twice, e.g. "0,0" to test the layout
//    on one GPU) peer copies (cudaMemcpyPeerAsync) push each block to the
//    other members.
// NCCL is loaded at run time (dlopen "libnccl.so.2": the process's copy when
// one is already loaded, e.g. torch's, else FMGP_NCCL_LIB, else the system's), so the library has
// no link-time NCCL dependency and single-GPU use never touches it.
//
// Every row's arithmetic is the single-GPU kernels' (knn_grid / knn_tc / fp64
// brute force, then the fused solve), so S and C are bit-identical for any
// group size; a numeric failure reports the lowest failing row over all
// members (a MIN all-reduce of the device failure word).
#include <dlfcn.h>
#include <nccl.h>  // types only; the symbols are resolved with dlsym

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/fmgp_b200.h"
#include "capi_common.h"
#include "capi_model.h"
#include "fmgp_common.cuh"
#include "fmgp_internal.h"

using namespace fmgp_capi;

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // the process's copy if one is loaded; else FMGP_NCCL_LIB (the Python binding points it at the
    // NCCL wheel torch was built against, so a later `import torch` in the same process does not find
    // an older system libnccl under the same SONAME); else the system's
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (h == nullptr) {
      const char* pth = std::getenv("FMGP_NCCL_LIB");
      if (pth != nullptr && pth[0] != 0) h = dlopen(pth, RTLD_NOW | RTLD_LOCAL);
    }
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (h == nullptr) {
      const char* e = dlerror();
      a.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return a;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (fn == nullptr) {
        all = false;
        a.why = std::string("libnccl.so.2 lacks ") + name;
      }
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommInitAll, "ncclCommInitAll");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllGather, "ncclAllGather");
    sym(a.Broadcast, "ncclBroadcast");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    a.ok = all;
    return a;
  }();
  return api;
}

int nccl_fail(ncclResult_t r, const char* where) {
  const char* s = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
  return fail(FMGP_ECUDA, std::string(where) + ": NCCL error " + std::to_string(static_cast<int>(r)) + " (" + s + ")");
}

#define FMGP_NCCL(call)                                  \
  do {                                                   \
    ncclResult_t fmgp_r_ = (call);                       \
    if (fmgp_r_ != ncclSuccess) return nccl_fail(fmgp_r_, #call); \
  } while (0)

enum Backend { kNone = 0, kNccl = 1, kPeer = 2 };

// Reusable host barrier for the member threads of a device group.
class Barrier {
 public:
  explicit Barrier(int n) : n_(n) {}
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    const int gen = gen_;
    if (++count_ == n_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
    } else {
      cv_.wait(lk, [&] { return gen != gen_; });
    }
  }

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  int n_, count_ = 0, gen_ = 0;
};

// Block-cyclic row layout over G members with blocks of pc rows.
struct Cyclic {
  int64_t n = 0, pc = 1;
  int g = 1;
  int64_t rounds() const { return (n + g * pc - 1) / (g * pc); }
  void block(int64_t c, int r, int64_t& b, int64_t& e) const {
    b = std::min<int64_t>(n, (c * g + r) * pc);
    e = std::min<int64_t>(n, b + pc);
  }
  bool full_round(int64_t c) const { return (c + 1) * g * pc <= n; }
  int64_t rows_of(int r) const {
    int64_t s = 0;
    for (int64_t c = 0; c < rounds(); ++c) {
      int64_t b, e;
      block(c, r, b, e);
      s += e - b;
    }
    return s;
  }
};

Cyclic make_cyclic(int64_t n, int g) {
  // FMGP_GROUP_CHUNKS rounds (default 4): round c's exchange overlaps the
  // solve of round c+1; only the last round's exchange is exposed
  static const int rounds = [] {
    const char* e = std::getenv("FMGP_GROUP_CHUNKS");
    const int v = e != nullptr ? std::atoi(e) : 4;
    return v >= 1 ? v : 4;
  }();
  Cyclic cy;
  cy.n = n;
  cy.g = g;
  const int rd = g == 1 ? 1 : rounds;  // a group of one has nothing to exchange: one round
  cy.pc = std::max<int64_t>(1, (n + static_cast<int64_t>(g) * rd - 1) / (static_cast<int64_t>(g) * rd));
  return cy;
}

}  // namespace

struct fmgp_group_member {
  int device = 0;
  int rank = 0;
  ncclComm_t comm = nullptr;
};

struct fmgp_group {
  int nranks = 1;
  int backend = kNone;
  bool single_process = true;
  std::vector<fmgp_group_member> local;
  std::mutex mu;  // one collective call at a time per group
};

namespace {

// Shared state of one group call: every member's full-size device buffers
// (the peer backend pushes into the other members' buffers).
struct CallCtx {
  fmgp_group* g = nullptr;
  Cyclic cy;
  std::vector<int32_t*> S;
  std::vector<double*> C;
  Barrier* bar = nullptr;
};

// Round c's blocks of `base` (rows of `row_bytes`) from every member to every
// member, stream-ordered on `side` of member `mi`.
int exchange_round(CallCtx& cx, int mi, char* const* bases, size_t row_bytes, int64_t c, cudaStream_t side) {
  fmgp_group& g = *cx.g;
  const fmgp_group_member& mb = g.local[mi];
  const Cyclic& cy = cx.cy;
  char* base = bases[mi];
  if (g.backend == kNone) return FMGP_OK;
  if (g.backend == kNccl) {
    NcclApi& api = nccl();
    if (cy.full_round(c)) {
      const size_t cnt = static_cast<size_t>(cy.pc) * row_bytes;
      char* recv = base + static_cast<size_t>(c * cy.g * cy.pc) * row_bytes;
      FMGP_NCCL(api.AllGather(recv + static_cast<size_t>(mb.rank) * cnt, recv, cnt, ncclUint8, mb.comm, side));
    } else {
      FMGP_NCCL(api.GroupStart());
      for (int q = 0; q < cy.g; ++q) {
        int64_t b, e;
        cy.block(c, q, b, e);
        if (e <= b) continue;
        char* p = base + static_cast<size_t>(b) * row_bytes;
        const ncclResult_t r = api.Broadcast(p, p, static_cast<size_t>(e - b) * row_bytes, ncclUint8, q, mb.comm, side);
        if (r != ncclSuccess) {
          api.GroupEnd();
          return nccl_fail(r, "ncclBroadcast");
        }
      }
      FMGP_NCCL(api.GroupEnd());
    }
    return FMGP_OK;
  }
  // peer copies: push this member's block of round c into every other member's buffer
  int64_t b, e;
  cy.block(c, mb.rank, b, e);
  if (e <= b) return FMGP_OK;
  const size_t off = static_cast<size_t>(b) * row_bytes, bytes = static_cast<size_t>(e - b) * row_bytes;
  for (size_t q = 0; q < g.local.size(); ++q) {
    if (static_cast<int>(q) == mi) continue;
    FMGP_CUDA(cudaMemcpyPeerAsync(bases[q] + off, g.local[q].device, base + off, mb.device, bytes, side));
  }
  return FMGP_OK;
}

struct MemberStreams {
  cudaStream_t work = nullptr, side = nullptr, rb = nullptr;
  std::vector<cudaEvent_t> evs;
  cudaError_t handoff(cudaStream_t from, cudaStream_t to) {
    cudaEvent_t e;
    cudaError_t err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (err != cudaSuccess) return err;
    evs.push_back(e);
    err = cudaEventRecord(e, from);
    return err == cudaSuccess ? cudaStreamWaitEvent(to, e, 0) : err;
  }
  ~MemberStreams() {
    for (auto e : evs) cudaEventDestroy(e);
  }
};

// One member's share of a group precompute on its device: K1 for its rows
// (written at their global rows of S), the S exchange on the side stream,
// then per round K2 of its block and that round's C exchange on the side
// stream. With S_host/C_host the member's own blocks are also read back on
// the rb stream as soon as they are computed. The work stream joins the side
// (and rb) streams before returning; fmin (device word) collects failures.
int member_precompute(CallCtx& cx, int mi, const double* X, const double* Y, int64_t n, int d, int m,
                      const fmgp::KParams& kp, int k, MemberStreams& st, unsigned long long* fmin, int32_t* S_host,
                      double* C_host) {
  const Cyclic& cy = cx.cy;
  const int r = cx.g->local[mi].rank;
  int32_t* S = cx.S[mi];
  double* C = cx.C[mi];
  const int sms = num_sms_current();
  const int64_t myrows = cy.rows_of(r);
  cudaEvent_t tev[3] = {};
  const bool timing = stage_timing_on();
  if (timing) {
    for (auto& e : tev) FMGP_CUDA(cudaEventCreate(&e));
    FMGP_CUDA(cudaEventRecord(tev[0], st.work));
  }
  if (k > 1) {
    if (cy.g == 1) {
      // a group of one: the plain search over every row (walks the rows in cell order)
      FMGP_CUDA(fmgp::knn_exact(X, n, X, n, d, k - 1, 0, nullptr, 1, S, nullptr, sms, st.work));
    } else if (myrows > 0 && fmgp::knn_grid_supported(d, k - 1) && std::getenv("FMGP_KNN") == nullptr) {
      FMGP_CUDA(fmgp::knn_grid_rows_cyclic(X, n, d, k - 1, myrows, cy.pc, cy.g, r, S, sms, st.work));
    } else {
      for (int64_t c = 0; c < cy.rounds(); ++c) {
        int64_t b, e;
        cy.block(c, r, b, e);
        if (e > b)
          FMGP_CUDA(fmgp::knn_exact(X + b * d, e - b, X, n, d, k - 1, b, nullptr, 1, S + b * k, nullptr, sms,
                                    st.work));
      }
    }
  } else {
    for (int64_t c = 0; c < cy.rounds(); ++c) {
      int64_t b, e;
      cy.block(c, r, b, e);
      if (e > b) FMGP_CUDA(fmgp::self_rows_launch(S + b * k, e - b, b, st.work));
    }
  }
  if (timing) FMGP_CUDA(cudaEventRecord(tev[1], st.work));
  FMGP_CUDA(st.handoff(st.work, st.side));
  std::vector<char*> sb(cx.S.size()), cb(cx.C.size());
  for (size_t q = 0; q < sb.size(); ++q) {
    sb[q] = reinterpret_cast<char*>(cx.S[q]);
    cb[q] = reinterpret_cast<char*>(cx.C[q]);
  }
  for (int64_t c = 0; c < cy.rounds(); ++c) {
    int rc = exchange_round(cx, mi, sb.data(), sizeof(int32_t) * k, c, st.side);
    if (rc != FMGP_OK) return rc;
  }
  if (S_host != nullptr) {
    FMGP_CUDA(st.handoff(st.work, st.rb));
    for (int64_t c = 0; c < cy.rounds(); ++c) {
      int64_t b, e;
      cy.block(c, r, b, e);
      if (e > b)
        FMGP_CUDA(cudaMemcpyAsync(S_host + b * k, S + b * k, sizeof(int32_t) * (e - b) * k, cudaMemcpyDeviceToHost,
                                  st.rb));
    }
  }
  for (int64_t c = 0; c < cy.rounds(); ++c) {
    int64_t b, e;
    cy.block(c, r, b, e);
    if (e > b)
      FMGP_CUDA(fmgp::fused_solve(X, Y, d, m, S + b * k, e - b, b, k, kp, C + b * k * m, nullptr, fmin, sms,
                                  st.work));
    FMGP_CUDA(st.handoff(st.work, st.side));
    int rc = exchange_round(cx, mi, cb.data(), sizeof(double) * k * m, c, st.side);
    if (rc != FMGP_OK) return rc;
    if (C_host != nullptr && e > b) {
      FMGP_CUDA(st.handoff(st.work, st.rb));
      FMGP_CUDA(cudaMemcpyAsync(C_host + b * k * m, C + b * k * m, sizeof(double) * (e - b) * k * m,
                                cudaMemcpyDeviceToHost, st.rb));
    }
  }
  if (timing) {
    FMGP_CUDA(cudaEventRecord(tev[2], st.work));
    stage_push(tev[0], tev[1], tev[2]);
  }
  // the failure word: lowest failing row over every member
  if (cx.g->backend == kNccl && cx.g->nranks > 1) {
    FMGP_CUDA(st.handoff(st.side, st.work));  // keep the communicator's calls in one stream order
    FMGP_NCCL(nccl().AllReduce(fmin, fmin, 1, ncclUint64, ncclMin, cx.g->local[mi].comm, st.work));
  }
  FMGP_CUDA(st.handoff(st.side, st.work));
  if (S_host != nullptr) FMGP_CUDA(st.handoff(st.rb, st.work));
  return FMGP_OK;
}

int validate(const fmgp_kernel_params* params, int64_t n, int32_t d, int32_t m, int32_t k, fmgp::KParams* kp) {
  int rc;
  if ((rc = make_kparams(params, kp)) != FMGP_OK) return rc;
  if (k < 1 || k > n) return fail(FMGP_EINVAL, "precompute: k out of range");
  if ((rc = check_points(nullptr, n, d)) != FMGP_OK) return rc;
  if (m < 1) return fail(FMGP_EINVAL, "number of outputs m must be >= 1");
  return FMGP_OK;
}

int numeric_fail(unsigned long long row, int64_t* failed_row) {
  if (failed_row) *failed_row = static_cast<int64_t>(row);
  return fail(FMGP_ENUMERIC, "Cholesky factorization failed in precompute row " + std::to_string(row) +
                                 " after jitter escalation up to 1e-6");
}

}  // namespace

extern "C" {

int fmgp_group_unique_id(uint8_t* id_out) {
  if (id_out == nullptr) return fail(FMGP_EINVAL, "unique id buffer is null");
  NcclApi& api = nccl();
  if (!api.ok) return fail(FMGP_ECUDA, api.why);
  ncclUniqueId id;
  FMGP_NCCL(api.GetUniqueId(&id));
  std::memcpy(id_out, id.internal, sizeof(id.internal));
  return FMGP_OK;
}

int fmgp_group_create_rank(const uint8_t* id, int32_t nranks, int32_t rank, int32_t device, fmgp_group** out) {
  if (out == nullptr) return fail(FMGP_EINVAL, "group output pointer is null");
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(FMGP_EINVAL, "group: bad rank or size");
  int rc;
  if ((rc = require_device()) != FMGP_OK) return rc;
  DeviceGuard dg;
  FMGP_CUDA(cudaSetDevice(device));
  auto* g = new fmgp_group();
  g->nranks = nranks;
  g->single_process = false;
  g->local.push_back(fmgp_group_member{device, rank, nullptr});
  if (nranks > 1) {
    if (id == nullptr) {
      delete g;
      return fail(FMGP_EINVAL, "group: a unique id is required for more than one rank");
    }
    NcclApi& api = nccl();
    if (!api.ok) {
      delete g;
      return fail(FMGP_ECUDA, api.why);
    }
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    const ncclResult_t r = api.CommInitRank(&g->local[0].comm, nranks, uid, rank);
    if (r != ncclSuccess) {
      delete g;
      return nccl_fail(r, "ncclCommInitRank");
    }
    g->backend = kNccl;
  }
  *out = g;
  return FMGP_OK;
}

int fmgp_group_create_devices(const int32_t* devices, int32_t ndev, fmgp_group** out) {
  if (out == nullptr) return fail(FMGP_EINVAL, "group output pointer is null");
  *out = nullptr;
  if (devices == nullptr || ndev < 1) return fail(FMGP_EINVAL, "group: empty device list");
  int rc;
  if ((rc = require_device()) != FMGP_OK) return rc;
  int count = 0;
  FMGP_CUDA(cudaGetDeviceCount(&count));
  for (int i = 0; i < ndev; ++i)
    if (devices[i] < 0 || devices[i] >= count) return fail(FMGP_EINVAL, "group: device index out of range");
  auto* g = new fmgp_group();
  g->nranks = ndev;
  g->single_process = true;
  for (int i = 0; i < ndev; ++i) g->local.push_back(fmgp_group_member{devices[i], i, nullptr});
  const char* be_env = std::getenv("FMGP_GROUP_BACKEND");  // "peer" / "nccl": force a backend (tests, A/B)
  if (ndev == 1 && be_env != nullptr && std::string(be_env) == "nccl") {
    // a one-rank NCCL communicator: exercises the NCCL exchange path on one GPU
    if (!nccl().ok) {
      delete g;
      return fail(FMGP_ECUDA, nccl().why);
    }
    DeviceGuard dg;
    const ncclResult_t r = nccl().CommInitAll(&g->local[0].comm, 1, devices);
    if (r != ncclSuccess) {
      delete g;
      return nccl_fail(r, "ncclCommInitAll");
    }
    g->backend = kNccl;
  }
  if (ndev > 1) {
    bool distinct = true;
    for (int i = 0; i < ndev; ++i)
      for (int j = 0; j < i; ++j) distinct &= devices[i] != devices[j];
    const bool want_peer = be_env != nullptr && std::string(be_env) == "peer";
    if (distinct && !want_peer && nccl().ok) {
      std::vector<ncclComm_t> comms(ndev);
      std::vector<int> devs(devices, devices + ndev);
      DeviceGuard dg;
      const ncclResult_t r = nccl().CommInitAll(comms.data(), ndev, devs.data());
      if (r != ncclSuccess) {
        delete g;
        return nccl_fail(r, "ncclCommInitAll");
      }
      for (int i = 0; i < ndev; ++i) g->local[i].comm = comms[i];
      g->backend = kNccl;
    } else {
      DeviceGuard dg;
      for (int i = 0; i < ndev; ++i)  // direct peer access where the topology allows it
        for (int j = 0; j < ndev; ++j) {
          if (devices[i] == devices[j]) continue;
          int can = 0;
          cudaDeviceCanAccessPeer(&can, devices[i], devices[j]);
          if (can) {
            cudaSetDevice(devices[i]);
            cudaDeviceEnablePeerAccess(devices[j], 0);
            cudaGetLastError();  // already enabled is fine
          }
        }
      g->backend = kPeer;
    }
  }
  *out = g;
  return FMGP_OK;
}

int fmgp_group_info(const fmgp_group* g, int32_t* nranks, int32_t* local_members, int32_t* backend) {
  if (g == nullptr) return fail(FMGP_EINVAL, "null group");
  if (nranks) *nranks = g->nranks;
  if (local_members) *local_members = static_cast<int32_t>(g->local.size());
  if (backend) *backend = g->backend;
  return FMGP_OK;
}

void fmgp_group_destroy(fmgp_group* g) {
  if (g == nullptr) return;
  DeviceGuard dg;
  for (auto& mb : g->local)
    if (mb.comm != nullptr) {
      cudaSetDevice(mb.device);
      nccl().CommDestroy(mb.comm);
    }
  delete g;
}

int fmgp_group_rows(int64_t n, int32_t nranks, int32_t member, int64_t* nblocks, int64_t* ranges) {
  if (n < 0 || nranks < 1 || member < 0 || member >= nranks) return fail(FMGP_EINVAL, "group rows: bad arguments");
  const Cyclic cy = make_cyclic(n, nranks);
  int64_t cnt = 0;
  for (int64_t c = 0; c < cy.rounds(); ++c) {
    int64_t b, e;
    cy.block(c, member, b, e);
    if (e <= b) continue;
    if (ranges != nullptr) {
      ranges[2 * cnt] = b;
      ranges[2 * cnt + 1] = e;
    }
    ++cnt;
  }
  if (nblocks) *nblocks = cnt;
  return FMGP_OK;
}

int fmgp_group_precompute_device(fmgp_group* g, const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                                 const fmgp_kernel_params* params, int32_t k, int32_t* S_out, double* C_out,
                                 int64_t* failed_row, void* stream) {
  if (failed_row) *failed_row = -1;
  if (g == nullptr) return fail(FMGP_EINVAL, "null group");
  if (g->local.size() != 1)
    return fail(FMGP_EINVAL, "group: device-pointer precompute needs one member per process (a rank group)");
  fmgp::KParams kp;
  int rc;
  if ((rc = validate(params, n, d, m, k, &kp)) != FMGP_OK) return rc;
  if ((rc = require_device()) != FMGP_OK) return rc;
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg;
  FMGP_CUDA(cudaSetDevice(g->local[0].device));
  CallCtx cx;
  cx.g = g;
  cx.cy = make_cyclic(n, g->nranks);
  cx.S = {S_out};
  cx.C = {C_out};
  MemberStreams st;
  st.work = static_cast<cudaStream_t>(stream);
  Stream side;
  FMGP_CUDA(side.create());
  st.side = side.s;
  DevBuf<unsigned long long> fmin;
  FMGP_CUDA(fmin.alloc(1, st.work));
  FMGP_CUDA(cudaMemsetAsync(fmin.p, 0xFF, sizeof(unsigned long long), st.work));
  if ((rc = member_precompute(cx, 0, X, Y, n, d, m, kp, k, st, fmin.p, nullptr, nullptr)) != FMGP_OK) return rc;
  unsigned long long host_min = ~0ull;
  FMGP_CUDA(cudaMemcpyAsync(&host_min, fmin.p, sizeof(host_min), cudaMemcpyDeviceToHost, st.work));
  FMGP_CUDA(cudaStreamSynchronize(st.work));
  if (host_min != ~0ull) return numeric_fail(host_min, failed_row);
  return FMGP_OK;
}

int fmgp_group_precompute(fmgp_group* g, const double* X, const double* Y, int64_t n, int32_t d, int32_t m,
                          const fmgp_kernel_params* params, int32_t k, const double* mean_offset, int32_t* S_out,
                          double* C_out, int64_t* failed_row, fmgp_model** model_out) {
  if (failed_row) *failed_row = -1;
  if (model_out) *model_out = nullptr;
  if (g == nullptr) return fail(FMGP_EINVAL, "null group");
  fmgp::KParams kp;
  int rc;
  if ((rc = validate(params, n, d, m, k, &kp)) != FMGP_OK) return rc;
  if (model_out != nullptr && mean_offset == nullptr) return fail(FMGP_EINVAL, "group: a model needs mean offsets");
  if ((rc = require_device()) != FMGP_OK) return rc;
  std::lock_guard<std::mutex> lk(g->mu);
  DeviceGuard dg;
  const int G = static_cast<int>(g->local.size());
  CallCtx cx;
  cx.g = g;
  cx.cy = make_cyclic(n, g->nranks);
  cx.S.assign(G, nullptr);
  cx.C.assign(G, nullptr);
  Barrier bar(G);
  cx.bar = &bar;
  std::vector<double*> Xd(G, nullptr), Yd(G, nullptr);
  std::vector<int> rcs(G, FMGP_OK);
  std::vector<std::string> msgs(G);
  std::vector<unsigned long long> mins(G, ~0ull);

  std::vector<int> pre(G, FMGP_OK);
  // phase 1 (before any collective): streams, buffers, uploads, the X check.
  // Every member reaches the barrier exactly once, then all of them see every
  // member's phase-1 outcome, so either all start the collectives or none does.
  auto phase1 = [&](int mi, MemberStreams& st) -> int {
    FMGP_CUDA(cudaSetDevice(g->local[mi].device));
    // replicas are plain allocations (they may outlive the call as model replicas)
    FMGP_CUDA(cudaMalloc(&Xd[mi], sizeof(double) * n * d));
    FMGP_CUDA(cudaMalloc(&Yd[mi], sizeof(double) * n * m));
    FMGP_CUDA(cudaMalloc(&cx.S[mi], sizeof(int32_t) * n * k));
    FMGP_CUDA(cudaMalloc(&cx.C[mi], sizeof(double) * n * k * m));
    FMGP_CUDA(cudaMemcpyAsync(Xd[mi], X, sizeof(double) * n * d, cudaMemcpyHostToDevice, st.work));
    FMGP_CUDA(cudaMemcpyAsync(Yd[mi], Y, sizeof(double) * n * m, cudaMemcpyHostToDevice, st.rb));
    FMGP_CUDA(st.handoff(st.rb, st.work));
    // NeighborIndex::build's finiteness check on the device copy (every member sees the same X)
    DevBuf<unsigned int> nbad;
    FMGP_CUDA(nbad.alloc(1, st.work));
    FMGP_CUDA(fmgp::nonfinite_count_launch(Xd[mi], n * d, nbad.p, num_sms_current(), st.work));
    unsigned int hb = 0;
    FMGP_CUDA(cudaMemcpyAsync(&hb, nbad.p, sizeof(hb), cudaMemcpyDeviceToHost, st.work));
    FMGP_CUDA(cudaStreamSynchronize(st.work));
    if (hb != 0) return fail(FMGP_EINVAL, "NeighborIndex: non-finite coordinates");
    return FMGP_OK;
  };
  auto run = [&](int mi) {
    MemberStreams st;
    Stream work, side, rbs;
    cudaSetDevice(g->local[mi].device);
    int rc1 = FMGP_OK;
    if (work.create() != cudaSuccess || side.create() != cudaSuccess || rbs.create() != cudaSuccess)
      rc1 = fail(FMGP_ECUDA, "group: stream creation failed");
    st.work = work.s;
    st.side = side.s;
    st.rb = rbs.s;
    if (rc1 == FMGP_OK) rc1 = phase1(mi, st);
    pre[mi] = rc1;
    if (rc1 != FMGP_OK) msgs[mi] = g_err;
    bar.wait();
    for (int q = 0; q < G; ++q)
      if (pre[q] != FMGP_OK) {
        rcs[mi] = pre[q];
        msgs[mi] = msgs[q];
        return;
      }
    auto phase2 = [&]() -> int {
      DevBuf<unsigned long long> fmin;
      FMGP_CUDA(fmin.alloc(1, st.work));
      FMGP_CUDA(cudaMemsetAsync(fmin.p, 0xFF, sizeof(unsigned long long), st.work));
      int rc2 = member_precompute(cx, mi, Xd[mi], Yd[mi], n, d, m, kp, k, st, fmin.p, S_out, C_out);
      if (rc2 != FMGP_OK) return rc2;
      FMGP_CUDA(cudaMemcpyAsync(&mins[mi], fmin.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st.work));
      FMGP_CUDA(cudaStreamSynchronize(st.work));
      return FMGP_OK;
    };
    rcs[mi] = phase2();
    if (rcs[mi] != FMGP_OK) msgs[mi] = g_err;
    // the peer backend writes into other members' buffers: nobody leaves
    // (and frees) before every member's pushes are complete
    cudaDeviceSynchronize();
  };
  if (G == 1) {
    run(0);
  } else {
    std::vector<std::thread> th;
    for (int mi = 0; mi < G; ++mi)
      th.emplace_back([&, mi] {
        run(mi);
      });
    for (auto& t : th) t.join();
  }
  int worst = -1;
  for (int mi = 0; mi < G; ++mi)
    if (rcs[mi] != FMGP_OK && worst < 0) worst = mi;
  unsigned long long low = ~0ull;
  for (auto v : mins) low = std::min(low, v);
  auto release = [&] {
    for (int mi = 0; mi < G; ++mi) {
      cudaSetDevice(g->local[mi].device);
      if (Xd[mi]) cudaFree(Xd[mi]);
      if (Yd[mi]) cudaFree(Yd[mi]);
      if (cx.S[mi]) cudaFree(cx.S[mi]);
      if (cx.C[mi]) cudaFree(cx.C[mi]);
    }
  };
  if (worst >= 0) {
    release();
    return fail(rcs[worst], msgs[worst]);
  }
  if (low != ~0ull) {
    release();
    return numeric_fail(low, failed_row);
  }
  if (model_out == nullptr) {
    release();
    return FMGP_OK;
  }
  // the members' device results become the model's replicas (no copy)
  auto* mdl = new fmgp_model();
  mdl->n = n;
  mdl->d = d;
  mdl->k = k;
  mdl->m = m;
  mdl->kp = kp;
  cudaError_t e = cudaSuccess;
  for (int mi = 0; mi < G; ++mi) {
    cudaSetDevice(g->local[mi].device);
    cudaFree(Yd[mi]);
    Yd[mi] = nullptr;
    mdl->reps.emplace_back();
    fmgp_model_replica& r = mdl->reps.back();
    r.device = g->local[mi].device;
    r.X = Xd[mi];
    r.S = cx.S[mi];
    r.C = cx.C[mi];
    Xd[mi] = nullptr;
    cx.S[mi] = nullptr;
    cx.C[mi] = nullptr;
    if (e == cudaSuccess) e = replica_finish(r, n, d, k, m, mean_offset);
  }
  if (e != cudaSuccess) {
    fmgp_model_destroy(mdl);
    return cuda_fail(e, "fmgp_group_precompute (model replicas)");
  }
  *model_out = mdl;
  return FMGP_OK;
}

}  // extern "C"
