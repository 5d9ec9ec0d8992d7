"""Python mirror of the reference's public API for the FastMuyGPs path.

Same names, argument meanings and error behaviour as
/root/reference/proj/core/include/fastmuygps/{kernel,nn_index,fast_predict,
dataset,linalg,errors}.hpp, over the C ABI (include/fmgp_b200.h). Every
compute call runs on the GPU through libfmgp_b200.so; the host side only
validates arguments and moves buffers.

Deviations (documented in DESIGN.md):
  * `threads` in precompute is accepted and ignored (the GPU result is the
    same for any thread count, as the reference guarantees, fast_predict.hpp:35-37).
  * `IndexMode.ApproxGraph` is accepted by NeighborIndex.build but queries are
    always exact (parity is defined against IndexMode::Exact).
  * Y may carry m > 1 outputs (BASELINE cfg3); C is then n x k x m.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import DomainError, NumericError, CudaError, FmgpError  # noqa: F401  (re-export)


class KernelKind(enum.IntEnum):
    Matern = 0
    RBF = 1


class IndexMode(enum.IntEnum):
    Exact = 0
    ApproxGraph = 1


@dataclass(frozen=True)
class GraphParams:
    """nn_index.hpp:14-19 (query_beam <= 0: max(64, 2k) at query time)."""
    max_degree: int = 16
    build_beam: int = 100
    query_beam: int = 0
    seed: int = 0


@dataclass(frozen=True)
class KernelParams:
    """kernel.hpp:12-33; validated like kernel.cpp:13-28."""
    sigma: float
    rho: float
    nu: float
    tau: float

    def __post_init__(self):
        if not (math.isfinite(self.sigma) and self.sigma > 0):
            raise DomainError(N.FMGP_EINVAL, "KernelParams: sigma must be positive and finite")
        if not (math.isfinite(self.rho) and self.rho > 0):
            raise DomainError(N.FMGP_EINVAL, "KernelParams: rho must be positive and finite")
        if not (math.isfinite(self.nu) and self.nu > 0):
            raise DomainError(N.FMGP_EINVAL, "KernelParams: nu must be positive and finite")
        if not (math.isfinite(self.tau) and self.tau >= 0):
            raise DomainError(N.FMGP_EINVAL, "KernelParams: tau must be non-negative and finite")

    def with_rho(self, rho):
        return KernelParams(self.sigma, rho, self.nu, self.tau)

    def with_nu(self, nu):
        return KernelParams(self.sigma, self.rho, nu, self.tau)

    def with_tau(self, tau):
        return KernelParams(self.sigma, self.rho, self.nu, tau)

    def with_sigma(self, sigma):
        return KernelParams(sigma, self.rho, self.nu, self.tau)

    def c(self, kind: KernelKind) -> N.KernelParamsC:
        return N.KernelParamsC(int(kind), self.sigma, self.rho, self.nu, self.tau)


@dataclass
class FittedParams:
    """muygps.hpp:41-47 (only theta_hat and kind reach the path)."""
    theta_hat: KernelParams
    kind: KernelKind = KernelKind.Matern
    final_loss: float = 0.0
    evaluations: int = 0
    improved: bool = False


@dataclass
class TrainingSet:
    """dataset.hpp:12-16 (X n x d; Y n or n x m detrended; mean_offset per output)."""
    X: np.ndarray
    Y: np.ndarray
    mean_offset: float | np.ndarray = 0.0


def detrend(X, raw_y) -> TrainingSet:
    """dataset.cpp:24-36."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.asarray(raw_y, dtype=np.float64)
    if X.ndim != 2 or X.shape[0] != y.shape[0] or X.shape[0] < 1:
        raise DomainError(N.FMGP_EINVAL, "detrend: features and responses disagree on n")
    if not np.all(np.isfinite(y)):
        raise DomainError(N.FMGP_EINVAL, "detrend: non-finite response")
    mu = y.mean(axis=0)
    return TrainingSet(X, y - mu, mu)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class NeighborList:
    """nn_index.hpp:22-27."""
    indices: list
    distances: list


class NeighborIndex:
    """Neighbour index (nn_index.hpp:33-60) on the GPU. Immutable.

    Exact: exact search (cell grid / tcgen05 / brute force). ApproxGraph: the
    GPU navigable-small-world graph of graph.cu (fmgp_graph_build; the
    reference's seeded levels, layers linked to their exact nearest
    neighbours), searched with the reference's graph search; `dist_evals`
    counts its distance evaluations (nn_index.hpp:39-44)."""

    def __init__(self, points: np.ndarray, mode: IndexMode, params: GraphParams | None = None):
        self._pts = points
        self._mode = IndexMode(mode)
        self._params = params or GraphParams()
        self._dev = None  # device-resident copy + nearest-point grid (fmgp_index), made on first query
        self.dist_evals = 0
        if self._mode == IndexMode.ApproxGraph:
            g = C.c_void_p()
            p = self._params
            N.check(N.LIB.fmgp_graph_build(self._handle(), p.max_degree, p.build_beam, p.query_beam,
                                           C.c_uint64(p.seed), C.byref(g)))
            self._dev.g = g.value

    @property
    def _graph_h(self):
        return self._dev.g if self._dev is not None else None

    def _handle(self):
        if self._dev is None:
            h = C.c_void_p()
            N.check(N.LIB.fmgp_index_create(_ptr(self._pts), self.size(), self.dim(), -1, C.byref(h)))
            self._dev = _IndexHandle(h)
        return self._dev.h

    @staticmethod
    def build(points, mode: IndexMode = IndexMode.Exact, params: GraphParams | None = None) -> "NeighborIndex":
        p = params or GraphParams()
        if p.max_degree < 2 or p.build_beam < 1:
            raise DomainError(N.FMGP_EINVAL, "NeighborIndex: invalid graph parameters")
        P = _f64(points)
        if P.ndim != 2 or P.shape[0] < 1:
            raise DomainError(N.FMGP_EINVAL, "NeighborIndex: empty point set")
        if not np.all(np.isfinite(P)):
            raise DomainError(N.FMGP_EINVAL, "NeighborIndex: non-finite coordinates")
        return NeighborIndex(P, mode, p)

    def params(self) -> GraphParams:
        return self._params

    def graph_arrays(self):
        """ApproxGraph: (entry, max_level, levels, counts, ids) in the reference's
        serialization order (nn_index.cpp:397-416)."""
        if self._graph_h is None:
            raise DomainError(N.FMGP_EINVAL, "not an ApproxGraph index")
        entry, ml = C.c_int32(), C.c_int32()
        ct, it = C.c_int64(), C.c_int64()
        N.check(N.LIB.fmgp_graph_info(self._graph_h, C.byref(entry), C.byref(ml), C.byref(ct), C.byref(it)))
        levels = np.empty(self.size(), dtype=np.int32)
        counts = np.empty(ct.value, dtype=np.uint32)
        ids = np.empty(max(it.value, 1), dtype=np.int32)
        N.check(N.LIB.fmgp_graph_export(self._graph_h, _ptr(levels), _ptr(counts), _ptr(ids)))
        return entry.value, ml.value, levels, counts, ids[:it.value]

    @staticmethod
    def from_graph_arrays(points, params: GraphParams, entry, max_level, levels, counts, ids) -> "NeighborIndex":
        """A serialized graph (e.g. reference-written) over `points`."""
        ix = NeighborIndex.build(points, IndexMode.Exact)
        ix._mode = IndexMode.ApproxGraph
        ix._params = params
        lv = np.ascontiguousarray(levels, dtype=np.int32)
        ct = np.ascontiguousarray(counts, dtype=np.uint32)
        idv = np.ascontiguousarray(ids if len(ids) else [0], dtype=np.int32)
        g = C.c_void_p()
        N.check(N.LIB.fmgp_graph_load(ix._handle(), params.max_degree, params.build_beam, params.query_beam,
                                      C.c_uint64(params.seed), int(entry), int(max_level), _ptr(lv), _ptr(ct),
                                      _ptr(idv), C.byref(g)))
        ix._dev.g = g.value
        return ix

    def size(self) -> int:
        return self._pts.shape[0]

    def dim(self) -> int:
        return self._pts.shape[1]

    def mode(self) -> IndexMode:
        return self._mode

    @property
    def points(self) -> np.ndarray:
        return self._pts

    def query_knn_batch(self, Q, k: int, exclude=None):
        """Batched query_knn: (indices nq x k int32, distances nq x k)."""
        Q = _f64(Q)
        if Q.ndim != 2 or Q.shape[1] != self.dim():
            raise DomainError(N.FMGP_EINVAL, "query_knn: query dimension mismatch")
        nq = Q.shape[0]
        idx = np.empty((nq, k), dtype=np.int32)
        dist = np.empty((nq, k), dtype=np.float64)
        ex = None if exclude is None else np.ascontiguousarray(exclude, dtype=np.int32)
        if self._graph_h is not None:
            ev = C.c_uint64(0)
            N.check(N.LIB.fmgp_graph_query_knn(self._graph_h, _ptr(Q), nq, k, _ptr(ex), _ptr(idx), _ptr(dist),
                                               C.byref(ev)))
            self.dist_evals += ev.value
            return idx, dist
        N.check(N.LIB.fmgp_index_query_knn(self._handle(), _ptr(Q), nq, k, _ptr(ex), _ptr(idx), _ptr(dist)))
        self.dist_evals += nq * (self.size() - (0 if ex is None else int(np.count_nonzero(ex >= 0)) // max(nq, 1)))
        return idx, dist

    def query_knn(self, q, k: int, exclude_index: int = -1) -> NeighborList:
        q = _f64(q).reshape(-1)
        if q.size != self.dim():
            raise DomainError(N.FMGP_EINVAL, "query_knn: query dimension mismatch")
        idx, dist = self.query_knn_batch(q[None, :], k, np.array([exclude_index], dtype=np.int32))
        return NeighborList(idx[0].tolist(), dist[0].tolist())

    def nearest_batch(self, Q) -> np.ndarray:
        Q = _f64(Q)
        if Q.ndim != 2 or Q.shape[1] != self.dim():
            raise DomainError(N.FMGP_EINVAL, "nearest_training_point: dimension mismatch")
        out = np.empty(Q.shape[0], dtype=np.int32)
        if self._graph_h is not None:
            ev = C.c_uint64(0)
            N.check(N.LIB.fmgp_graph_nearest(self._graph_h, _ptr(Q), Q.shape[0], _ptr(out), C.byref(ev)))
            self.dist_evals += ev.value
            return out
        N.check(N.LIB.fmgp_index_nearest(self._handle(), _ptr(Q), Q.shape[0], _ptr(out)))
        self.dist_evals += Q.shape[0] * self.size()
        return out

    def nearest_training_point(self, q) -> int:
        q = _f64(q).reshape(-1)
        if q.size != self.dim():
            raise DomainError(N.FMGP_EINVAL, "nearest_training_point: dimension mismatch")
        return int(self.nearest_batch(q[None, :])[0])


@dataclass
class PrecomputedModel:
    """fast_predict.hpp:25-33; C is n x k (m = 1) or n x k x m."""
    X: np.ndarray
    S: np.ndarray
    C: np.ndarray
    params: KernelParams
    kind: KernelKind
    mean_offset: float | np.ndarray
    index: NeighborIndex
    _handle: object = field(default=None, repr=False)

    @property
    def m(self) -> int:
        return 1 if self.C.ndim == 2 else self.C.shape[2]

    def _offsets(self) -> np.ndarray:
        return np.ascontiguousarray(np.broadcast_to(np.asarray(self.mean_offset, dtype=np.float64),
                                                    (self.m,)))

    def handle(self):
        """Lazily created device-resident replica (fmgp_model_create) on the
        calling thread's current CUDA device."""
        if self._handle is None:
            h = C.c_void_p()
            n, k = self.S.shape
            mo = self._offsets()
            kp = self.params.c(self.kind)
            N.check(N.LIB.fmgp_model_create(_ptr(self.X), _ptr(self.S), _ptr(self.C), n, self.X.shape[1], k,
                                            self.m, C.byref(kp), _ptr(mo), -1, C.byref(h)))
            self._handle = _ModelHandle(h)
        return self._handle.h

    table = property(lambda self: self.S)


class _IndexHandle:
    """fmgp_index and, in ApproxGraph mode, its fmgp_graph: one owner, so the
    graph is always destroyed before the points it searches (a garbage
    collection of both in one cycle finalizes them in arbitrary order)."""

    def __init__(self, h):
        self.h = h
        self.g = None

    def __del__(self):
        if self.g:
            N.LIB.fmgp_graph_destroy(self.g)
            self.g = None
        if self.h:
            N.LIB.fmgp_index_destroy(self.h)
            self.h = None


class _ModelHandle:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        if self.h:
            N.LIB.fmgp_model_destroy(self.h)
            self.h = None


def precompute(train: TrainingSet, fitted: FittedParams, index: NeighborIndex, k: int,
               threads: int = 1) -> PrecomputedModel:
    """fast_predict.cpp:70-130 on the GPU."""
    X = _f64(train.X)
    n = X.shape[0]
    if k < 1 or k > n:
        raise DomainError(N.FMGP_EINVAL, "precompute: k out of range")
    if index.size() != n:
        raise DomainError(N.FMGP_EINVAL, "precompute: index was not built on the training set")
    Y = _f64(train.Y)
    m = 1 if Y.ndim == 1 else Y.shape[1]
    S = np.empty((n, k), dtype=np.int32)
    Cm = np.empty((n, k, m), dtype=np.float64)
    failed = C.c_int64(-1)
    kp = fitted.theta_hat.c(fitted.kind)
    rc = N.LIB.fmgp_precompute(_ptr(X), _ptr(Y), n, X.shape[1], m, C.byref(kp), k, _ptr(S), _ptr(Cm),
                               C.byref(failed))
    N.check(rc, failed.value)
    return PrecomputedModel(X.copy(), S, Cm[:, :, 0].copy() if Y.ndim == 1 else Cm, fitted.theta_hat,
                            fitted.kind, train.mean_offset, index)


def fast_predict_batch(model: PrecomputedModel, Z) -> np.ndarray:
    """fast_predict.cpp:146-156 on the GPU."""
    Z = _f64(Z)
    if Z.ndim != 2 or Z.shape[1] != model.X.shape[1]:
        raise DomainError(N.FMGP_EINVAL, "fast_predict_batch: test dimension mismatch")
    out = np.empty((Z.shape[0], model.m), dtype=np.float64)
    N.check(N.LIB.fmgp_model_predict(model.handle(), _ptr(Z), Z.shape[0], _ptr(out), None))
    return out[:, 0] if model.C.ndim == 2 else out


def fast_predict_one(model: PrecomputedModel, z):
    """fast_predict.cpp:132-144."""
    z = _f64(z).reshape(1, -1)
    r = fast_predict_batch(model, z)
    return float(r[0]) if model.C.ndim == 2 else r[0]


def kernel_value(d: float, kind: KernelKind, p: KernelParams) -> float:
    """kernel.cpp:88-90 (evaluated on the device)."""
    return float(kernel_values(np.array([d], dtype=np.float64), kind, p)[0])


def kernel_values(dists, kind: KernelKind, p: KernelParams) -> np.ndarray:
    dd = _f64(dists).reshape(-1)
    out = np.empty_like(dd)
    kp = p.c(kind)
    N.check(N.LIB.fmgp_kernel_values(_ptr(dd), dd.size, C.byref(kp), _ptr(out)))
    return out


def matern_value(d: float, p: KernelParams) -> float:
    return kernel_value(d, KernelKind.Matern, p)


def rbf_value(d: float, p: KernelParams) -> float:
    return kernel_value(d, KernelKind.RBF, p)


def cov_matrix(A, B, kind: KernelKind, p: KernelParams) -> np.ndarray:
    """kernel.cpp:92-104."""
    A, B = _f64(A), _f64(B)
    if A.shape[1] != B.shape[1]:
        raise DomainError(N.FMGP_EINVAL, "cov_matrix: point sets have mismatched dimension")
    K = np.empty((A.shape[0], B.shape[0]), dtype=np.float64)
    kp = p.c(kind)
    N.check(N.LIB.fmgp_cov_matrix(_ptr(A), A.shape[0], _ptr(B), B.shape[0], A.shape[1], C.byref(kp), _ptr(K)))
    return K


def cov_matrix_self(A, kind: KernelKind, p: KernelParams) -> np.ndarray:
    """kernel.cpp:106-119."""
    A = _f64(A)
    K = np.empty((A.shape[0], A.shape[0]), dtype=np.float64)
    kp = p.c(kind)
    N.check(N.LIB.fmgp_cov_matrix(_ptr(A), A.shape[0], None, 0, A.shape[1], C.byref(kp), _ptr(K)))
    return K


def solve_spd_batched(K, B):
    """linalg.cpp:10-36 over a batch: returns (X, applied_jitter)."""
    K = _f64(K)
    B = _f64(B)
    if K.ndim == 2:
        K = K[None]
    batch, k, _ = K.shape
    B3 = B.reshape(batch, k, -1)
    m = B3.shape[2]
    X = np.empty_like(B3)
    jit = np.empty(batch, dtype=np.float64)
    failed = C.c_int64(-1)
    rc = N.LIB.fmgp_solve_spd_batched(_ptr(K), _ptr(np.ascontiguousarray(B3)), batch, k, m, _ptr(X), _ptr(jit),
                                      C.byref(failed))
    N.check(rc, failed.value)
    return X, jit


def solve_spd(K, B, context: str = "solve_spd") -> np.ndarray:
    """linalg.cpp:33-36."""
    B = _f64(B)
    try:
        X, _ = solve_spd_batched(K, B)
    except NumericError as e:
        raise NumericError(e.code, f"Cholesky factorization failed in {context} after jitter escalation up to 1e-6",
                           e.failed_row) from None
    return X[0].reshape(B.shape)


# ---------------------------------------------------------------------------
# Device-resident stage calls (torch tensors on the current CUDA device).
# Used by bench.py and the multi-GPU sharding in parallel.py.

def _dp(t) -> int:
    return int(t.data_ptr())


def precompute_device(X, Y, fitted: FittedParams, k: int, row_begin: int, row_end: int, S_out, C_out,
                      stream=None) -> None:
    """fmgp_precompute_device: rows [row_begin, row_end) of precompute, all buffers in HBM."""
    import torch
    n, d = X.shape
    m = 1 if Y.dim() == 1 else Y.shape[1]
    s = stream if stream is not None else torch.cuda.current_stream()
    failed = C.c_int64(-1)
    kp = fitted.theta_hat.c(fitted.kind)
    rc = N.LIB.fmgp_precompute_device(_dp(X), _dp(Y), n, d, m, C.byref(kp), k, row_begin, row_end, _dp(S_out),
                                      _dp(C_out), C.byref(failed), C.c_void_p(s.cuda_stream))
    N.check(rc, failed.value)


def predict_device(X, S, Cmat, fitted: FittedParams, mean_offset, Z, out, nn_out=None, stream=None) -> None:
    """fmgp_predict_device: posterior means for Z, all buffers in HBM."""
    import torch
    n, d = X.shape
    k = S.shape[1]
    m = 1 if Cmat.dim() == 2 else Cmat.shape[2]
    s = stream if stream is not None else torch.cuda.current_stream()
    mo = np.ascontiguousarray(np.broadcast_to(np.asarray(mean_offset, dtype=np.float64), (m,)))
    kp = fitted.theta_hat.c(fitted.kind)
    rc = N.LIB.fmgp_predict_device(_dp(X), _dp(S), _dp(Cmat), n, d, k, m, C.byref(kp), _ptr(mo), _dp(Z), Z.shape[0],
                                   _dp(out), None if nn_out is None else _dp(nn_out), C.c_void_p(s.cuda_stream))
    N.check(rc)


# ------------------------------------------------------------------ MuyGPs
# muygps.hpp: the training inner loop (LOOCV over a batch, Nelder-Mead) and
# the localized baseline predictor, on the device (include/fmgp_b200.h).

@dataclass
class BatchSpec:
    """muygps.hpp:15-21."""
    b: int = 0
    seed: int = 0
    indices: list = field(default_factory=list)

    @staticmethod
    def sample(n: int, b: int, seed: int) -> "BatchSpec":
        """muygps.cpp:15-30 (partial Fisher-Yates over std::mt19937_64)."""
        from . import datagen
        if b < 1 or b > n:
            raise DomainError(N.FMGP_EINVAL, "BatchSpec: batch size out of range")
        return BatchSpec(b, seed, datagen.batch_sample(n, b, seed))


@dataclass
class Bounds:
    lo: float
    hi: float


@dataclass
class TrainConfig:
    """muygps.hpp:28-39."""
    k: int = 50
    kind: KernelKind = KernelKind.Matern
    rho_bounds: Bounds | None = None
    nu_bounds: Bounds | None = None
    tau_bounds: Bounds | None = None
    max_evals: int = 200
    tol: float = 1e-8


def _lists_to_arrays(neighbor_lists) -> tuple[np.ndarray, np.ndarray]:
    k = len(neighbor_lists[0].indices)
    nbr = np.array([list(nl.indices) for nl in neighbor_lists], dtype=np.int32).reshape(len(neighbor_lists), k)
    dist = np.array([list(nl.distances) for nl in neighbor_lists], dtype=np.float64).reshape(len(neighbor_lists), k)
    return nbr, dist


def local_predictions(train: TrainingSet, batch_indices, nbr, dist, kind: KernelKind, p: KernelParams) -> np.ndarray:
    """fmgp_local_predictions: local_prediction (muygps.cpp:32-62) for b entries with k-neighbour lists."""
    X = _f64(train.X)
    Y = _f64(train.Y)
    bi = np.ascontiguousarray(batch_indices, dtype=np.int32)
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    dist = _f64(dist)
    b = bi.shape[0]
    k = nbr.shape[1] if nbr.ndim == 2 else 0
    out = np.empty(b, dtype=np.float64)
    failed = C.c_int64(-1)
    kp = p.c(kind)
    rc = N.LIB.fmgp_local_predictions(_ptr(X), _ptr(Y), X.shape[0], X.shape[1], _ptr(bi), _ptr(nbr), _ptr(dist),
                                      b, k, C.byref(kp), _ptr(out), C.byref(failed))
    N.check(rc, failed.value)
    return out


def local_prediction(train: TrainingSet, i: int, neighbors: NeighborList, kind: KernelKind,
                     p: KernelParams) -> float:
    """muygps.cpp:32-62 (one entry)."""
    k = len(neighbors.indices)
    nbr = np.asarray(neighbors.indices, dtype=np.int32).reshape(1, k)
    dist = np.asarray(neighbors.distances, dtype=np.float64).reshape(1, k)
    return float(local_predictions(train, [i], nbr, dist, kind, p)[0])


def loocv_loss(train: TrainingSet, batch: BatchSpec, neighbor_lists, kind: KernelKind, p: KernelParams) -> float:
    """muygps.cpp:64-78: mean squared leave-one-out residual over the batch (sequential sum)."""
    if len(neighbor_lists) != len(batch.indices) or not batch.indices:
        raise DomainError(N.FMGP_EINVAL, "loocv_loss: batch and neighbor lists disagree")
    sizes = {len(nl.indices) for nl in neighbor_lists}
    Y = np.asarray(train.Y, dtype=np.float64)
    if len(sizes) == 1:
        nbr, dist = _lists_to_arrays(neighbor_lists)
        preds = local_predictions(train, batch.indices, nbr, dist, kind, p)
    else:  # ragged lists: entry by entry, in batch order (the reference's error order)
        preds = [local_prediction(train, i, nl, kind, p) for i, nl in zip(batch.indices, neighbor_lists)]
    s = 0.0
    for i, pr in zip(batch.indices, preds):
        r = float(Y[i]) - float(pr)
        s += r * r
    return s / float(len(batch.indices))


class LoocvSession:
    """fmgp_loocv_*: device-resident LOOCV data for repeated loss evaluations."""

    def __init__(self, train: TrainingSet, batch: BatchSpec, neighbor_lists):
        if len(neighbor_lists) != len(batch.indices) or not batch.indices:
            raise DomainError(N.FMGP_EINVAL, "loocv_loss: batch and neighbor lists disagree")
        X = _f64(train.X)
        Y = _f64(train.Y)
        bi = np.ascontiguousarray(batch.indices, dtype=np.int32)
        nbr, dist = _lists_to_arrays(neighbor_lists)
        h = C.c_void_p()
        N.check(N.LIB.fmgp_loocv_create(_ptr(X), _ptr(Y), X.shape[0], X.shape[1], _ptr(bi), _ptr(nbr), _ptr(dist),
                                        bi.shape[0], nbr.shape[1], C.byref(h)))
        self._h = h
        self.b = bi.shape[0]

    def loss(self, kind: KernelKind, p: KernelParams, with_predictions: bool = False):
        kp = p.c(kind)
        val = C.c_double(0.0)
        failed = C.c_int64(-1)
        preds = np.empty(self.b, dtype=np.float64) if with_predictions else None
        N.check(N.LIB.fmgp_loocv_eval(self._h, C.byref(kp), C.byref(val), _ptr(preds), C.byref(failed)),
                failed.value)
        return (val.value, preds) if with_predictions else val.value

    def close(self):
        if self._h:
            N.LIB.fmgp_loocv_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 (interpreter shutdown)
            pass


def train(data: TrainingSet, initial: KernelParams, config: TrainConfig, batch: BatchSpec,
          index: NeighborIndex) -> FittedParams:
    """muygps.cpp:214-270 — neighbour lists and every LOOCV evaluation on the device."""
    X = _f64(data.X)
    Y = _f64(data.Y)
    if config.k < 2:
        raise DomainError(N.FMGP_EINVAL, "train: k must be at least 2")
    if index.size() != X.shape[0]:
        raise DomainError(N.FMGP_EINVAL, "train: index was not built on the training set")
    bi = np.ascontiguousarray(batch.indices, dtype=np.int32)
    cfg = N.TrainConfigC()
    cfg.k, cfg.kind, cfg.max_evals, cfg.tol = config.k, int(config.kind), config.max_evals, config.tol
    for name in ("rho", "nu", "tau"):
        bnd = getattr(config, name + "_bounds")
        setattr(cfg, "has_" + name, 1 if bnd is not None else 0)
        if bnd is not None:
            setattr(cfg, name + "_lo", bnd.lo)
            setattr(cfg, name + "_hi", bnd.hi)
    kp0 = initial.c(config.kind)
    th = N.KernelParamsC()
    loss = C.c_double(0.0)
    evals = C.c_int32(0)
    imp = C.c_int32(0)
    N.check(N.LIB.fmgp_train(_ptr(X), _ptr(Y), X.shape[0], X.shape[1], _ptr(bi), bi.shape[0], C.byref(kp0),
                             C.byref(cfg), C.byref(th), C.byref(loss), C.byref(evals), C.byref(imp)))
    theta = KernelParams(th.sigma, th.rho, th.nu, th.tau)
    return FittedParams(theta, config.kind, loss.value, evals.value, bool(imp.value))


def muygps_predict(train: TrainingSet, Z, fitted: FittedParams, index: NeighborIndex, k: int) -> np.ndarray:
    """muygps.cpp:272-295: each test point conditioned on its own k exact neighbours."""
    X = _f64(train.X)
    Y = _f64(train.Y)
    Z = _f64(Z)
    if Z.ndim == 1:
        Z = Z.reshape(1, -1)
    if Z.shape[1] != X.shape[1]:
        raise DomainError(N.FMGP_EINVAL, "muygps_predict: test dimension mismatch")
    out = np.empty(Z.shape[0], dtype=np.float64)
    failed = C.c_int64(-1)
    kp = fitted.theta_hat.c(fitted.kind)
    rc = N.LIB.fmgp_muygps_predict(_ptr(X), _ptr(Y), X.shape[0], X.shape[1], _ptr(Z), Z.shape[0], k, C.byref(kp),
                                   float(np.asarray(train.mean_offset).reshape(-1)[0]), _ptr(out), C.byref(failed))
    N.check(rc, failed.value)
    return out
