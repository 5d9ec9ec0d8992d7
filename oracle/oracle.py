"""ORACLE TEST INFRASTRUCTURE — ctypes front-ends of the two CPU checkers.

  Port       oracle/build/libfmgp_oracle.so  the C restatement (fmgp_oracle.c)
  Reference  oracle/_ref/libfmgp_ref.so      the reference's own TUs compiled
                                             unmodified against the shims, driven
                                             through its public API (harness/ref_harness.cpp)

Both take/return row-major numpy arrays. Used only as the checker (tests/,
__graft_entry__.smoke()) and as the CPU baseline (bench.py).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_PATH = HERE / "build" / "libfmgp_oracle.so"
REF_PATH = HERE / "_ref" / "libfmgp_ref.so"

_V = C.c_void_p


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, code, msg, failed_row=-1):
        super().__init__(msg)
        self.code = code
        self.failed_row = failed_row


class Port:
    """The C restatement (fmgp_oracle.c)."""

    kind = "port"

    def __init__(self, path: Path = PORT_PATH):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing; run make -C oracle")
        L = C.CDLL(str(path))
        L.fmgp_oracle_dist_sq.restype = C.c_double
        L.fmgp_oracle_dist_sq.argtypes = [_V, _V, C.c_int]
        L.fmgp_oracle_kernel_value.restype = C.c_double
        L.fmgp_oracle_kernel_value.argtypes = [C.c_double, C.c_int] + [C.c_double] * 4
        L.fmgp_oracle_query_knn.restype = C.c_int
        L.fmgp_oracle_query_knn.argtypes = [_V, C.c_int64, C.c_int, _V, C.c_int, C.c_int64, _V, _V]
        L.fmgp_oracle_nearest.restype = C.c_int32
        L.fmgp_oracle_nearest.argtypes = [_V, C.c_int64, C.c_int, _V]
        L.fmgp_oracle_cov_self.restype = None
        L.fmgp_oracle_cov_self.argtypes = [_V, C.c_int, C.c_int, C.c_int] + [C.c_double] * 4 + [_V]
        L.fmgp_oracle_cholesky_jitter.restype = C.c_int
        L.fmgp_oracle_cholesky_jitter.argtypes = [_V, C.c_int, _V]
        L.fmgp_oracle_precompute_rows.restype = C.c_int
        L.fmgp_oracle_precompute_rows.argtypes = ([_V, _V, C.c_int64, C.c_int, C.c_int, C.c_int] + [C.c_double] * 4 +
                                                  [C.c_int, _V, C.c_int64, C.c_int, _V, _V, _V])
        L.fmgp_oracle_predict.restype = C.c_int
        L.fmgp_oracle_predict.argtypes = ([_V, _V, _V, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int] +
                                          [C.c_double] * 5 + [_V, C.c_int64, C.c_int, _V, _V])
        L.fmgp_oracle_local_predictions.restype = C.c_int
        L.fmgp_oracle_local_predictions.argtypes = ([_V, _V, C.c_int64, C.c_int, _V, _V, C.c_int64, C.c_int,
                                                     C.c_int] + [C.c_double] * 4 + [_V, _V])
        L.fmgp_oracle_muygps_predict.restype = C.c_int
        L.fmgp_oracle_muygps_predict.argtypes = ([_V, _V, C.c_int64, C.c_int, C.c_double, _V, C.c_int64, C.c_int,
                                                  C.c_int] + [C.c_double] * 4 + [_V, _V])
        self.L = L

    def local_predictions(self, X, Y, nbr, dist, kind, sigma, rho, nu, tau):
        """muygps.cpp:32-62 per entry (no argument validation)."""
        X = _f64(X)
        Y = _f64(Y).reshape(-1)
        nbr = np.ascontiguousarray(nbr, dtype=np.int32)
        dist = _f64(dist)
        b, k = nbr.shape
        out = np.empty(b, dtype=np.float64)
        fe = C.c_int64(-1)
        rc = self.L.fmgp_oracle_local_predictions(_p(X), _p(Y), X.shape[0], X.shape[1], _p(nbr), _p(dist), b, k,
                                                  kind, sigma, rho, nu, tau, _p(out), C.byref(fe))
        if rc != 0:
            raise OracleError(rc, "local_prediction: Cholesky factorization failed", fe.value)
        return out

    def muygps_predict(self, X, Y, mean_offset, Z, k, kind, sigma, rho, nu, tau):
        """muygps.cpp:272-295."""
        X = _f64(X)
        Y = _f64(Y).reshape(-1)
        Z = _f64(Z)
        out = np.empty(Z.shape[0], dtype=np.float64)
        fr = C.c_int64(-1)
        rc = self.L.fmgp_oracle_muygps_predict(_p(X), _p(Y), X.shape[0], X.shape[1], mean_offset, _p(Z), Z.shape[0],
                                               k, kind, sigma, rho, nu, tau, _p(out), C.byref(fr))
        if rc != 0:
            raise OracleError(rc, "muygps_predict: Cholesky factorization failed", fr.value)
        return out

    def kernel_value(self, dist, kind, sigma, rho, nu, tau):
        return self.L.fmgp_oracle_kernel_value(dist, kind, sigma, rho, nu, tau)

    def query_knn(self, X, q, k, exclude=-1):
        X = _f64(X)
        q = _f64(q)
        idx = np.empty(k, dtype=np.int32)
        dsq = np.empty(k, dtype=np.float64)
        rc = self.L.fmgp_oracle_query_knn(_p(X), X.shape[0], X.shape[1], _p(q), k, exclude, _p(idx), _p(dsq))
        if rc != 0:
            raise OracleError(1, "query_knn: k out of range")
        return idx, dsq

    def nearest(self, X, Q):
        X = _f64(X)
        Q = _f64(Q).reshape(-1, X.shape[1])
        return np.array([self.L.fmgp_oracle_nearest(_p(X), X.shape[0], X.shape[1], _p(Q[i]))
                         for i in range(Q.shape[0])], dtype=np.int32)

    def cov_self(self, xs, kind, sigma, rho, nu, tau):
        xs = _f64(xs)
        K = np.empty((xs.shape[0], xs.shape[0]))
        self.L.fmgp_oracle_cov_self(_p(xs), xs.shape[0], xs.shape[1], kind, sigma, rho, nu, tau, _p(K))
        return K

    def precompute_rows(self, X, Y, kind, sigma, rho, nu, tau, k, rows=None, threads=1):
        X = _f64(X)
        Y = _f64(Y)
        Y2 = Y.reshape(Y.shape[0], -1)
        n, d = X.shape
        m = Y2.shape[1]
        rows = np.arange(n, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
        S = np.empty((rows.size, k), dtype=np.int32)
        Cm = np.empty((rows.size, k, m), dtype=np.float64)
        failed = C.c_int64(-1)
        rc = self.L.fmgp_oracle_precompute_rows(_p(X), _p(Y2), n, d, m, kind, sigma, rho, nu, tau, k, _p(rows),
                                                rows.size, threads, _p(S), _p(Cm), C.byref(failed))
        if rc == 1:
            raise OracleError(1, "precompute: k out of range")
        if rc == 2:
            raise OracleError(2, f"Cholesky factorization failed in precompute row {failed.value} after jitter "
                                 "escalation up to 1e-6", failed.value)
        return S, Cm

    def predict(self, X, S, Cm, kind, sigma, rho, nu, tau, mean_offset, Z, threads=1):
        X = _f64(X)
        Z = _f64(Z)
        S = np.ascontiguousarray(S, dtype=np.int32)
        n, d = X.shape
        k = S.shape[1]
        C3 = _f64(Cm).reshape(n, k, -1)
        m = C3.shape[2]
        out = np.empty((Z.shape[0], m))
        nn = np.empty(Z.shape[0], dtype=np.int32)
        mo = float(np.asarray(mean_offset).reshape(-1)[0]) if m == 1 else None
        if m == 1:
            self.L.fmgp_oracle_predict(_p(X), _p(S), _p(C3), n, d, k, 1, kind, sigma, rho, nu, tau, mo, _p(Z),
                                       Z.shape[0], threads, _p(out), _p(nn))
        else:
            mos = np.asarray(mean_offset, dtype=np.float64).reshape(-1)
            for c in range(m):
                Cc = np.ascontiguousarray(C3[:, :, c])
                oc = np.empty((Z.shape[0], 1))
                self.L.fmgp_oracle_predict(_p(X), _p(S), _p(Cc), n, d, k, 1, kind, sigma, rho, nu, tau,
                                           float(mos[c]), _p(Z), Z.shape[0], threads, _p(oc), _p(nn))
                out[:, c] = oc[:, 0]
        return out, nn


class Reference:
    """The reference's own TUs (oracle/_ref), through its public C++ API."""

    kind = "reference"

    def __init__(self, path: Path = REF_PATH):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing; run make -C oracle ref (needs /root/reference)")
        L = C.CDLL(str(path))
        L.fmgp_ref_last_error.restype = C.c_char_p
        L.fmgp_ref_kernel_value.restype = C.c_double
        L.fmgp_ref_kernel_value.argtypes = [C.c_double, C.c_int] + [C.c_double] * 4
        L.fmgp_ref_precompute.restype = C.c_int
        L.fmgp_ref_precompute.argtypes = ([_V, _V, C.c_int64, C.c_int, C.c_int] + [C.c_double] * 4 +
                                          [C.c_int, C.c_int, _V, _V])
        L.fmgp_ref_precompute_rows.restype = C.c_int
        L.fmgp_ref_precompute_rows.argtypes = ([_V, _V, C.c_int64, C.c_int, C.c_int, C.c_int] + [C.c_double] * 4 +
                                               [C.c_int, _V, C.c_int64, C.c_int, _V, _V])
        L.fmgp_ref_predict.restype = C.c_int
        L.fmgp_ref_predict.argtypes = ([_V, _V, _V, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int] +
                                       [C.c_double] * 5 + [_V, C.c_int64, C.c_int, _V, _V])
        L.fmgp_ref_query_knn.restype = C.c_int
        L.fmgp_ref_query_knn.argtypes = [_V, C.c_int64, C.c_int, _V, C.c_int, C.c_int, _V, _V]
        L.fmgp_ref_nearest.restype = C.c_int
        L.fmgp_ref_nearest.argtypes = [_V, C.c_int64, C.c_int, _V, C.c_int64, _V]
        L.fmgp_ref_local_predictions.restype = C.c_int
        L.fmgp_ref_local_predictions.argtypes = ([_V, _V, C.c_int64, C.c_int, _V, _V, _V, C.c_int64, C.c_int,
                                                  C.c_int] + [C.c_double] * 4 + [_V])
        L.fmgp_ref_loocv_loss.restype = C.c_int
        L.fmgp_ref_loocv_loss.argtypes = ([_V, _V, C.c_int64, C.c_int, _V, _V, _V, C.c_int64, C.c_int, C.c_int] +
                                          [C.c_double] * 4 + [_V])
        L.fmgp_ref_train.restype = C.c_int
        L.fmgp_ref_train.argtypes = ([_V, _V, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int] +
                                     [C.c_double] * 4 + [_V, _V, C.c_int, C.c_double, _V, _V, _V, _V, _V])
        L.fmgp_ref_muygps_predict.restype = C.c_int
        L.fmgp_ref_muygps_predict.argtypes = ([_V, _V, C.c_int64, C.c_int, C.c_double, _V, C.c_int64, C.c_int,
                                               C.c_int] + [C.c_double] * 4 + [_V])
        L.fmgp_ref_predict_session.restype = C.c_void_p
        L.fmgp_ref_predict_session.argtypes = ([_V, _V, _V, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int] +
                                               [C.c_double] * 5)
        L.fmgp_ref_predict_run.restype = C.c_int
        L.fmgp_ref_predict_run.argtypes = [_V, _V, C.c_int64, C.c_int, _V]
        L.fmgp_ref_predict_free.restype = None
        L.fmgp_ref_predict_free.argtypes = [_V]
        L.fmgp_ref_save_model.restype = C.c_int
        L.fmgp_ref_save_model.argtypes = ([_V, _V, _V, C.c_int64, C.c_int, C.c_int, C.c_int] + [C.c_double] * 5 +
                                          [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_char_p])
        L.fmgp_ref_load_model.restype = C.c_int
        L.fmgp_ref_load_model.argtypes = [C.c_char_p, _V, C.c_int64, _V, _V]
        L.fmgp_ref_resave.restype = C.c_int
        L.fmgp_ref_resave.argtypes = [C.c_char_p, C.c_char_p]
        self.L = L

    def predict_session(self, X, S, Cm, kind, sigma, rho, nu, tau, mean_offset):
        """A reference model built once; .run(Z, threads) times fast_predict_batch / fast_predict_one."""
        return _RefPredictSession(self, X, S, Cm, kind, sigma, rho, nu, tau, mean_offset)

    def save_model(self, path, X, S, Cm, kind, sigma, rho, nu, tau, mean_offset, mode=0, max_degree=16,
                   build_beam=100, seed=0):
        X = _f64(X)
        S = np.ascontiguousarray(S, dtype=np.int32)
        Cm = _f64(Cm).reshape(S.shape)
        self._check(self.L.fmgp_ref_save_model(_p(X), _p(S), _p(Cm), X.shape[0], X.shape[1], S.shape[1], kind, sigma,
                                               rho, nu, tau, float(mean_offset), mode, max_degree, build_beam, seed,
                                               str(path).encode()))

    def resave(self, path_in, path_out):
        """load_model then save_model through the reference."""
        self._check(self.L.fmgp_ref_resave(str(path_in).encode(), str(path_out).encode()))

    def load_model_predict(self, path, Z):
        """load_model, then fast_predict_batch(Z): (dims (n, d, k, mode), predictions)."""
        Z = _f64(Z)
        dims = np.zeros(4, dtype=np.int64)
        out = np.empty(Z.shape[0])
        self._check(self.L.fmgp_ref_load_model(str(path).encode(), _p(Z), Z.shape[0], _p(dims), _p(out)))
        return dims, out

    def local_predictions(self, X, Y, batch, nbr, dist, kind, sigma, rho, nu, tau):
        X = _f64(X)
        Y = _f64(Y).reshape(-1)
        bi = np.ascontiguousarray(batch, dtype=np.int32)
        nbr = np.ascontiguousarray(nbr, dtype=np.int32)
        dist = _f64(dist)
        out = np.empty(bi.size, dtype=np.float64)
        self._check(self.L.fmgp_ref_local_predictions(_p(X), _p(Y), X.shape[0], X.shape[1], _p(bi), _p(nbr),
                                                      _p(dist), bi.size, nbr.shape[1], kind, sigma, rho, nu, tau,
                                                      _p(out)))
        return out

    def loocv_loss(self, X, Y, batch, nbr, dist, kind, sigma, rho, nu, tau):
        X = _f64(X)
        Y = _f64(Y).reshape(-1)
        bi = np.ascontiguousarray(batch, dtype=np.int32)
        nbr = np.ascontiguousarray(nbr, dtype=np.int32)
        dist = _f64(dist)
        loss = C.c_double(0.0)
        self._check(self.L.fmgp_ref_loocv_loss(_p(X), _p(Y), X.shape[0], X.shape[1], _p(bi), _p(nbr), _p(dist),
                                               bi.size, nbr.shape[1], kind, sigma, rho, nu, tau, C.byref(loss)))
        return loss.value

    def train(self, X, Y, b, seed, k, kind, sigma, rho, nu, tau, bounds, max_evals=200, tol=1e-8):
        """bounds: dict with optional 'rho'/'nu'/'tau' -> (lo, hi). Returns
        ((sigma, rho, nu, tau), final_loss, evaluations, improved, batch indices)."""
        X = _f64(X)
        Y = _f64(Y).reshape(-1)
        has = np.array([int(n in bounds) for n in ("rho", "nu", "tau")], dtype=np.int32)
        bnd = np.array([v for n in ("rho", "nu", "tau") for v in bounds.get(n, (0.0, 0.0))], dtype=np.float64)
        theta = np.empty(4, dtype=np.float64)
        loss = C.c_double(0.0)
        ev = C.c_int32(0)
        imp = C.c_int32(0)
        batch = np.empty(b, dtype=np.int32)
        self._check(self.L.fmgp_ref_train(_p(X), _p(Y), X.shape[0], X.shape[1], b, seed, k, kind, sigma, rho, nu,
                                          tau, _p(has), _p(bnd), max_evals, tol, _p(theta), C.byref(loss),
                                          C.byref(ev), C.byref(imp), _p(batch)))
        return tuple(theta.tolist()), loss.value, ev.value, bool(imp.value), batch.tolist()

    def muygps_predict(self, X, Y, mean_offset, Z, k, kind, sigma, rho, nu, tau):
        X = _f64(X)
        Y = _f64(Y).reshape(-1)
        Z = _f64(Z)
        out = np.empty(Z.shape[0], dtype=np.float64)
        self._check(self.L.fmgp_ref_muygps_predict(_p(X), _p(Y), X.shape[0], X.shape[1], mean_offset, _p(Z),
                                                   Z.shape[0], k, kind, sigma, rho, nu, tau, _p(out)))
        return out

    def _check(self, rc):
        if rc != 0:
            msg = self.L.fmgp_ref_last_error().decode()
            row = -1
            if rc == 2 and "precompute row " in msg:
                row = int(msg.split("precompute row ")[1].split()[0])
            raise OracleError(rc, msg, row)

    def kernel_value(self, dist, kind, sigma, rho, nu, tau):
        return self.L.fmgp_ref_kernel_value(dist, kind, sigma, rho, nu, tau)

    def precompute(self, X, Y, kind, sigma, rho, nu, tau, k, threads=1):
        X = _f64(X)
        Y = _f64(Y).reshape(-1)
        n, d = X.shape
        S = np.empty((n, k), dtype=np.int32)
        Cm = np.empty((n, k), dtype=np.float64)
        self._check(self.L.fmgp_ref_precompute(_p(X), _p(Y), n, d, kind, sigma, rho, nu, tau, k, threads, _p(S),
                                               _p(Cm)))
        return S, Cm

    def precompute_rows(self, X, Y, kind, sigma, rho, nu, tau, k, rows=None, threads=1):
        X = _f64(X)
        Y2 = _f64(Y).reshape(X.shape[0], -1)
        n, d = X.shape
        m = Y2.shape[1]
        rows = np.arange(n, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
        S = np.empty((rows.size, k), dtype=np.int32)
        Cm = np.empty((rows.size, k, m), dtype=np.float64)
        self._check(self.L.fmgp_ref_precompute_rows(_p(X), _p(Y2), n, d, m, kind, sigma, rho, nu, tau, k,
                                                    _p(rows), rows.size, threads, _p(S), _p(Cm)))
        return S, Cm

    def predict(self, X, S, Cm, kind, sigma, rho, nu, tau, mean_offset, Z, threads=1):
        X = _f64(X)
        Z = _f64(Z)
        S = np.ascontiguousarray(S, dtype=np.int32)
        n, d = X.shape
        k = S.shape[1]
        C3 = _f64(Cm).reshape(n, k, -1)
        m = C3.shape[2]
        mos = np.broadcast_to(np.asarray(mean_offset, dtype=np.float64).reshape(-1), (m,))
        out = np.empty((Z.shape[0], m))
        nn = np.empty(Z.shape[0], dtype=np.int32)
        for c in range(m):  # one reference model per output; mean offset is per model
            Cc = np.ascontiguousarray(C3[:, :, c])
            oc = np.empty(Z.shape[0])
            self._check(self.L.fmgp_ref_predict(_p(X), _p(S), _p(Cc), n, d, k, 1, kind, sigma, rho, nu, tau,
                                                float(mos[c]), _p(Z), Z.shape[0], threads, _p(oc), _p(nn)))
            out[:, c] = oc
        return out, nn

    def query_knn(self, X, q, k, exclude=-1):
        X = _f64(X)
        q = _f64(q)
        idx = np.empty(k, dtype=np.int32)
        dist = np.empty(k, dtype=np.float64)
        self._check(self.L.fmgp_ref_query_knn(_p(X), X.shape[0], X.shape[1], _p(q), k, exclude, _p(idx), _p(dist)))
        return idx, dist

    def nearest(self, X, Q):
        X = _f64(X)
        Q = _f64(Q).reshape(-1, X.shape[1])
        out = np.empty(Q.shape[0], dtype=np.int32)
        self._check(self.L.fmgp_ref_nearest(_p(X), X.shape[0], X.shape[1], _p(Q), Q.shape[0], _p(out)))
        return out


class _RefPredictSession:
    def __init__(self, ref, X, S, Cm, kind, sigma, rho, nu, tau, mean_offset):
        X = _f64(X)
        S = np.ascontiguousarray(S, dtype=np.int32)
        n, k = S.shape
        C3 = _f64(Cm).reshape(n, k, -1)
        self.ref, self.d, self.m = ref, X.shape[1], C3.shape[2]
        self.h = ref.L.fmgp_ref_predict_session(_p(X), _p(S), _p(C3), n, X.shape[1], k, self.m, kind, sigma, rho, nu,
                                                tau, float(np.asarray(mean_offset).reshape(-1)[0]))
        if not self.h:
            raise OracleError(3, ref.L.fmgp_ref_last_error().decode())

    def run(self, Z, threads=1):
        Z = _f64(Z).reshape(-1, self.d)
        out = np.empty((Z.shape[0], self.m))
        self.ref._check(self.ref.L.fmgp_ref_predict_run(self.h, _p(Z), Z.shape[0], threads, _p(out)))
        return out

    def close(self):
        if self.h:
            self.ref.L.fmgp_ref_predict_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


def best_available():
    """oracle/_ref when it was built (reference-compiled), else the C port."""
    if REF_PATH.exists():
        return Reference()
    return Port()


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
