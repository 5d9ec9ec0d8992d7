"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle.

Neighbour indices bit-exact; coefficients ||dC_i||/||C_i|| <= 1e-9 and
posterior means |a-b|/(1+|b|) <= 1e-9 (north_star tolerance), on seeded
inputs from the BASELINE configs at sizes the oracle finishes in seconds.
"""
import numpy as np
import pytest

from helpers import C_TOL, MEAN_TOL, kparams, mean_rel_err, row_rel_err

pytestmark = pytest.mark.gpu


def _fit(fm, info):
    return fm.FittedParams(fm.KernelParams(info.sigma, info.rho, info.nu, info.tau), fm.KernelKind(info.kind))


def _run(fm, X, Y, info, k, Z=None, mean_offset=0.0):
    train = fm.TrainingSet(X, Y if Y.shape[1] > 1 else Y[:, 0], mean_offset)
    index = fm.NeighborIndex.build(X, fm.IndexMode.Exact)
    model = fm.precompute(train, _fit(fm, info), index, k)
    pred = None if Z is None else fm.fast_predict_batch(model, Z)
    return model, pred


@pytest.mark.parametrize("cfg,n,nt", [(1, 10000, 2000), (2, 4000, 500), (3, 800, 100), (4, 1500, 200),
                                      (5, 4000, 500)])
def test_precompute_and_predict_match_oracle(fm, port, cfg, n, nt):
    from paper_2205_10879_b200 import datagen
    ds = datagen.generate(cfg, n, nt)
    info = ds.info
    k = info.k
    model, pred = _run(fm, ds.X, ds.Y, info, k, ds.Z, ds.mean_offset if info.m > 1 else float(ds.mean_offset[0]))
    rows = np.arange(n) if n <= 4000 else np.arange(0, n, 3)
    S_o, C_o = port.precompute_rows(ds.X, ds.Y, *kparams(info), k, rows, threads=8)
    S = model.S[rows]
    assert S.dtype == np.int32
    assert np.array_equal(S, S_o), f"neighbour table differs in {np.sum(np.any(S != S_o, axis=1))} rows"
    Cg = model.C.reshape(n, k, -1)[rows]
    err = row_rel_err(Cg, C_o)
    assert err.max() <= C_TOL, err.max()
    out_o, nn_o = port.predict(ds.X, model.S, model.C.reshape(n, k, -1), *kparams(info), ds.mean_offset, ds.Z,
                               threads=8)
    assert mean_rel_err(pred, out_o.reshape(pred.shape)).max() <= MEAN_TOL
    nn = model.index.nearest_batch(ds.Z)
    assert np.array_equal(nn, nn_o)
    # the fused predict path's own 1-NN (fmgp_predict nn_out) is the reference's too
    import ctypes as C
    from paper_2205_10879_b200 import _native as N
    k_, m_ = model.S.shape[1], info.m
    out2 = np.empty((ds.Z.shape[0], m_))
    nn2 = np.empty(ds.Z.shape[0], dtype=np.int32)
    kp = model.params.c(model.kind)
    mo = np.ascontiguousarray(np.broadcast_to(np.asarray(ds.mean_offset, dtype=np.float64), (m_,)))
    Cc = np.ascontiguousarray(model.C.reshape(n, k_, m_))
    N.check(N.LIB.fmgp_predict(ds.X.ctypes.data, model.S.ctypes.data, Cc.ctypes.data, n, info.d, k_, m_,
                               C.byref(kp), mo.ctypes.data, ds.Z.ctypes.data, ds.Z.shape[0], out2.ctypes.data,
                               nn2.ctypes.data))
    assert np.array_equal(nn2, nn_o)
    assert mean_rel_err(out2, out_o).max() <= MEAN_TOL


def test_ties_resolve_by_ascending_index(fm):
    # test_nn_index.cpp:57-70: four copies of one point plus fillers.
    X = np.array([[0, 0], [0, 0], [0, 0], [0, 0], [5, 5], [6, 6]], dtype=np.float64)
    index = fm.NeighborIndex.build(X, fm.IndexMode.Exact)
    nl = index.query_knn([0.1, 0.0], 4)
    assert nl.indices == [0, 1, 2, 3]
    assert index.nearest_training_point([0.1, 0.0]) == 0


def test_exclusion_is_by_index_identity(fm):
    # test_nn_index.cpp:72-84
    X = np.array([[1.0], [1.0], [2.0], [3.0]])
    index = fm.NeighborIndex.build(X, fm.IndexMode.Exact)
    nl = index.query_knn(X[0], 3, 0)
    assert 0 not in nl.indices
    assert nl.indices[0] == 1
    assert nl.distances[0] == 0.0


def test_exact_mode_matches_brute_force_sort(fm, port):
    # test_nn_index.cpp:40-55 (300 pts, d=5, k=12, 25 queries) + an independent sort.
    rng = np.random.default_rng(1)
    X = rng.random((300, 5))
    Q = rng.random((25, 5))
    index = fm.NeighborIndex.build(X, fm.IndexMode.Exact)
    idx, dist = index.query_knn_batch(Q, 12)
    for r in range(25):
        dsq = np.array([port.L.fmgp_oracle_dist_sq(Q[r].ctypes.data, X[i].ctypes.data, 5) for i in range(300)])
        order = sorted(range(300), key=lambda i: (dsq[i], i))[:12]
        assert idx[r].tolist() == order
        assert np.all(np.diff(dist[r]) >= 0)


def test_one_training_point_scalar_ratio(fm):
    # test_fast_predict.cpp:46-59
    X = np.array([[0.3, 0.4]])
    train = fm.TrainingSet(X, np.array([2.0]), 0.5)
    p = fm.KernelParams(1.0, 0.7, 0.5, 0.0)
    model = fm.precompute(train, fm.FittedParams(p, fm.KernelKind.Matern), fm.NeighborIndex.build(X), 1)
    z = np.array([0.6, 0.8])
    d = np.linalg.norm(z - X[0])
    expected = np.exp(-d / 0.7) * 2.0 + 0.5
    got = fm.fast_predict_one(model, z)
    assert abs(got - expected) < 1e-12 * (1 + abs(expected))


def test_rows_solve_their_local_systems(fm, port):
    # test_fast_predict.cpp:61-79 (n=120, d=3, k=12, Matern 1.5, tau=1e-6): residual <= 1e-8.
    from paper_2205_10879_b200 import datagen
    X, Y, mo = datagen.random_set(120, 3, 1)
    p = fm.KernelParams(1.2, 0.5, 1.5, 1e-6)
    model = fm.precompute(fm.TrainingSet(X, Y, mo), fm.FittedParams(p, fm.KernelKind.Matern),
                          fm.NeighborIndex.build(X), 12)
    for i in range(120):
        assert model.S[i, 0] == i
        xs = X[model.S[i]]
        K = port.cov_self(xs, 0, 1.2, 0.5, 1.5, 1e-6)
        res = K @ model.C[i] - Y[model.S[i]]
        assert np.abs(res).max() <= 1e-8


def test_k_equals_n_recovers_dense_posterior(fm):
    # test_fast_predict.cpp:81-93: RBF, k = n = 50. As in the reference test the
    # dense GP uses the same implementation's kernel and SPD solve (here the
    # GPU cov_matrix / solve_spd); cond(K) ~ 7e11, so an independent LU solve
    # would itself sit at ~6e-9 from the reference (measured with oracle/_ref).
    from paper_2205_10879_b200 import datagen
    X, Y, mo = datagen.random_set(50, 2, 2)
    Z, _, _ = datagen.random_set(25, 2, 3)
    p = fm.KernelParams(1.0, 0.4, 2.5, 1e-6)
    fit = fm.FittedParams(p, fm.KernelKind.RBF)
    model = fm.precompute(fm.TrainingSet(X, Y, mo), fit, fm.NeighborIndex.build(X), 50)
    fast = fm.fast_predict_batch(model, Z)
    Kxx = fm.cov_matrix_self(X, fm.KernelKind.RBF, p)
    Kzx = fm.cov_matrix(Z, X, fm.KernelKind.RBF, p)
    dense = Kzx @ fm.solve_spd(Kxx, Y) + mo
    err = np.abs(fast - dense) / (1 + np.abs(dense))
    assert err.max() <= 1e-8, err.max()


def test_linear_in_y_and_sigma_invariant(fm):
    # test_fast_predict.cpp:107-134
    from paper_2205_10879_b200 import datagen
    X, Y, mo = datagen.random_set(150, 3, 5)
    Z, _, _ = datagen.random_set(20, 3, 6)
    p = fm.KernelParams(1.0, 0.5, 2.5, 1e-6)
    idx = fm.NeighborIndex.build(X)
    fit = fm.FittedParams(p, fm.KernelKind.Matern)
    a = fm.fast_predict_batch(fm.precompute(fm.TrainingSet(X, Y, mo), fit, idx, 15), Z)
    b = fm.fast_predict_batch(fm.precompute(fm.TrainingSet(X, -2.0 * Y, 0.0), fit, idx, 15), Z)
    c = fm.fast_predict_batch(fm.precompute(fm.TrainingSet(X, Y, 0.0), fit, idx, 15), Z)
    assert np.abs(b + 2.0 * c).max() <= 1e-10
    s = fm.fast_predict_batch(fm.precompute(fm.TrainingSet(X, Y, mo), fm.FittedParams(p.with_sigma(10.0),
                                                                                        fm.KernelKind.Matern),
                                            idx, 15), Z)
    assert np.abs(s - a).max() <= 1e-10


@pytest.mark.parametrize("k,d", [(8, 2), (30, 2), (50, 2), (50, 3), (100, 2), (100, 40), (30, 40)])
def test_numeric_error_names_lowest_failing_row(fm, port, k, d):
    # Exact duplicates with tau = 0 give an exactly singular block; with sigma = 1e6
    # the jitter rungs (<= 1e-6) are below one ulp of the diagonal, so the ladder
    # is exhausted -> NumericError naming the lowest failing row (linalg.cpp:28-30,
    # fast_predict.cpp:105; threads = 1 semantics). k = 30/50 run the register
    # solve, k = 100 the CTA solve, k = 8 the scalar one.
    from oracle.oracle import OracleError
    n = 2 * k + 40
    X = np.zeros((n, d))
    X[:, 0] = np.arange(n) * 10.0
    X[k + 21] = X[k + 20]
    Y = np.arange(n, dtype=np.float64)
    p = fm.KernelParams(1e6, 1.0, 2.5, 0.0)
    with pytest.raises(OracleError) as eo:
        port.precompute_rows(X, Y, 1, 1e6, 1.0, 2.5, 0.0, k)
    with pytest.raises(fm.NumericError) as ei:
        fm.precompute(fm.TrainingSet(X, Y, 0.0), fm.FittedParams(p, fm.KernelKind.RBF), fm.NeighborIndex.build(X), k)
    assert ei.value.failed_row == eo.value.failed_row
    assert str(ei.value) == (f"Cholesky factorization failed in precompute row {eo.value.failed_row} "
                             "after jitter escalation up to 1e-6")


@pytest.mark.parametrize("k", [2, 3, 7, 8, 9, 17, 33, 64, 65, 100, 127, 128, 129, 170])
@pytest.mark.parametrize("m", [1, 3, 10])
def test_solve_widths_match_oracle(fm, port, k, m):
    # every tile/row-slot width class of the fused solve (DMMA tiles of 8, warp
    # row slots of 32, the CTA fallback above 128) and multi-output RHS blocks
    rng = np.random.default_rng(1000 * k + m)
    n = 400
    X = rng.random((n, 3))
    Y = rng.standard_normal((n, m))
    p = fm.KernelParams(1.3, 0.6, 2.5, 0.05)
    model = fm.precompute(fm.TrainingSet(X, Y if m > 1 else Y[:, 0], 0.0), fm.FittedParams(p, fm.KernelKind.Matern),
                          fm.NeighborIndex.build(X), k)
    rows = np.arange(0, n, 7)
    S_o, C_o = port.precompute_rows(X, Y, 0, 1.3, 0.6, 2.5, 0.05, k, rows)
    assert np.array_equal(model.S[rows], S_o)
    err = row_rel_err(model.C.reshape(n, k, -1)[rows], C_o)
    assert err.max() <= C_TOL, err.max()


def test_host_row_shards_equal_full_precompute(fm):
    # fmgp_precompute_rows (one process per GPU, host buffers): shards are
    # bit-identical to the corresponding rows of the full precompute, for any split
    import ctypes as C
    from paper_2205_10879_b200 import _native as N, datagen
    ds = datagen.generate(2, 20000, 10)
    i = ds.info
    n, d, k = ds.X.shape[0], ds.X.shape[1], i.k
    p = fm.KernelParams(i.sigma, i.rho, i.nu, i.tau)
    model = fm.precompute(fm.TrainingSet(ds.X, ds.Y, ds.mean_offset), fm.FittedParams(p, fm.KernelKind(i.kind)),
                          fm.NeighborIndex.build(ds.X), k)
    kp = p.c(fm.KernelKind(i.kind))
    for b, e in [(0, 7000), (7000, 13001), (13001, 20000), (5, 6)]:
        S = np.empty((e - b, k), dtype=np.int32)
        Cm = np.empty((e - b, k), dtype=np.float64)
        failed = C.c_int64(-1)
        N.check(N.LIB.fmgp_precompute_rows(ds.X.ctypes.data, ds.Y.ctypes.data, n, d, 1, C.byref(kp), k, b, e,
                                           S.ctypes.data, Cm.ctypes.data, C.byref(failed)), failed.value)
        assert np.array_equal(S, model.S[b:e])
        assert np.array_equal(Cm, model.C[b:e].reshape(e - b, k))


def test_fmgp_devices_split_is_bit_identical(fm, monkeypatch):
    # FMGP_DEVICES: rows split over a device list inside one process (here the
    # same device listed several times, exercising the shard/join logic)
    from paper_2205_10879_b200 import datagen
    ds = datagen.generate(2, 30000, 10)
    i = ds.info
    args = (fm.TrainingSet(ds.X, ds.Y, ds.mean_offset),
            fm.FittedParams(fm.KernelParams(i.sigma, i.rho, i.nu, i.tau), fm.KernelKind(i.kind)),
            fm.NeighborIndex.build(ds.X), i.k)
    monkeypatch.delenv("FMGP_DEVICES", raising=False)
    ref = fm.precompute(*args)
    for devs in ("0,0", "0,0,0", "0"):
        monkeypatch.setenv("FMGP_DEVICES", devs)
        got = fm.precompute(*args)
        assert np.array_equal(got.S, ref.S) and np.array_equal(got.C, ref.C), devs
    # numeric failure: the lowest failing row over all shards (as with one device)
    X = np.zeros((90, 2))
    X[:, 0] = np.arange(90) * 10.0
    X[71] = X[70]
    X[21] = X[20]
    Y = np.arange(90, dtype=np.float64)
    p = fm.KernelParams(1e6, 1.0, 2.5, 0.0)
    monkeypatch.delenv("FMGP_DEVICES", raising=False)
    with pytest.raises(fm.NumericError) as e1:
        fm.precompute(fm.TrainingSet(X, Y, 0.0), fm.FittedParams(p, fm.KernelKind.RBF), fm.NeighborIndex.build(X), 8)
    monkeypatch.setenv("FMGP_DEVICES", "0,0,0")
    with pytest.raises(fm.NumericError) as e3:
        fm.precompute(fm.TrainingSet(X, Y, 0.0), fm.FittedParams(p, fm.KernelKind.RBF), fm.NeighborIndex.build(X), 8)
    assert e1.value.failed_row == e3.value.failed_row and str(e1.value) == str(e3.value)


def test_split_knn_and_chunked_async_solve_equal_precompute_device(fm):
    # the entry points behind bench.py's overlapped multi-GPU step: K1 for a row
    # range, then K2 in chunks with the asynchronous failure word
    import ctypes as C
    import torch
    from paper_2205_10879_b200 import _native as N, datagen
    ds = datagen.generate(5, 40000, 10)
    i = ds.info
    n, d, k = ds.X.shape[0], ds.X.shape[1], i.k
    X = torch.from_numpy(ds.X).cuda()
    Y = torch.from_numpy(ds.Y).cuda()
    fit = fm.FittedParams(fm.KernelParams(i.sigma, i.rho, i.nu, i.tau), fm.KernelKind(i.kind))
    kp = fit.theta_hat.c(fit.kind)
    s = torch.cuda.current_stream()
    b, e = 13000, 29001
    S_ref = torch.empty((e - b, k), dtype=torch.int32, device="cuda")
    C_ref = torch.empty((e - b, k, 1), dtype=torch.float64, device="cuda")
    fm.precompute_device(X, Y, fit, k, b, e, S_ref, C_ref, s)
    S = torch.empty_like(S_ref)
    Cm = torch.full_like(C_ref, float("nan"))
    N.check(N.LIB.fmgp_knn_rows_device(C.c_void_p(X.data_ptr()), n, d, k, b, e, C.c_void_p(S.data_ptr()),
                                       C.c_void_p(s.cuda_stream)))
    fail = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    for lo in range(0, e - b, 5000):
        hi = min(e - b, lo + 5000)
        N.check(N.LIB.fmgp_solve_rows_device(C.c_void_p(X.data_ptr()), C.c_void_p(Y.data_ptr()), n, d, 1,
                                             C.byref(kp), k, C.c_void_p(S[lo:hi].data_ptr()), hi - lo, b + lo,
                                             C.c_void_p(Cm[lo:hi].data_ptr()), C.c_void_p(fail.data_ptr()), None,
                                             C.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    assert int(fail.item()) == -1
    assert torch.equal(S, S_ref) and torch.equal(Cm, C_ref)
    # failures: the word holds the lowest failing global row (exact duplicates, tau = 0, sigma = 1e6)
    Xf = np.zeros((90, 2))
    Xf[:, 0] = np.arange(90) * 10.0
    Xf[71] = Xf[70]
    Xf[21] = Xf[20]
    Xt = torch.from_numpy(Xf).cuda()
    Yt = torch.arange(90, dtype=torch.float64, device="cuda")
    kpf = fm.KernelParams(1e6, 1.0, 2.5, 0.0).c(fm.KernelKind.RBF)
    Sf = torch.empty((90, 8), dtype=torch.int32, device="cuda")
    Cf = torch.empty((90, 8, 1), dtype=torch.float64, device="cuda")
    N.check(N.LIB.fmgp_knn_rows_device(C.c_void_p(Xt.data_ptr()), 90, 2, 8, 0, 90, C.c_void_p(Sf.data_ptr()),
                                       C.c_void_p(s.cuda_stream)))
    fail.fill_(-1)
    for lo in (60, 0, 30):  # out of order: the word keeps the minimum
        N.check(N.LIB.fmgp_solve_rows_device(C.c_void_p(Xt.data_ptr()), C.c_void_p(Yt.data_ptr()), 90, 2, 1,
                                             C.byref(kpf), 8, C.c_void_p(Sf[lo:lo + 30].data_ptr()), 30, lo,
                                             C.c_void_p(Cf[lo:lo + 30].data_ptr()), C.c_void_p(fail.data_ptr()),
                                             None, C.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    with pytest.raises(fm.NumericError) as ei:
        fm.precompute(fm.TrainingSet(Xf, Yt.cpu().numpy(), 0.0),
                      fm.FittedParams(fm.KernelParams(1e6, 1.0, 2.5, 0.0), fm.KernelKind.RBF),
                      fm.NeighborIndex.build(Xf), 8)
    assert int(fail.item()) == ei.value.failed_row


@pytest.mark.parametrize("offset", [0.0, 1e3])
@pytest.mark.parametrize("m", [1, 10])
@pytest.mark.parametrize("d", [32, 100, 784])
def test_gram_build_matches_oracle(fm, port, d, m, offset):
    # k = 30 at d >= 32 builds the neighbourhood matrices from a DMMA Gram
    # matrix (solve_reg.cu build_gram), on sparse cfg3-like rows. Exact
    # duplicates (d^2 = 0 -> nugget, an exactly singular block) are covered by
    # test_numeric_error_names_lowest_failing_row[30-40]: the ladder is only
    # exhausted there if the Gram path detects the zero distance exactly.
    # offset = 1e3: every point moved far from the origin compared with the
    # neighbour spacing (the Gram form then needs the centring on the query
    # point, else d^2 = G_ii + G_jj - 2 G_ij loses ~eps |x|^2 / d^2 digits)
    rng = np.random.default_rng(7 * d + m)
    n, k = 600, 30
    X = rng.random((n, d)) * (rng.random((n, d)) < 0.2) + offset
    Y = rng.standard_normal((n, m))
    p = fm.KernelParams(1.0, 10.0, 0.5, 0.1)
    model = fm.precompute(fm.TrainingSet(X, Y if m > 1 else Y[:, 0], 0.0),
                          fm.FittedParams(p, fm.KernelKind.Matern), fm.NeighborIndex.build(X), k)
    rows = np.arange(0, n, 9)
    S_o, C_o = port.precompute_rows(X, Y, 0, 1.0, 10.0, 0.5, 0.1, k, rows)
    assert np.array_equal(model.S[rows], S_o)
    err = row_rel_err(model.C.reshape(n, k, -1)[rows], C_o)
    assert err.max() <= C_TOL, err.max()
