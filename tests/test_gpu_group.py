"""GPU: the multi-GPU precompute of the C ABI (csrc/group.cu) on one B200.

The block-cyclic layout and the in-place exchanges are exercised with device
groups that list the same GPU several times (peer-copy backend: each member
is a separate replica with its own buffers and host thread) and with a
one-rank NCCL communicator (FMGP_GROUP_BACKEND=nccl), so both exchange
backends run; results must be bit-identical to the single-GPU fmgp_precompute
(rows are independent), and the model the group returns (one replica per
member) must predict exactly what a single-device model predicts.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _single(N, ds, k, kp):
    n, d = ds.X.shape
    m = ds.Y.shape[1]
    S = np.empty((n, k), dtype=np.int32)
    Cm = np.empty((n, k, m))
    f = C.c_int64(-1)
    N.check(N.LIB.fmgp_precompute(_p(ds.X), _p(ds.Y), n, d, m, C.byref(kp), k, _p(S), _p(Cm), C.byref(f)), f.value)
    return S, Cm


def _group_run(N, devices, ds, k, kp, with_model=True):
    n, d = ds.X.shape
    m = ds.Y.shape[1]
    g = C.c_void_p()
    devs = (C.c_int32 * len(devices))(*devices)
    N.check(N.LIB.fmgp_group_create_devices(devs, len(devices), C.byref(g)))
    try:
        info = (C.c_int32(), C.c_int32(), C.c_int32())
        N.check(N.LIB.fmgp_group_info(g, *[C.byref(x) for x in info]))
        S = np.full((n, k), -7, dtype=np.int32)
        Cm = np.full((n, k, m), np.nan)
        mo = np.ascontiguousarray(np.asarray(ds.mean_offset, dtype=np.float64).reshape(-1))
        f = C.c_int64(-1)
        model = C.c_void_p()
        N.check(N.LIB.fmgp_group_precompute(g, _p(ds.X), _p(ds.Y), n, d, m, C.byref(kp), k, _p(mo), _p(S), _p(Cm),
                                            C.byref(f), C.byref(model) if with_model else None), f.value)
        return S, Cm, model, [x.value for x in info]
    finally:
        N.LIB.fmgp_group_destroy(g)


@pytest.mark.parametrize("cfg,n,nt,devices,backend", [
    (2, 200_001, 20_000, [0, 0], "peer"),
    (5, 300_007, 30_000, [0, 0, 0], "peer"),
    (5, 100_003, 10_000, [0], "nccl"),
    (3, 3_001, 500, [0, 0], "peer"),
])
def test_device_group_is_bit_identical_to_one_gpu(fm, monkeypatch, cfg, n, nt, devices, backend):
    from paper_2205_10879_b200 import _native as N, datagen
    monkeypatch.setenv("FMGP_GROUP_BACKEND", backend)
    ds = datagen.generate(cfg, n, nt)
    i = ds.info
    kp = N.KernelParamsC(i.kind, i.sigma, i.rho, i.nu, i.tau)
    S1, C1 = _single(N, ds, i.k, kp)
    S2, C2, model, (nranks, members, be) = _group_run(N, devices, ds, i.k, kp)
    try:
        assert nranks == len(devices) and members == len(devices)
        assert be == (1 if backend == "nccl" else 2)
        assert np.array_equal(S1, S2)
        assert np.array_equal(C1, C2)  # same kernels per row: bit-identical, not just within tolerance
        assert N.LIB.fmgp_model_replicas(model) == len(devices)
        # the group's model (one replica per member, test points split over them)
        out_g = np.empty((nt, i.m))
        nn_g = np.empty(nt, dtype=np.int32)
        N.check(N.LIB.fmgp_model_predict(model, _p(ds.Z), nt, _p(out_g), _p(nn_g)))
        single = C.c_void_p()
        mo = np.ascontiguousarray(np.asarray(ds.mean_offset, dtype=np.float64).reshape(-1))
        N.check(N.LIB.fmgp_model_create(_p(ds.X), _p(S1), _p(C1), n, i.d, i.k, i.m, C.byref(kp), _p(mo), -1,
                                        C.byref(single)))
        out_1 = np.empty((nt, i.m))
        nn_1 = np.empty(nt, dtype=np.int32)
        N.check(N.LIB.fmgp_model_predict(single, _p(ds.Z), nt, _p(out_1), _p(nn_1)))
        N.LIB.fmgp_model_destroy(single)
        assert np.array_equal(nn_g, nn_1) and np.array_equal(out_g, out_1)
    finally:
        N.LIB.fmgp_model_destroy(model)


def test_rank_group_device_path_matches_one_gpu(fm):
    # the bench's value path: a one-rank group, device buffers, stream-ordered
    import torch
    from paper_2205_10879_b200 import _native as N, datagen
    ds = datagen.generate(5, 200_000, 1000)
    i = ds.info
    n, d, k, m = ds.X.shape[0], i.d, i.k, i.m
    kp = N.KernelParamsC(i.kind, i.sigma, i.rho, i.nu, i.tau)
    g = C.c_void_p()
    N.check(N.LIB.fmgp_group_create_rank(None, 1, 0, 0, C.byref(g)))
    X = torch.from_numpy(ds.X).cuda()
    Y = torch.from_numpy(ds.Y).cuda()
    S = torch.empty((n, k), dtype=torch.int32, device="cuda")
    Cm = torch.empty((n, k, m), dtype=torch.float64, device="cuda")
    f = C.c_int64(-1)
    s = torch.cuda.current_stream()
    N.check(N.LIB.fmgp_group_precompute_device(g, C.c_void_p(X.data_ptr()), C.c_void_p(Y.data_ptr()), n, d, m,
                                               C.byref(kp), k, C.c_void_p(S.data_ptr()), C.c_void_p(Cm.data_ptr()),
                                               C.byref(f), C.c_void_p(s.cuda_stream)), f.value)
    N.LIB.fmgp_group_destroy(g)
    S1, C1 = _single(N, ds, k, kp)
    assert np.array_equal(S.cpu().numpy(), S1) and np.array_equal(Cm.cpu().numpy(), C1)
    # the wrapped device model predicts what the host model predicts
    mo = np.ascontiguousarray(np.asarray(ds.mean_offset, dtype=np.float64).reshape(-1))
    h = C.c_void_p()
    N.check(N.LIB.fmgp_model_wrap_device(C.c_void_p(X.data_ptr()), C.c_void_p(S.data_ptr()),
                                         C.c_void_p(Cm.data_ptr()), n, d, k, m, C.byref(kp), _p(mo), C.byref(h)))
    Z = torch.from_numpy(ds.Z).cuda()
    out = torch.empty((ds.Z.shape[0], m), dtype=torch.float64, device="cuda")
    nn = torch.empty(ds.Z.shape[0], dtype=torch.int32, device="cuda")
    N.check(N.LIB.fmgp_model_predict_device(h, C.c_void_p(Z.data_ptr()), ds.Z.shape[0], C.c_void_p(out.data_ptr()),
                                            C.c_void_p(nn.data_ptr()), C.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    N.LIB.fmgp_model_destroy(h)
    out_1 = np.empty((ds.Z.shape[0], m))
    nn_1 = np.empty(ds.Z.shape[0], dtype=np.int32)
    N.check(N.LIB.fmgp_predict(_p(ds.X), _p(S1), _p(C1), n, d, k, m, C.byref(kp), _p(mo), _p(ds.Z), ds.Z.shape[0],
                               _p(out_1), _p(nn_1)))
    assert np.array_equal(nn.cpu().numpy(), nn_1) and np.array_equal(out.cpu().numpy(), out_1)


def test_group_errors_match_single_gpu(fm, monkeypatch):
    from paper_2205_10879_b200 import _native as N, datagen
    monkeypatch.setenv("FMGP_GROUP_BACKEND", "peer")
    ds = datagen.generate(1, 3000, 10)
    i = ds.info
    kp = N.KernelParamsC(i.kind, i.sigma, i.rho, i.nu, i.tau)
    X = ds.X.copy()
    X[1234, 1] = np.nan
    n, d = X.shape
    g = C.c_void_p()
    devs = (C.c_int32 * 2)(0, 0)
    N.check(N.LIB.fmgp_group_create_devices(devs, 2, C.byref(g)))
    S = np.empty((n, i.k), dtype=np.int32)
    Cm = np.empty((n, i.k, 1))
    f = C.c_int64(-1)
    rc = N.LIB.fmgp_group_precompute(g, _p(X), _p(ds.Y), n, d, 1, C.byref(kp), i.k, None, _p(S), _p(Cm),
                                     C.byref(f), None)
    assert rc == N.FMGP_EINVAL and "non-finite" in N.LIB.fmgp_last_error().decode()
    # a NumericError row: a duplicated point with tau = 0 and a huge sigma fails every jitter rung;
    # the group names the lowest failing row, like the single-GPU call
    X2 = ds.X.copy()
    X2[2000] = X2[17]
    X2[2500] = X2[17]
    kp0 = N.KernelParamsC(i.kind, 1e4, i.rho, i.nu, 0.0)
    f1, f2 = C.c_int64(-1), C.c_int64(-1)
    rc1 = N.LIB.fmgp_precompute(_p(X2), _p(ds.Y), n, d, 1, C.byref(kp0), i.k, _p(S), _p(Cm), C.byref(f1))
    rc2 = N.LIB.fmgp_group_precompute(g, _p(X2), _p(ds.Y), n, d, 1, C.byref(kp0), i.k, None, _p(S), _p(Cm),
                                      C.byref(f2), None)
    N.LIB.fmgp_group_destroy(g)
    assert rc1 == rc2
    if rc1 == N.FMGP_ENUMERIC:
        assert f1.value == f2.value
