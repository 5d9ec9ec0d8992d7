"""The host-buffer precompute's stage trace (FMGP_TRACE=1) and
the device-side finiteness check that replaced the host scan of X on that
path (NeighborIndex::build semantics, nn_index.cpp:56-71: non-finite
coordinates -> FMGP_EINVAL / std::domain_error, nothing launched on them)."""
import ctypes as C
import os
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parents[1]


def test_trace_line_reports_monotone_stage_times():
    code = (
        "import numpy as np\n"
        "import paper_2205_10879_b200 as fm\n"
        "rng = np.random.default_rng(0)\n"
        "X = rng.random((20000, 2)); Y = rng.standard_normal(20000)\n"
        "p = fm.KernelParams(1.0, 0.05, 1.5, 0.03)\n"
        "fm.precompute(fm.TrainingSet(X, Y, 0.0), fm.FittedParams(p, fm.KernelKind.Matern),\n"
        "              fm.NeighborIndex.build(X), 50)\n"
    )
    env = dict(os.environ, FMGP_TRACE="1", PYTHONPATH=str(REPO))
    r = subprocess.run([sys.executable, "-c", code], cwd=REPO, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stderr.splitlines() if ln.startswith("[fmgp trace] precompute rows 20000:")]
    assert lines, r.stderr[-2000:]
    done = [float(x) for x in re.findall(r"done ([0-9.]+)", lines[-1])]
    assert len(done) == 4 and all(b >= a for a, b in zip(done, done[1:])), lines[-1]


def test_non_finite_coordinates_rejected_on_device_path():
    from paper_2205_10879_b200 import _native as N
    from paper_2205_10879_b200.api import KernelParams, KernelKind
    rng = np.random.default_rng(1)
    n, k = 5000, 30
    X = rng.random((n, 2))
    X[1234, 1] = np.inf
    Y = rng.standard_normal(n)
    S = np.empty((n, k), dtype=np.int32)
    Cm = np.empty((n, k))
    kp = KernelParams(1.0, 0.05, 1.5, 0.03).c(KernelKind.Matern)
    f = C.c_int64()
    rc = N.LIB.fmgp_precompute(X.ctypes.data, Y.ctypes.data, n, 2, 1, C.byref(kp), k, S.ctypes.data, Cm.ctypes.data,
                               C.byref(f))
    assert rc == N.FMGP_EINVAL and N.LIB.fmgp_last_error() == b"NeighborIndex: non-finite coordinates"


def test_large_host_batch_predict_is_chunked_and_checked_on_device():
    # fmgp_model_predict with >= 65536 test points (d <= 3): chunks on three streams, finiteness of Z
    # checked on the device copy. Same means and 1-NN as the same points sent in small batches
    # (host-checked, one stream); a NaN / inf test point gives FMGP_EINVAL with the reference-side
    # message, and the handle keeps working afterwards (no fault from the bad point).
    import paper_2205_10879_b200 as fm
    from paper_2205_10879_b200 import _native as N
    rng = np.random.default_rng(5)
    n, k, nz = 30000, 30, 600000
    X = rng.random((n, 3))
    Y = rng.standard_normal(n)
    p = fm.KernelParams(1.0, 0.2, 2.5, 0.05)
    model = fm.precompute(fm.TrainingSet(X, Y, 0.25), fm.FittedParams(p, fm.KernelKind.Matern),
                          fm.NeighborIndex.build(X), k)
    Z = rng.random((nz, 3)) * 1.2 - 0.1  # some outside the training box
    h = model.handle()
    out = np.empty(nz)
    nn = np.empty(nz, dtype=np.int32)
    N.check(N.LIB.fmgp_model_predict(h, Z.ctypes.data, nz, out.ctypes.data, nn.ctypes.data))
    out_s = np.empty(nz)
    nn_s = np.empty(nz, dtype=np.int32)
    step = 50000
    for b in range(0, nz, step):
        e = min(nz, b + step)
        N.check(N.LIB.fmgp_model_predict(h, Z[b:e].ctypes.data, e - b, out_s[b:e].ctypes.data, nn_s[b:e].ctypes.data))
    assert np.array_equal(nn, nn_s)
    assert np.array_equal(out, out_s)
    for bad in (np.nan, np.inf):
        Zb = Z.copy()
        Zb[nz - 7, 1] = bad
        rc = N.LIB.fmgp_model_predict(h, Zb.ctypes.data, nz, out.ctypes.data, nn.ctypes.data)
        assert rc == N.FMGP_EINVAL and N.LIB.fmgp_last_error() == b"fast_predict: non-finite test point"
    N.check(N.LIB.fmgp_model_predict(h, Z.ctypes.data, nz, out.ctypes.data, nn.ctypes.data))
    assert np.array_equal(out, out_s)


@pytest.mark.parametrize("nz", [1000, 100000])
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_device_pointer_predict_survives_non_finite_test_points(nz, bad):
    # The stream-ordered entry points cannot return a status for the contents of Z: a non-finite
    # test point gets nn = -1 and NaN means, the other points their normal result, and nothing
    # faults (a NaN coordinate used to index the cell grid out of range).
    import torch
    import paper_2205_10879_b200 as fm
    from paper_2205_10879_b200 import _native as N
    rng = np.random.default_rng(6)
    n, k = 20000, 30
    X = rng.random((n, 3))
    Y = rng.standard_normal(n)
    p = fm.KernelParams(1.0, 0.2, 2.5, 0.05)
    model = fm.precompute(fm.TrainingSet(X, Y, 0.25), fm.FittedParams(p, fm.KernelKind.Matern),
                          fm.NeighborIndex.build(X), k)
    Z = rng.random((nz, 3))
    ref = fm.fast_predict_batch(model, Z)
    Zb = Z.copy()
    Zb[nz // 2, 2] = bad
    h = model.handle()
    Zd = torch.from_numpy(Zb).cuda()
    out = torch.empty(nz, dtype=torch.float64, device="cuda")
    nn = torch.empty(nz, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    N.check(N.LIB.fmgp_model_predict_device(h, C.c_void_p(Zd.data_ptr()), nz, C.c_void_p(out.data_ptr()),
                                            C.c_void_p(nn.data_ptr()), C.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    assert np.isnan(o[nz // 2]) and nn[nz // 2].item() == -1
    keep = np.arange(nz) != nz // 2
    assert np.array_equal(o[keep], ref[keep])
