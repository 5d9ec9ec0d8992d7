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
