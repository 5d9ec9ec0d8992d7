"""GPU: the C++ drop-in facade's model residency and model-file contract.

* fast_predict_one on a cfg2-sized model (1e6 training points) reuses the
  model's device replica (created once, at the first predict): a call costs
  a query upload, the grid walk and a read-back, not a model upload.
* FMGP v1 model files move between the reference (oracle/_ref, the
  reference's own TUs) and the facade in both directions: predictions agree
  to the parity bar, and re-saving a loaded file reproduces it byte for byte
  (Exact and ApproxGraph indexes: a reference-written graph is searched by
  the facade, a facade-built graph by the reference).
"""
import json
import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

from helpers import MEAN_TOL, mean_rel_err

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parents[1]
TOOL = REPO / "tests" / "cpp" / "_build" / "facade_tool"


def _tool(*args, timeout=600):
    if not TOOL.exists():
        pytest.fail(f"{TOOL} missing: python -m paper_2205_10879_b200.build")
    out = subprocess.run([str(TOOL), *map(str, args)], capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_fast_predict_one_reuses_the_device_model(fm):
    r = _tool("bench_one", 1_000_000, 300)
    print("facade fast_predict_one on a 1e6-point model:", r)
    assert r["median_us"] < 1000.0, r
    assert r["p90_us"] < 2000.0, r


def _dataset(n=3000, seed=3):
    rng = np.random.default_rng(seed)
    X = rng.random((n, 2))
    y = np.sin(6.0 * X[:, 0]) * np.cos(4.0 * X[:, 1]) + 0.01 * rng.standard_normal(n)
    mo = float(y.mean())
    return X, y - mo, mo


def _write_data(path, X, Y, k, mode, kind, sigma, rho, nu, tau, mo):
    n, d = X.shape
    with open(path, "wb") as f:
        f.write(struct.pack("<qqqqI", n, d, k, mode, kind))
        f.write(struct.pack("<5d", sigma, rho, nu, tau, mo))
        f.write(np.ascontiguousarray(X, dtype="<f8").tobytes())
        f.write(np.ascontiguousarray(Y, dtype="<f8").tobytes())


def _write_z(path, Z):
    with open(path, "wb") as f:
        f.write(struct.pack("<qq", *Z.shape))
        f.write(np.ascontiguousarray(Z, dtype="<f8").tobytes())


KP = (0, 1.0, 0.1, 1.5, 0.03)  # Matern nu = 1.5, rho = 0.1, tau = 0.03


@pytest.mark.parametrize("mode", [0, 1])
def test_reference_written_model_loads_into_the_facade(fm, ref, tmp_path, mode):
    X, Y, mo = _dataset()
    k = 20
    S, Cm = ref.precompute(X, Y, *KP, k)
    p_ref = tmp_path / "ref.fmgp"
    ref.save_model(p_ref, X, S, Cm, *KP, mo, mode=mode, max_degree=8, build_beam=32, seed=5)
    Z = np.random.default_rng(9).random((200, 2))
    _write_z(tmp_path / "z.bin", Z)
    dims, pred_ref = ref.load_model_predict(p_ref, Z)
    assert dims[3] == mode
    p_re = tmp_path / "facade_resave.fmgp"
    pred_fac = np.asarray(_tool("load", p_ref, tmp_path / "z.bin", p_re)["pred"])
    assert mean_rel_err(pred_fac, pred_ref).max() <= MEAN_TOL
    assert p_re.read_bytes() == p_ref.read_bytes()  # byte-identical round trip (graph blob kept verbatim)


@pytest.mark.parametrize("mode", [0, 1])
def test_facade_written_model_loads_into_the_reference(fm, ref, tmp_path, mode):
    """mode 1: the facade's GPU-built ApproxGraph is written in the reference's
    layout; the reference loads it and its fast_predict searches that graph."""
    X, Y, mo = _dataset(seed=4)
    k = 20
    data = tmp_path / "data.bin"
    _write_data(data, X, Y, k, mode, *KP, mo)
    p_fac = tmp_path / "facade.fmgp"
    pred_fac = np.asarray(_tool("save", data, p_fac)["pred"])
    Z = X[: pred_fac.size] + 1e-3
    dims, pred_ref = ref.load_model_predict(p_fac, Z)
    assert list(dims[:3]) == [X.shape[0], 2, k] and dims[3] == mode
    assert mean_rel_err(pred_fac, pred_ref).max() <= MEAN_TOL
    # the file holds the facade's S (bit-exact with the reference's) and C (within the parity bar)
    S_ref, C_ref = ref.precompute(X, Y, *KP, k)
    raw = p_fac.read_bytes()
    hdr = 4 + 4 + 3 * 8 + 4 * 8 + 4
    n = X.shape[0]
    off = hdr + n * 2 * 8
    S_fac = np.frombuffer(raw[off:off + n * k * 4], dtype="<i4").reshape(n, k)
    C_fac = np.frombuffer(raw[off + n * k * 4:off + n * k * 12], dtype="<f8").reshape(n, k)
    assert np.array_equal(S_fac, S_ref)
    err = np.linalg.norm(C_fac - C_ref.reshape(n, k), axis=1) / np.linalg.norm(C_ref.reshape(n, k), axis=1)
    assert err.max() <= 1e-9
    # the reference re-writes the facade's file byte for byte
    p_re = tmp_path / "ref_resave.fmgp"
    ref.resave(p_fac, p_re)
    assert p_re.read_bytes() == raw
