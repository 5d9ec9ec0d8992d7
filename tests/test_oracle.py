"""CPU: the oracle is pinned to the reference.

* The C restatement (oracle/fmgp_oracle.c) reproduces the golden fixtures,
  which were produced by the reference's own TUs (oracle/_ref) — neighbour
  tables bit-exact, coefficients/means to 1e-12.
* When oracle/_ref is present, the reference's own hot-path doctest suites
  pass against the shim build, and the port matches the reference on fresh
  random cases (ties, duplicates, exclusion, multi-output).
"""
import hashlib
import subprocess
from pathlib import Path

import numpy as np
import pytest

from helpers import kparams, mean_rel_err, row_rel_err

GOLD = Path(__file__).resolve().parent / "golden"
REF_DIR = Path(__file__).resolve().parents[1] / "oracle" / "_ref"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_port_reproduces_reference_golden(port, cfg):
    from paper_2205_10879_b200 import datagen
    g = np.load(GOLD / f"cfg{cfg}.npz")
    ds = datagen.generate(cfg, int(g["n"]), int(g["nt"]), int(g["seed"]))
    assert sha(ds.X) == str(g["sha_X"]) and sha(ds.Y) == str(g["sha_Y"]) and sha(ds.Z) == str(g["sha_Z"]), \
        "datagen drifted from the golden inputs"
    info = ds.info
    S, C = port.precompute_rows(ds.X, ds.Y, *kparams(info), info.k, threads=4)
    assert np.array_equal(S, g["S"])
    assert row_rel_err(C, g["C"]).max() <= 1e-12
    out, nn = port.predict(ds.X, g["S"], g["C"], *kparams(info), ds.mean_offset, ds.Z, threads=4)
    assert np.array_equal(nn, g["nn"])
    assert mean_rel_err(out, g["pred"]).max() <= 1e-12


def test_port_reproduces_reference_unit_test_sets(port):
    from paper_2205_10879_b200 import datagen
    g = np.load(GOLD / "reftests.npz")
    for j in range(int(g["ncases"])):
        n, d, seed, k, kind = (int(g[f"c{j}_{x}"]) for x in ("n", "d", "seed", "k", "kind"))
        p = g[f"c{j}_p"]
        X, Y, mo = datagen.random_set(n, d, seed)
        assert sha(X) == str(g[f"c{j}_sha_X"])
        S, C = port.precompute_rows(X, Y, kind, *p, k)
        assert np.array_equal(S, g[f"c{j}_S"])
        assert row_rel_err(C[:, :, 0], g[f"c{j}_C"]).max() <= 1e-12
        Z, _, _ = datagen.random_set(25, d, seed + 100)
        out, nn = port.predict(X, S, C, kind, *p, mo, Z)
        assert np.array_equal(nn, g[f"c{j}_nn"])
        assert mean_rel_err(out[:, 0], g[f"c{j}_pred"]).max() <= 1e-12


def test_port_ties_and_exclusion(port):
    g = np.load(GOLD / "ties.npz")
    idx, dsq = port.query_knn(g["X"], np.array([0.1, 0.0]), 4)
    assert idx.tolist() == [0, 1, 2, 3] == g["idx4"].tolist()
    assert np.array_equal(np.sqrt(dsq), g["d4"])
    assert port.nearest(g["X"], np.array([[0.1, 0.0], [0.0, 0.0], [5.5, 5.5]])).tolist() == g["nn"].tolist()
    idx, dsq = port.query_knn(g["X1"], g["X1"][0], 3, 0)
    assert idx.tolist() == g["ex_idx"].tolist() and idx[0] == 1 and dsq[0] == 0.0
    S, C = port.precompute_rows(g["grid"], g["Yg"], 0, 1.0, 1.5, 1.5, 0.1, 9)
    assert np.array_equal(S, g["Sg"])
    assert row_rel_err(C[:, :, 0], g["Cg"]).max() <= 1e-12


def test_port_kernel_closed_forms(port):
    # test_kernel.cpp:13-32 and :57-64
    for dd in (1e-8, 0.01, 0.5, 1.0, 2.3, 7.0, 25.0):
        assert port.kernel_value(dd, 0, 1.7, 2.3, 0.5, 0.0) == pytest.approx(1.7 ** 2 * np.exp(-dd / 2.3), rel=1e-12)
    for dd in (0.05, 0.3, 1.0, 2.8, 6.0):
        a15 = np.sqrt(3.0) * dd / 1.4
        a25 = np.sqrt(5.0) * dd / 1.4
        assert port.kernel_value(dd, 0, 0.9, 1.4, 1.5, 0.0) == pytest.approx(0.81 * (1 + a15) * np.exp(-a15), rel=1e-12)
        assert port.kernel_value(dd, 0, 0.9, 1.4, 2.5, 0.0) == pytest.approx(
            0.81 * (1 + a25 + a25 * a25 / 3) * np.exp(-a25), rel=1e-12)
    assert port.kernel_value(0.0, 0, 2.0, 1.0, 1.5, 0.3) == 4.0 * (1.0 + 0.09)
    assert port.kernel_value(0.0, 1, 2.0, 1.0, 1.5, 0.3) == 4.0 * (1.0 + 0.09)
    assert port.kernel_value(1e-300, 0, 2.0, 1.0, 1.5, 0.3) < 4.0 * 1.0000001


def test_port_exact_knn_matches_independent_sort(port):
    # test_nn_index.cpp:25-55: ordering by (distance, index) from an independent full sort.
    rng = np.random.default_rng(1)
    X = rng.random((300, 5))
    for _ in range(25):
        q = rng.random(5)
        idx, dsq = port.query_knn(X, q, 12)
        d = np.array([np.sum((q - x) ** 2) for x in X])  # numpy: same sequential order for d=5
        truth = sorted(range(300), key=lambda i: (np.linalg.norm(X[i] - q), i))[:12]
        assert idx.tolist() == truth
        assert np.all(np.diff(dsq) >= 0)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_port_matches_reference_on_random_cases(port, ref, seed):
    rng = np.random.default_rng(100 + seed)
    n, d = 300, 1 + seed
    X = np.round(rng.random((n, d)) * 8) / 8  # coarse lattice: many exact ties and duplicates
    Y = rng.standard_normal((n, 2))
    for kind, p in ((0, (1.0, 0.4, 1.5, 0.05)), (1, (1.3, 0.3, 2.5, 0.1))):
        S_r, C_r = ref.precompute_rows(X, Y, kind, *p, 11, threads=2)
        S_p, C_p = port.precompute_rows(X, Y, kind, *p, 11, threads=3)
        assert np.array_equal(S_r, S_p)
        assert row_rel_err(C_p, C_r).max() <= 1e-12
        Z = np.round(rng.random((40, d)) * 8) / 8
        o_r, nn_r = ref.predict(X, S_r, C_r, kind, *p, [0.5, -0.5], Z)
        o_p, nn_p = port.predict(X, S_r, C_r, kind, *p, [0.5, -0.5], Z)
        assert np.array_equal(nn_r, nn_p)
        assert mean_rel_err(o_p, o_r).max() <= 1e-12


def test_threads_do_not_change_results(port):
    # test_fast_predict.cpp:95-105: thread-count invariance, bit-exact.
    from paper_2205_10879_b200 import datagen
    X, Y, _ = datagen.random_set(200, 3, 4)
    S1, C1 = port.precompute_rows(X, Y, 0, 1.0, 0.5, 1.5, 1e-6, 10, threads=1)
    S4, C4 = port.precompute_rows(X, Y, 0, 1.0, 0.5, 1.5, 1e-6, 10, threads=4)
    assert np.array_equal(S1, S4) and np.array_equal(C1, C4)


@pytest.mark.parametrize("suite", ["test_kernel", "test_nn_index", "test_fast_predict", "test_muygps"])
def test_reference_own_suites_pass_against_shim_build(suite, tmp_path):
    exe = REF_DIR / suite
    if not exe.exists():
        pytest.skip("oracle/_ref not built")
    r = subprocess.run([str(exe)], cwd=tmp_path, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed: 0" in r.stdout


@pytest.mark.parametrize("kind,nu,tau", [(0, 0.5, 0.0), (0, 1.5, 0.1), (0, 2.5, 1e-3), (1, 2.5, 0.05)])
def test_port_muygps_matches_reference(port, ref, kind, nu, tau):
    # the restatement of local_prediction / muygps_predict (muygps.cpp:32-62,
    # :272-295) is bit-identical to the reference's own TU
    rng = np.random.default_rng(int(nu * 10) + kind)
    X = rng.random((400, 2))
    Y = np.sin(5 * X[:, 0]) - X[:, 1]
    batch = list(range(0, 400, 9))
    nbr, dist = [], []
    for i in batch:
        idx, dsq = port.query_knn(X, X[i], 12, i)
        nbr.append(idx)
        dist.append(np.sqrt(dsq))
    nbr, dist = np.array(nbr), np.array(dist)
    a = port.local_predictions(X, Y, nbr, dist, kind, 1.0, 0.2, nu, tau)
    b = ref.local_predictions(X, Y, batch, nbr, dist, kind, 1.0, 0.2, nu, tau)
    assert np.array_equal(a, b)
    Z = rng.random((50, 2))
    assert np.array_equal(port.muygps_predict(X, Y, 0.25, Z, 15, kind, 1.0, 0.2, nu, tau),
                          ref.muygps_predict(X, Y, 0.25, Z, 15, kind, 1.0, 0.2, nu, tau))


def test_batch_sampler_matches_reference(ref):
    # BatchSpec::sample (muygps.cpp:15-30): the host sampler is bit-exact
    from paper_2205_10879_b200 import datagen
    X = np.random.default_rng(0).random((300, 1))
    Y = np.sin(8 * X[:, 0])
    for b, seed in [(100, 1), (300, 7), (1, 0)]:
        *_, batch = ref.train(X, Y, b, seed, 5, 0, 1.0, 0.3, 1.5, 0.1, {}, max_evals=10)
        assert datagen.batch_sample(300, b, seed) == batch
