"""GPU: the two exact kNN algorithms (cell grid for d <= 3, brute force)
against each other and against the oracle — bit-exact indices and keys —
including ties, duplicates, clustered/degenerate data, queries outside the
bounding box, every top-k width class, and full BASELINE sizes
(size-independent property: two independent exact algorithms agree)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent
KS = [1, 2, 31, 32, 33, 64, 65, 100, 128]


def run_dump(tmp_path, cases, brute=False, tag="a"):
    """cases: list of (P, k, Q or None). Returns list of result dicts."""
    inp = tmp_path / f"in_{tag}.npz"
    outp = tmp_path / f"out_{tag}.npz"
    kw = {"ncases": len(cases)}
    for c, (P, k, Q) in enumerate(cases):
        kw[f"c{c}_P"] = P
        kw[f"c{c}_k"] = k
        if Q is not None:
            kw[f"c{c}_Q"] = Q
    np.savez(inp, **kw)
    env = dict(os.environ)
    if brute:
        env["FMGP_KNN"] = "brute"
    else:
        env.pop("FMGP_KNN", None)
    r = subprocess.run([sys.executable, str(HERE / "knn_dump.py"), str(inp), str(outp)], env=env,
                       capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stderr[-3000:]
    z = np.load(outp)
    out = []
    for c in range(len(cases)):
        out.append({key[len(f"c{c}_"):]: z[key] for key in z.files if key.startswith(f"c{c}_")})
    return out


def datasets():
    rng = np.random.default_rng(7)
    yield "uniform2", rng.random((3000, 2))
    yield "uniform3", rng.random((3000, 3))
    yield "uniform1", rng.random((2000, 1))
    yield "lattice2", np.round(rng.random((3000, 2)) * 20) / 20          # heavy ties + duplicates
    yield "lattice3", np.round(rng.random((3000, 3)) * 6) / 6
    yield "clusters2", np.concatenate([rng.normal(0, 1e-3, (1500, 2)), rng.normal(5, 1.0, (1500, 2))])
    yield "degenerate3", np.column_stack([rng.random(2000), np.zeros(2000), rng.random(2000)])  # a flat dim
    yield "line2", np.column_stack([np.linspace(0, 1, 1000), np.linspace(0, 1, 1000)])
    # far from the origin compared with the spacing (|lo| / h ~ 1e13): the cell
    # bounds' rounding (~eps |x|) exceeds 1e-7 h, the grid margin must carry it
    yield "far2", rng.random((3000, 2)) * 1e-3 + np.array([1e9, -3e8])
    yield "far3", rng.random((3000, 3)) * 1e-2 + 5e8


def test_grid_matches_oracle_small(tmp_path, port):
    cases, meta = [], []
    for name, P in datasets():
        for k in KS:
            rng = np.random.default_rng(k)
            Q = np.concatenate([rng.random((40, P.shape[1])) * 1.2 - 0.1, P[:10]])  # incl. outside the bbox
            cases.append((P, k, Q))
            meta.append((name, k))
    got = run_dump(tmp_path, cases)
    for (P, k, Q), (name, _), g in zip(cases, meta, got):
        n = P.shape[0]
        rows = np.random.default_rng(k + 1).choice(n, 12, replace=False)
        for i in rows:
            idx, dsq = port.query_knn(P, P[i], k, i)
            assert g["self_idx"][i].tolist() == idx.tolist(), (name, k, i)
            assert np.array_equal(g["self_dsq"][i], dsq), (name, k, i)
        for j in range(0, Q.shape[0], 5):
            idx, dsq = port.query_knn(P, Q[j], k)
            assert g["ext_idx"][j].tolist() == idx.tolist(), (name, k, j)
            assert np.array_equal(g["ext_d"][j], np.sqrt(dsq))
        assert np.array_equal(g["nn"], port.nearest(P, Q)), name


def test_grid_matches_bruteforce_every_row(tmp_path):
    cases = [(P, k, None) for name, P in datasets() for k in (1, 33, 100)]
    g = run_dump(tmp_path, cases, tag="g")
    b = run_dump(tmp_path, cases, brute=True, tag="b")
    for a, c in zip(g, b):
        assert np.array_equal(a["self_idx"], c["self_idx"])
        assert np.array_equal(a["self_dsq"], c["self_dsq"])


@pytest.mark.parametrize("cfg,n,k", [(1, 10000, 29), (2, 1000000, 49), (5, 1000000, 49)])
def test_grid_matches_bruteforce_at_scale(tmp_path, cfg, n, k):
    from paper_2205_10879_b200 import datagen
    ds = datagen.generate(cfg, n, 20000)
    g = run_dump(tmp_path, [(ds.X, k, ds.Z)], tag="grid")[0]
    b = run_dump(tmp_path, [(ds.X, k, ds.Z)], brute=True, tag="brute")[0]
    assert np.array_equal(g["self_idx"], b["self_idx"])
    assert np.array_equal(g["self_dsq"], b["self_dsq"])
    assert np.array_equal(g["ext_idx"], b["ext_idx"])
    assert np.array_equal(g["nn"], b["nn"])
    # rows are sorted by (key, index) and never contain the query itself
    d, i = g["self_dsq"], g["self_idx"]
    assert np.all((d[:, 1:] > d[:, :-1]) | ((d[:, 1:] == d[:, :-1]) & (i[:, 1:] > i[:, :-1])))
    assert not np.any(i == np.arange(n)[:, None])


@pytest.mark.parametrize("d", [3, 6, 40])
def test_bruteforce_few_queries_many_points(tmp_path, port, d):
    # few query blocks -> up to 512 point chunks and the warp-per-query merge
    # (the shape of the tensor-core path's overflow redo)
    rng = np.random.default_rng(d)
    P = rng.standard_normal((200_000, d))
    P[7] = P[3]
    Q = np.concatenate([rng.standard_normal((6, d)), P[3:4]])
    cases = [(P, k, Q) for k in (1, 50, 100)]
    got = run_dump(tmp_path, cases, brute=True, tag=f"few{d}")
    for (P_, k, Q_), g in zip(cases, got):
        for j in range(Q_.shape[0]):
            idx, dsq = port.query_knn(P_, Q_[j], k)
            assert g["ext_idx"][j].tolist() == idx.tolist(), (d, k, j)
            assert np.array_equal(g["ext_d"][j], np.sqrt(dsq)), (d, k, j)
