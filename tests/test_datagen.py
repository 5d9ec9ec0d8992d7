"""CPU: seeded workload generators (shapes, determinism, distributions)."""
import numpy as np
import pytest


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_config_shapes_and_determinism(cfg):
    from paper_2205_10879_b200 import datagen
    info = datagen.config_info(cfg)
    a = datagen.generate(cfg, 500, 60)
    b = datagen.generate(cfg, 500, 60)
    assert a.X.shape == (500, info.d) and a.Z.shape == (60, info.d) and a.Y.shape == (500, info.m)
    assert np.array_equal(a.X, b.X) and np.array_equal(a.Y, b.Y) and np.array_equal(a.Z, b.Z)
    assert np.allclose(a.Y.mean(axis=0), 0.0, atol=1e-12)  # detrended (dataset.cpp:24-36)
    assert np.all(np.isfinite(a.X)) and np.all(np.isfinite(a.Y))


def test_baseline_config_table():
    from paper_2205_10879_b200 import datagen
    rows = {c: datagen.config_info(c) for c in range(1, 6)}
    assert [(r.d, r.n, r.n_test, r.k, r.m) for r in rows.values()] == [
        (2, 10000, 2000, 30, 1), (2, 1000000, 1000000, 50, 1), (784, 60000, 10000, 30, 10),
        (40, 2000000, 500000, 100, 1), (3, 8000000, 8000000, 50, 1)]
    assert [r.kind for r in rows.values()] == [1, 0, 0, 1, 0]
    assert [r.rho for r in rows.values()] == [0.1, 0.05, 10.0, 3.0, 0.02]
    assert rows[1].tau ** 2 == pytest.approx(1e-4) and rows[3].tau ** 2 == pytest.approx(1e-2)


def test_cfg3_is_sparse_one_hot():
    from paper_2205_10879_b200 import datagen
    a = datagen.generate(3, 400, 10)
    assert 0.75 < np.mean(a.X == 0.0) < 0.85
    raw = np.round(a.Y + a.mean_offset, 9)
    assert np.all(np.isin(raw, [-1.0, 1.0])) and np.all((raw == 1.0).sum(axis=1) == 1)
