"""GPU parity at the BASELINE full sizes (BASELINE.json configs 2-5, the exact
n_train / n_test / d / k / m / kernel of each): the whole training set goes
through the GPU precompute, and a random sample of rows is checked against the
C restatement of the reference (oracle.Port, the same seeded inputs): the
neighbour rows S bit-exact, the coefficient rows C within 1e-9 relative, and
for a sample of test points the 1-NN index bit-exact and the posterior mean
within 1e-9 relative. (The full tables cannot be recomputed on the CPU in a
test's time: the reference needs hours for cfg4/cfg5.)"""
import numpy as np
import pytest

from helpers import C_TOL, MEAN_TOL, mean_rel_err, row_rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_full_size_sampled_parity(fm, port, cfg):
    from oracle.oracle import host_threads
    from paper_2205_10879_b200 import datagen
    info = datagen.config_info(cfg)
    ds = datagen.generate(cfg, info.n, info.n_test)
    kind = fm.KernelKind(info.kind)
    p = fm.KernelParams(info.sigma, info.rho, info.nu, info.tau)
    Y = ds.Y if info.m > 1 else ds.Y.reshape(-1)
    mo = ds.mean_offset if info.m > 1 else float(np.asarray(ds.mean_offset).reshape(-1)[0])
    index = fm.NeighborIndex.build(ds.X)
    model = fm.precompute(fm.TrainingSet(ds.X, Y, mo), fm.FittedParams(p, kind), index, info.k)
    thr = host_threads()
    rng = np.random.default_rng(cfg)

    rows = np.sort(rng.choice(info.n, size=48, replace=False)).astype(np.int64)
    S_o, C_o = port.precompute_rows(ds.X, ds.Y, info.kind, info.sigma, info.rho, info.nu, info.tau, info.k, rows,
                                    threads=thr)
    assert np.array_equal(model.S[rows], S_o), cfg
    err = row_rel_err(np.asarray(model.C).reshape(info.n, info.k, -1)[rows], C_o)
    assert err.max() <= C_TOL, (cfg, err.max())

    zs = np.sort(rng.choice(info.n_test, size=96, replace=False))
    Z = ds.Z[zs]
    got = np.asarray(fm.fast_predict_batch(model, Z)).reshape(len(zs), -1)
    want, nn = port.predict(ds.X, model.S, model.C, info.kind, info.sigma, info.rho, info.nu, info.tau,
                            ds.mean_offset, Z, threads=thr)
    assert np.array_equal(index.nearest_batch(Z), nn), cfg
    assert mean_rel_err(got, np.asarray(want).reshape(len(zs), -1)).max() <= MEAN_TOL, cfg
