"""GPU parity of the MuyGPs training inner loop and the localized predictor
(muygps.cpp:15-295) against the oracle: the C
restatement (Port) and the reference's own muygps.cpp compiled under
oracle/_ref (Reference). Predictions and losses within 1e-9 relative
(north_star fp64 bar); batch samples and neighbour lists bit-exact."""
import numpy as np
import pytest

from helpers import MEAN_TOL, mean_rel_err

pytestmark = pytest.mark.gpu


def spatial_set(n, d, seed):
    rng = np.random.default_rng(seed)
    X = rng.random((n, d))
    y = np.sin(6.0 * X[:, 0]) * np.cos(4.0 * X[:, -1]) + 0.05 * rng.standard_normal(n)
    return X, y - y.mean(), float(y.mean())


def lists_of(port, X, batch, k):
    nbr, dist = [], []
    for i in batch:
        idx, dsq = port.query_knn(X, X[i], k, i)
        nbr.append(idx)
        dist.append(np.sqrt(dsq))
    return np.array(nbr, dtype=np.int32), np.array(dist)


CASES = [  # (d, n, k, kind, sigma, rho, nu, tau)
    (2, 3000, 30, 0, 1.0, 0.05, 1.5, 0.0316),
    (2, 3000, 50, 0, 1.0, 0.05, 2.5, 0.1),
    (3, 2000, 50, 1, 1.0, 0.2, 2.5, 0.1),
    (5, 1500, 100, 1, 1.0, 0.8, 2.5, 0.1),
    (4, 1500, 12, 0, 1.3, 0.6, 0.5, 0.2),
    (2, 1500, 20, 0, 1.0, 0.1, 1.25, 0.1),  # general nu (Bessel K)
]


@pytest.mark.parametrize("d,n,k,kind,s,rho,nu,tau", CASES)
def test_local_predictions_and_loss_match_oracle(fm, port, ref, d, n, k, kind, s, rho, nu, tau):
    X, Y, _ = spatial_set(n, d, 7 * d + k)
    batch = fm.BatchSpec.sample(n, 200, 11)
    nbr, dist = lists_of(port, X, batch.indices, k)
    train = fm.TrainingSet(X, Y, 0.0)
    p = fm.KernelParams(s, rho, nu, tau)
    got = fm.local_predictions(train, batch.indices, nbr, dist, fm.KernelKind(kind), p)
    want = ref.local_predictions(X, Y, batch.indices, nbr, dist, kind, s, rho, nu, tau)
    assert mean_rel_err(got, want).max() <= MEAN_TOL
    if nu in (0.5, 1.5, 2.5) or kind == 1:
        assert np.array_equal(port.local_predictions(X, Y, nbr, dist, kind, s, rho, nu, tau), want)
    lists = [fm.NeighborList(list(a), list(b)) for a, b in zip(nbr, dist)]
    loss = fm.loocv_loss(train, batch, lists, fm.KernelKind(kind), p)
    loss_ref = ref.loocv_loss(X, Y, batch.indices, nbr, dist, kind, s, rho, nu, tau)
    assert abs(loss - loss_ref) <= 1e-9 * abs(loss_ref)
    # the device-resident session gives the same loss, repeatedly
    sess = fm.LoocvSession(train, batch, lists)
    for _ in range(3):
        assert sess.loss(fm.KernelKind(kind), p) == loss
    sess.close()


def test_single_neighbor_closed_form(fm):
    # test_muygps.cpp:43-55: k = 1, exponential kernel, tau = 0 -> exp(-d/rho) y_j
    from paper_2205_10879_b200 import datagen
    X, Y, mo = datagen.sine_set(20, 1)
    train = fm.TrainingSet(X, Y, mo)
    ix = fm.NeighborIndex.build(X)
    nl = ix.query_knn(X[7], 1, 7)
    j, dd = nl.indices[0], nl.distances[0]
    got = fm.local_prediction(train, 7, nl, fm.KernelKind.Matern, fm.KernelParams(1.0, 0.3, 0.5, 0.0))
    assert got == pytest.approx(np.exp(-dd / 0.3) * Y[j], rel=1e-12)


def test_own_index_in_list_is_rejected_after_earlier_entries(fm, port):
    X, Y, _ = spatial_set(500, 2, 3)
    batch = [5, 9, 13]
    nbr, dist = lists_of(port, X, batch, 8)
    nbr[2, 3] = 13
    with pytest.raises(fm.DomainError, match="point 13 appears in its own neighbor list"):
        fm.local_predictions(fm.TrainingSet(X, Y, 0.0), batch, nbr, dist, fm.KernelKind.Matern,
                             fm.KernelParams(1.0, 0.1, 1.5, 0.1))


def test_numeric_failure_names_batch_index(fm, port, ref):
    # exact duplicate with tau = 0 and sigma = 1e6: the jitter ladder cannot help
    X = np.zeros((60, 2))
    X[:, 0] = np.arange(60) * 10.0
    X[31] = X[30]
    Y = np.arange(60, dtype=np.float64)
    batch = [3, 29, 44]
    nbr, dist = lists_of(port, X, batch, 6)
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as eo:
        ref.local_predictions(X, Y, batch, nbr, dist, 1, 1e6, 1.0, 2.5, 0.0)
    with pytest.raises(fm.NumericError) as ei:
        fm.local_predictions(fm.TrainingSet(X, Y, 0.0), batch, nbr, dist, fm.KernelKind.RBF,
                             fm.KernelParams(1e6, 1.0, 2.5, 0.0))
    assert str(ei.value) == str(eo.value)
    assert str(ei.value) == ("Cholesky factorization failed in local_prediction at index 29 "
                             "after jitter escalation up to 1e-6")


@pytest.mark.parametrize("bounds,kind,init", [
    ({"rho": (1e-3, 1e2)}, 0, (1.0, 5.0, 2.5, 0.05)),
    ({"rho": (0.05, 0.5), "tau": (0.01, 0.3)}, 0, (1.0, 0.1, 1.5, 0.1)),
    ({"rho": (1e-2, 1e1)}, 1, (1.0, 2.0, 2.5, 0.1)),
])
def test_train_matches_reference(fm, ref, bounds, kind, init):
    X, Y, _ = spatial_set(2000, 2, 5)
    b, seed, k = 200, 3, 20
    theta_r, loss_r, ev_r, imp_r, batch_r = ref.train(X, Y, b, seed, k, kind, *init, bounds, max_evals=60)
    batch = fm.BatchSpec.sample(2000, b, seed)
    assert batch.indices == batch_r  # the sampler is bit-exact
    cfg = fm.TrainConfig(k=k, kind=fm.KernelKind(kind), max_evals=60,
                         rho_bounds=fm.Bounds(*bounds["rho"]) if "rho" in bounds else None,
                         tau_bounds=fm.Bounds(*bounds["tau"]) if "tau" in bounds else None)
    fit = fm.train(fm.TrainingSet(X, Y, 0.0), fm.KernelParams(*init), cfg, batch, fm.NeighborIndex.build(X))
    assert fit.improved == imp_r
    # the simplex path is the reference's; losses agree to the LOOCV tolerance, so
    # the accepted vertices (and hence the parameters) agree to the same order
    assert abs(fit.final_loss - loss_r) <= 1e-8 * abs(loss_r)
    assert fit.evaluations == ev_r
    got = (fit.theta_hat.sigma, fit.theta_hat.rho, fit.theta_hat.nu, fit.theta_hat.tau)
    assert np.allclose(got, theta_r, rtol=1e-6, atol=0)


def test_train_argument_errors(fm):
    X, Y, _ = spatial_set(100, 2, 1)
    tr = fm.TrainingSet(X, Y, 0.0)
    ix = fm.NeighborIndex.build(X)
    batch = fm.BatchSpec.sample(100, 20, 0)
    with pytest.raises(fm.DomainError, match="train: k must be at least 2"):
        fm.train(tr, fm.KernelParams(1.0, 0.1, 1.5, 0.1), fm.TrainConfig(k=1), batch, ix)
    with pytest.raises(fm.DomainError, match="train: invalid bounds"):
        fm.train(tr, fm.KernelParams(1.0, 0.1, 1.5, 0.1), fm.TrainConfig(k=5, rho_bounds=fm.Bounds(1.0, 0.5)),
                 batch, ix)
    fit = fm.train(tr, fm.KernelParams(2.0, 0.4, 1.5, 0.01), fm.TrainConfig(k=5), batch, ix)
    assert not fit.improved and fit.evaluations == 1 and fit.theta_hat.rho == 0.4
    with pytest.raises(fm.DomainError, match="BatchSpec: batch size out of range"):
        fm.BatchSpec.sample(10, 11, 0)


@pytest.mark.parametrize("d,n,k,kind,s,rho,nu,tau", CASES)
def test_muygps_predict_matches_oracle(fm, port, ref, d, n, k, kind, s, rho, nu, tau):
    X, Y, mo = spatial_set(n, d, 3 * d + k)
    Z = np.random.default_rng(d + k).random((300, d))
    fit = fm.FittedParams(fm.KernelParams(s, rho, nu, tau), fm.KernelKind(kind))
    got = fm.muygps_predict(fm.TrainingSet(X, Y, mo), Z, fit, fm.NeighborIndex.build(X), k)
    want = ref.muygps_predict(X, Y, mo, Z, k, kind, s, rho, nu, tau)
    assert mean_rel_err(got, want).max() <= MEAN_TOL
    if nu in (0.5, 1.5, 2.5) or kind == 1:
        assert np.array_equal(port.muygps_predict(X, Y, mo, Z, k, kind, s, rho, nu, tau), want)


def test_muygps_predict_at_scale_is_consistent_with_fast_predict(fm):
    # At a training point z = x_j with k neighbours, muygps_predict conditions on
    # N(z) = x_j's own kNN incl. itself, i.e. fast_predict's row j: same value.
    X, Y, mo = spatial_set(200_000, 2, 9)
    fit = fm.FittedParams(fm.KernelParams(1.0, 0.05, 1.5, 0.0316), fm.KernelKind.Matern)
    tr = fm.TrainingSet(X, Y, mo)
    ix = fm.NeighborIndex.build(X)
    model = fm.precompute(tr, fit, ix, 50)
    Z = X[::997]
    a = fm.muygps_predict(tr, Z, fit, ix, 50)
    b = fm.fast_predict_batch(model, Z)
    assert mean_rel_err(a, b).max() <= 1e-9
