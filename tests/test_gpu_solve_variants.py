"""GPU parity of every fused-solve variant compiled in for the BASELINE low-d
shapes (k in {30, 50}, d in {2, 3}, m = 1): the DMMA-blocked solve (default,
solve_dm.cu), the row-per-lane register solve (FMGP_SOLVE_DM=0, solve_reg.cu)
and the 2-D cyclic solve (FMGP_SOLVE_2D=1, solve_2d.cu), each against the CPU
oracle: coefficients ||dC_i||/||C_i|| <= 1e-9 for every closed-form kernel,
the jitter ladder (linalg.cpp:10-31) taking the same rung as the reference,
and the NumericError row (fast_predict.cpp:105)."""
import numpy as np
import pytest

from helpers import C_TOL, row_rel_err

pytestmark = pytest.mark.gpu

VARIANTS = {"dm": {"FMGP_SOLVE_DM": "1", "FMGP_SOLVE_2D": "0"},
            "reg": {"FMGP_SOLVE_DM": "0", "FMGP_SOLVE_2D": "0"},
            "2d": {"FMGP_SOLVE_DM": "0", "FMGP_SOLVE_2D": "1"}}


def _set(monkeypatch, variant):
    for k, v in VARIANTS[variant].items():
        monkeypatch.setenv(k, v)


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("k,d", [(30, 2), (30, 3), (50, 2), (50, 3)])
@pytest.mark.parametrize("kind,nu", [(1, 2.5), (0, 0.5), (0, 1.5), (0, 2.5)])
def test_variant_matches_oracle(fm, port, monkeypatch, variant, k, d, kind, nu):
    _set(monkeypatch, variant)
    rng = np.random.default_rng(100 * k + 10 * d + kind + int(2 * nu))
    n = 3000
    X = rng.random((n, d))
    Y = rng.standard_normal(n)
    sigma, rho, tau = 1.3, 0.08 if d == 2 else 0.2, 0.03
    p = fm.KernelParams(sigma, rho, nu, tau)
    model = fm.precompute(fm.TrainingSet(X, Y, 0.0), fm.FittedParams(p, fm.KernelKind(kind)),
                          fm.NeighborIndex.build(X), k)
    rows = np.arange(0, n, 5)
    S_o, C_o = port.precompute_rows(X, Y[:, None], kind, sigma, rho, nu, tau, k, rows, threads=8)
    assert np.array_equal(model.S[rows], S_o)
    err = row_rel_err(model.C.reshape(n, k, -1)[rows], C_o)
    assert err.max() <= C_TOL, (variant, err.max())


@pytest.mark.parametrize("variant", list(VARIANTS))
@pytest.mark.parametrize("k,d", [(30, 3), (50, 2)])
def test_variant_singular_block_goes_through_the_ladder(fm, port, monkeypatch, variant, k, d):
    # One exact duplicate pair (its d == 0 entry equals the diagonal, kernel.cpp:58-60, :81-83) and
    # tau = 0: the block is exactly singular, rung 0 fails
    # (pivot <= 0) or passes on a rounding residue of ~1e-17, in the reference as well, so the
    # rows holding the pair are chaotic in both implementations (|C| ~ 1e10 with the 1e-10 rung,
    # ~1e17 on a residue) and are only required to be finite; every other row must match, and
    # the call must succeed or fail as the reference's does.
    _set(monkeypatch, variant)
    n = 2 * k + 40
    X = np.zeros((n, d))
    X[:, 0] = np.arange(n) * 0.37
    X[:, 1] = (np.arange(n) % 3) * 0.11
    X[k + 21] = X[k + 20]
    Y = np.sin(np.arange(n, dtype=np.float64))
    p = fm.KernelParams(1.0, 1.0, 0.5, 0.0)  # exponential kernel: well conditioned away from the pair
    try:
        S_o, C_o = port.precompute_rows(X, Y[:, None], 0, 1.0, 1.0, 0.5, 0.0, k)
    except Exception as e:  # the oracle exhausts the ladder too: then so must the GPU path
        with pytest.raises(fm.NumericError) as ei:
            fm.precompute(fm.TrainingSet(X, Y, 0.0), fm.FittedParams(p, fm.KernelKind.Matern),
                          fm.NeighborIndex.build(X), k)
        assert ei.value.failed_row == e.failed_row
        return
    model = fm.precompute(fm.TrainingSet(X, Y, 0.0), fm.FittedParams(p, fm.KernelKind.Matern),
                          fm.NeighborIndex.build(X), k)
    assert np.array_equal(model.S, S_o)
    Cg = model.C.reshape(n, k, -1)
    assert np.isfinite(Cg).all()
    dup_rows = np.flatnonzero((S_o == k + 20).any(axis=1) & (S_o == k + 21).any(axis=1))
    assert dup_rows.size > 0
    err = row_rel_err(Cg, C_o)
    clean = np.setdiff1d(np.arange(n), dup_rows)
    assert err[clean].max() <= C_TOL, err[clean].max()


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_variant_numeric_error_row(fm, port, monkeypatch, variant):
    from oracle.oracle import OracleError
    _set(monkeypatch, variant)
    k, d = 50, 3
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


# k = 100 CTA solve (solve_cta.cu): the lean kernel at several slice widths (FMGP_CTA_SLICE: 8 -> four
# neighbourhoods per SM, 24 -> three, the default), the full-footprint kernel (0) and the row-per-thread
# sweep (FMGP_CTA_BLOCKED=0), each against the oracle; d = 16 / 48 are the ends of the Gram + lean domain,
# d = 40 is cfg4's, d = 8 takes the pair-table build. A near-duplicate pair (offset 1e-6) takes the exact
# recompute of the squared distance in the Gram builds.
@pytest.mark.parametrize("env", [{"FMGP_CTA_SLICE": "0"}, {"FMGP_CTA_SLICE": "8"}, {"FMGP_CTA_SLICE": "16"},
                                 {"FMGP_CTA_SLICE": "24"}, {"FMGP_CTA_SLICE": "40"},
                                 {"FMGP_CTA_BLOCKED": "0"}], ids=lambda e: ",".join(f"{k[5:]}={v}" for k, v in e.items()))
@pytest.mark.parametrize("d", [8, 16, 40, 48])
def test_cta_solve_layouts_match_oracle(fm, port, monkeypatch, env, d):
    for k_, v in env.items():
        monkeypatch.setenv(k_, v)
    rng = np.random.default_rng(1000 + d)
    n, k = 1500, 100
    X = rng.standard_normal((n, d))
    X[700] = X[10] + 1e-6          # near-duplicate pair (an exact duplicate would make the block singular)
    Y = rng.standard_normal(n)
    kind, sigma, rho, nu, tau = 1, 1.1, 3.0 * np.sqrt(d / 40.0), 2.5, 0.1
    p = fm.KernelParams(sigma, rho, nu, tau)
    model = fm.precompute(fm.TrainingSet(X, Y, 0.0), fm.FittedParams(p, fm.KernelKind(kind)),
                          fm.NeighborIndex.build(X), k)
    rows = np.unique(np.concatenate([np.arange(0, n, 7), [10, 700]]))
    S_o, C_o = port.precompute_rows(X, Y[:, None], kind, sigma, rho, nu, tau, k, rows, threads=8)
    assert np.array_equal(model.S[rows], S_o)
    err = row_rel_err(model.C.reshape(n, k, -1)[rows], C_o)
    assert err.max() <= C_TOL, (env, d, err.max())
