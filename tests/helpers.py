"""Shared test helpers: tolerances (north_star: 1e-9 relative in fp64) and metrics."""
import numpy as np

C_TOL = 1e-9      # ||dC_i||_2 / ||C_i||_2 per row
MEAN_TOL = 1e-9   # |a - b| / (1 + |b|), the reference's metric (acceptance.cpp:120-121)


def row_rel_err(C, Cref):
    C = np.asarray(C).reshape(C.shape[0], -1)
    Cref = np.asarray(Cref).reshape(Cref.shape[0], -1)
    num = np.linalg.norm(C - Cref, axis=1)
    den = np.linalg.norm(Cref, axis=1)
    return num / np.where(den > 0, den, 1.0)


def mean_rel_err(a, b):
    a = np.asarray(a).reshape(-1)
    b = np.asarray(b).reshape(-1)
    return np.abs(a - b) / (1.0 + np.abs(b))


def kparams(info):
    """(kind, sigma, rho, nu, tau) of a datagen ConfigInfo."""
    return info.kind, info.sigma, info.rho, info.nu, info.tau
