"""Seeded host workload generators (libfmgp_datagen.so) for BASELINE configs 1-5.

Host-side input generation only (not part of the compute path): the same
arrays are fed to the oracle and to the GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent.parent / "lib" / "libfmgp_datagen.so"
_lib = None

BASE_SEED = 20261019  # seed = 20261019 + cfg


def _load():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(f"{_LIB_PATH} missing; run python -m paper_2205_10879_b200.build")
        lib = C.CDLL(str(_LIB_PATH))
        lib.fmgp_config_info.restype = C.c_int
        lib.fmgp_config_info.argtypes = [C.c_int] + [C.c_void_p] * 10
        lib.fmgp_generate.restype = C.c_int
        lib.fmgp_generate.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_uint64] + [C.c_void_p] * 4
        lib.fmgp_random_set.restype = None
        lib.fmgp_random_set.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.fmgp_sine_set.restype = None
        lib.fmgp_sine_set.argtypes = [C.c_int64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
        lib.fmgp_batch_sample.restype = C.c_int
        lib.fmgp_batch_sample.argtypes = [C.c_int32, C.c_int32, C.c_uint64, C.c_void_p]
        _lib = lib
    return _lib


@dataclass
class ConfigInfo:
    cfg: int
    d: int
    n: int
    n_test: int
    k: int
    m: int
    kind: int
    sigma: float
    rho: float
    nu: float
    tau: float


def config_info(cfg: int) -> ConfigInfo:
    lib = _load()
    d, k, m, kind = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    n, nt = C.c_int64(), C.c_int64()
    sg, rho, nu, tau = C.c_double(), C.c_double(), C.c_double(), C.c_double()
    rc = lib.fmgp_config_info(cfg, *[C.addressof(x) for x in (d, n, nt, k, m, kind, sg, rho, nu, tau)])
    if rc != 0:
        raise ValueError(f"unknown config {cfg}")
    return ConfigInfo(cfg, d.value, n.value, nt.value, k.value, m.value, kind.value, sg.value, rho.value,
                      nu.value, tau.value)


@dataclass
class Dataset:
    info: ConfigInfo
    X: np.ndarray           # n x d
    Y: np.ndarray           # n x m (detrended)
    Z: np.ndarray           # n_test x d
    mean_offset: np.ndarray  # m


def generate(cfg: int, n: int | None = None, n_test: int | None = None, seed: int | None = None) -> Dataset:
    """BASELINE config `cfg` at full size, or at (n, n_test) with the same distributions."""
    lib = _load()
    info = config_info(cfg)
    n = info.n if n is None else int(n)
    nt = info.n_test if n_test is None else int(n_test)
    seed = BASE_SEED + cfg if seed is None else int(seed)
    X = np.empty((n, info.d), dtype=np.float64)
    Y = np.empty((n, info.m), dtype=np.float64)
    Z = np.empty((nt, info.d), dtype=np.float64)
    mo = np.empty(info.m, dtype=np.float64)
    rc = lib.fmgp_generate(cfg, n, nt, seed, X.ctypes.data, Y.ctypes.data, Z.ctypes.data, mo.ctypes.data)
    if rc != 0:
        raise ValueError(f"generation failed for cfg {cfg}")
    return Dataset(info, X, Y, Z, mo)


def random_set(n: int, d: int, seed: int):
    """The reference tests' random_set (test_fast_predict.cpp:21-29): (X, Y, mean_offset)."""
    lib = _load()
    X = np.empty((n, d), dtype=np.float64)
    Y = np.empty(n, dtype=np.float64)
    mo = np.empty(1, dtype=np.float64)
    lib.fmgp_random_set(n, d, seed, X.ctypes.data, Y.ctypes.data, mo.ctypes.data)
    return X, Y, float(mo[0])


def sine_set(n: int, seed: int):
    """test_muygps.cpp:17-25: (X n x 1, detrended y, mean_offset)."""
    X = np.empty((n, 1), dtype=np.float64)
    Y = np.empty(n, dtype=np.float64)
    mo = np.zeros(1, dtype=np.float64)
    _load().fmgp_sine_set(n, seed, X.ctypes.data, Y.ctypes.data, mo.ctypes.data)
    return X, Y, float(mo[0])


def batch_sample(n: int, b: int, seed: int) -> list:
    """BatchSpec::sample (muygps.cpp:15-30); raises ValueError when b is not in [1, n]."""
    out = np.empty(max(b, 1), dtype=np.int32)
    if _load().fmgp_batch_sample(n, b, seed, out.ctypes.data) != 0:
        raise ValueError("BatchSpec: batch size out of range")
    return out[:b].tolist()
