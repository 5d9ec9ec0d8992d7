"""B200-native FastMuyGPs posterior-mean path (precompute + predict), plus the
MuyGPs training inner loop and localized predictor built from the same kernels.

Public names mirror the reference C++ API (namespace fastmuygps); they are
loaded lazily from `api` so that `python -m paper_2205_10879_b200.build` works
before the native library exists. Importing any of them without the built
libfmgp_b200.so raises ImportError: there is no CPU fallback.
"""
from __future__ import annotations

import importlib

_API = {
    "KernelKind", "KernelParams", "FittedParams", "TrainingSet", "detrend", "IndexMode", "GraphParams", "NeighborIndex",
    "NeighborList", "PrecomputedModel", "precompute", "fast_predict_one", "fast_predict_batch",
    "kernel_value", "kernel_values", "matern_value", "rbf_value", "cov_matrix", "cov_matrix_self",
    "solve_spd", "solve_spd_batched", "precompute_device", "predict_device", "DomainError", "NumericError",
    "CudaError", "FmgpError", "BatchSpec", "Bounds", "TrainConfig", "local_prediction", "local_predictions",
    "loocv_loss", "LoocvSession", "train", "muygps_predict",
}

__all__ = sorted(_API)


def __getattr__(name):
    if name in _API:
        return getattr(importlib.import_module(".api", __name__), name)
    raise AttributeError(name)
