"""ctypes binding of the C ABI in include/fmgp_b200.h (libfmgp_b200.so).

The library is loaded from this package's lib/ directory (or the A/B variant
build named by FMGP_LIB) only; if it is missing the import fails loudly — there is no Python or CPU fallback for any
compute entry point.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"
LIB_PATH = Path(os.environ["FMGP_LIB"]) if os.environ.get("FMGP_LIB") else LIB_DIR / "libfmgp_b200.so"  # FMGP_LIB: an A/B variant build

FMGP_OK, FMGP_EINVAL, FMGP_ENUMERIC, FMGP_ECUDA = 0, 1, 2, 3


class KernelParamsC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("sigma", C.c_double), ("rho", C.c_double),
                ("nu", C.c_double), ("tau", C.c_double)]


class TrainConfigC(C.Structure):
    _fields_ = [("k", C.c_int32), ("kind", C.c_int32), ("has_rho", C.c_int32), ("has_nu", C.c_int32),
                ("has_tau", C.c_int32), ("rho_lo", C.c_double), ("rho_hi", C.c_double), ("nu_lo", C.c_double),
                ("nu_hi", C.c_double), ("tau_lo", C.c_double), ("tau_hi", C.c_double), ("max_evals", C.c_int32),
                ("tol", C.c_double)]


_d = C.POINTER(C.c_double)
_i32 = C.POINTER(C.c_int32)
_i64 = C.POINTER(C.c_int64)
_kp = C.POINTER(KernelParamsC)
_vp = C.c_void_p

# name -> (restype, argtypes); exactly the symbols include/fmgp_b200.h declares.
SIGNATURES: dict[str, tuple] = {
    "fmgp_abi_version": (C.c_int, []),
    "fmgp_last_error": (C.c_char_p, []),
    "fmgp_launch_count": (C.c_int64, []),
    "fmgp_device_count": (C.c_int, []),
    "fmgp_validate_kernel": (C.c_int, [_kp]),
    "fmgp_precompute": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, C.c_int32, _kp, C.c_int32, _vp, _vp, _i64]),
    "fmgp_precompute_rows": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, C.c_int32, _kp, C.c_int32, C.c_int64,
                                       C.c_int64, _vp, _vp, _i64]),
    "fmgp_precompute_device": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, C.c_int32, _kp, C.c_int32, C.c_int64,
                                         C.c_int64, _vp, _vp, _i64, _vp]),
    "fmgp_knn_rows_device": (C.c_int, [_vp, C.c_int64, C.c_int32, C.c_int32, C.c_int64, C.c_int64, _vp, _vp]),
    "fmgp_solve_rows_device": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, C.c_int32, _kp, C.c_int32, _vp, C.c_int64,
                                         C.c_int64, _vp, _vp, _i64, _vp]),
    "fmgp_query_knn": (C.c_int, [_vp, C.c_int64, C.c_int32, _vp, C.c_int64, C.c_int32, _vp, _vp, _vp]),
    "fmgp_query_knn_device": (C.c_int, [_vp, C.c_int64, C.c_int32, _vp, C.c_int64, C.c_int32, C.c_int64, _vp,
                                        _vp, _vp]),
    "fmgp_nearest": (C.c_int, [_vp, C.c_int64, C.c_int32, _vp, C.c_int64, _vp]),
    "fmgp_nearest_device": (C.c_int, [_vp, C.c_int64, C.c_int32, _vp, C.c_int64, _vp, _vp]),
    "fmgp_index_create": (C.c_int, [_vp, C.c_int64, C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "fmgp_index_query_knn": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, _vp, _vp, _vp]),
    "fmgp_index_nearest": (C.c_int, [_vp, _vp, C.c_int64, _vp]),
    "fmgp_index_distances": (C.c_int, [_vp, _vp, _vp, C.c_int64, _vp]),
    "fmgp_index_destroy": (None, [_vp]),
    "fmgp_graph_build": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.POINTER(_vp)]),
    "fmgp_graph_load": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_uint64, C.c_int32, C.c_int32, _vp,
                                  _vp, _vp, C.POINTER(_vp)]),
    "fmgp_graph_info": (C.c_int, [_vp, _i32, _i32, _i64, _i64]),
    "fmgp_graph_export": (C.c_int, [_vp, _vp, _vp, _vp]),
    "fmgp_graph_query_knn": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, _vp, _vp, _vp, C.POINTER(C.c_uint64)]),
    "fmgp_graph_nearest": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.POINTER(C.c_uint64)]),
    "fmgp_graph_destroy": (None, [_vp]),
    "fmgp_predict": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _kp, _vp, _vp,
                               C.c_int64, _vp, _vp]),
    "fmgp_predict_device": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _kp, _vp, _vp,
                                      C.c_int64, _vp, _vp, _vp]),
    "fmgp_model_create": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _kp, _vp,
                                    C.c_int32, C.POINTER(_vp)]),
    "fmgp_model_predict": (C.c_int, [_vp, _vp, C.c_int64, _vp, _vp]),
    "fmgp_model_destroy": (None, [_vp]),
    "fmgp_model_wrap_device": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _kp, _vp,
                                         C.POINTER(_vp)]),
    "fmgp_model_predict_device": (C.c_int, [_vp, _vp, C.c_int64, _vp, _vp, _vp]),
    "fmgp_model_replicas": (C.c_int, [_vp]),
    "fmgp_group_unique_id": (C.c_int, [_vp]),
    "fmgp_group_create_rank": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.POINTER(_vp)]),
    "fmgp_group_create_devices": (C.c_int, [_vp, C.c_int32, C.POINTER(_vp)]),
    "fmgp_group_info": (C.c_int, [_vp, _i32, _i32, _i32]),
    "fmgp_group_rows": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, _i64, _vp]),
    "fmgp_group_destroy": (None, [_vp]),
    "fmgp_group_precompute": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, C.c_int32, _kp, C.c_int32, _vp, _vp,
                                        _vp, _i64, C.POINTER(_vp)]),
    "fmgp_group_precompute_device": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, C.c_int32, _kp, C.c_int32,
                                               _vp, _vp, _i64, _vp]),
    "fmgp_cov_matrix": (C.c_int, [_vp, C.c_int64, _vp, C.c_int64, C.c_int32, _kp, _vp]),
    "fmgp_kernel_values": (C.c_int, [_vp, C.c_int64, _kp, _vp]),
    "fmgp_solve_spd_batched": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, C.c_int32, _vp, _vp, _i64]),
    "fmgp_local_predictions": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, _vp, _vp, _vp, C.c_int64, C.c_int32,
                                         _kp, _vp, _i64]),
    "fmgp_loocv_create": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, _vp, _vp, _vp, C.c_int64, C.c_int32,
                                    C.POINTER(_vp)]),
    "fmgp_loocv_eval": (C.c_int, [_vp, _kp, _d, _vp, _i64]),
    "fmgp_loocv_destroy": (None, [_vp]),
    "fmgp_train": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, _vp, C.c_int64, _kp, C.POINTER(TrainConfigC), _kp,
                             _d, _i32, _i32]),
    "fmgp_muygps_predict": (C.c_int, [_vp, _vp, C.c_int64, C.c_int32, _vp, C.c_int64, C.c_int32, _kp, C.c_double,
                                      _vp, _i64]),
    "fmgp_set_stage_timing": (None, [C.c_int]),
    "fmgp_stage_times": (C.c_int, [_d, _d, _i64]),
    "fmgp_diag_fp64_peak": (C.c_int, [_d, _d]),
    "fmgp_debug_tc_tile": (C.c_int, [_vp, C.c_int64, _vp, C.c_int64, C.c_int32, _vp]),
}


class FmgpError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class DomainError(FmgpError, ValueError):
    """std::domain_error in the reference."""


class NumericError(FmgpError, ArithmeticError):
    """fastmuygps::NumericError (errors.hpp:11-14)."""

    def __init__(self, code: int, msg: str, failed_row: int = -1):
        super().__init__(code, msg)
        self.failed_row = failed_row


class CudaError(FmgpError):
    """No usable device or a CUDA failure (never silently falls back)."""


def load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2205_10879_b200.build` "
            "(the FastMuyGPs B200 path has no CPU fallback)")
    if not os.environ.get("FMGP_NCCL_LIB"):
        # device groups dlopen NCCL lazily; in a Python process prefer the NCCL wheel torch is built
        # against over an older system libnccl.so.2 (same SONAME: whichever loads first wins, and
        # torch imported later would miss symbols in the older one)
        import importlib.util
        try:
            spec = importlib.util.find_spec("nvidia.nccl")
        except (ImportError, ValueError):
            spec = None
        for loc in (spec.submodule_search_locations if spec is not None and spec.submodule_search_locations else []):
            cand = Path(loc) / "lib" / "libnccl.so.2"
            if cand.exists():
                os.environ["FMGP_NCCL_LIB"] = str(cand)
                break
    lib = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = load()


def check(rc: int, failed_row: int = -1) -> None:
    if rc == FMGP_OK:
        return
    msg = LIB.fmgp_last_error().decode()
    if rc == FMGP_EINVAL:
        raise DomainError(rc, msg)
    if rc == FMGP_ENUMERIC:
        raise NumericError(rc, msg, failed_row)
    raise CudaError(rc, msg)
