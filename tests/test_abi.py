"""CPU: the drop-in boundary library loads, exports exactly what include/fmgp_b200.h
declares, is built for sm_100a, validates arguments with the reference's error
conventions, and fails loudly (FMGP_ECUDA) instead of falling back to the CPU
when no GPU is present. No compute runs here."""
import ctypes as C
import re
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
HEADER = REPO / "include" / "fmgp_b200.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fmgp_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2205_10879_b200 import _native
    names = declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(_native.LIB, name), name
    assert sorted(_native.SIGNATURES) == names


def test_exported_dynamic_symbols_match_header():
    from paper_2205_10879_b200 import _native
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True,
                         text=True).stdout
    exported = sorted(set(re.findall(r"\bT (fmgp_[a-z0-9_]+)$", out, flags=re.M)))
    assert exported == declared()


def test_built_for_sm100a_only():
    from paper_2205_10879_b200 import _native
    if shutil.which("cuobjdump") is None and not Path("/usr/local/cuda/bin/cuobjdump").exists():
        pytest.skip("cuobjdump not available")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_abi_version():
    from paper_2205_10879_b200 import _native
    assert _native.LIB.fmgp_abi_version() == 2


def _kp(kind=0, sigma=1.0, rho=0.5, nu=1.5, tau=0.1):
    from paper_2205_10879_b200 import _native
    return _native.KernelParamsC(kind, sigma, rho, nu, tau)


@pytest.mark.parametrize("bad,msg", [
    (dict(sigma=0.0), "KernelParams: sigma must be positive and finite"),
    (dict(rho=-1.0), "KernelParams: rho must be positive and finite"),
    (dict(nu=0.0), "KernelParams: nu must be positive and finite"),
    (dict(tau=-0.1), "KernelParams: tau must be non-negative and finite"),
])
def test_kernel_param_errors_match_reference(bad, msg):
    # kernel.cpp:13-28
    from paper_2205_10879_b200 import _native
    kp = _kp(**bad)
    assert _native.LIB.fmgp_validate_kernel(C.byref(kp)) == _native.FMGP_EINVAL
    assert _native.LIB.fmgp_last_error().decode() == msg


def test_precompute_argument_errors():
    from paper_2205_10879_b200 import _native
    X = np.random.default_rng(0).random((10, 2))
    Y = np.zeros(10)
    S = np.empty((10, 11), np.int32)
    Cm = np.empty((10, 11))
    f = C.c_int64()
    kp = _kp()
    rc = _native.LIB.fmgp_precompute(X.ctypes.data, Y.ctypes.data, 10, 2, 1, C.byref(kp), 11, S.ctypes.data,
                                     Cm.ctypes.data, C.byref(f))
    assert rc == _native.FMGP_EINVAL and _native.LIB.fmgp_last_error() == b"precompute: k out of range"
    rc = _native.LIB.fmgp_precompute(X.ctypes.data, Y.ctypes.data, 10, 2, 1, C.byref(kp), 0, S.ctypes.data,
                                     Cm.ctypes.data, C.byref(f))
    assert rc == _native.FMGP_EINVAL
    X[3, 1] = np.nan
    rc = _native.LIB.fmgp_precompute(X.ctypes.data, Y.ctypes.data, 10, 2, 1, C.byref(kp), 5, S.ctypes.data,
                                     Cm.ctypes.data, C.byref(f))
    assert rc == _native.FMGP_EINVAL and _native.LIB.fmgp_last_error() == b"NeighborIndex: non-finite coordinates"


def test_general_nu_is_accepted():
    # The Bessel branch (kernel.cpp:40-51) is implemented on the device.
    from paper_2205_10879_b200 import _native
    for kind in (0, 1):
        kp = _kp(kind=kind, nu=3.7)
        assert _native.LIB.fmgp_validate_kernel(C.byref(kp)) == _native.FMGP_OK


def test_no_cpu_fallback_without_a_gpu():
    from paper_2205_10879_b200 import _native
    if _native.LIB.fmgp_device_count() > 0:
        pytest.skip("a GPU is present")
    X = np.random.default_rng(0).random((10, 2))
    Y = np.zeros(10)
    S = np.empty((10, 3), np.int32)
    Cm = np.empty((10, 3))
    f = C.c_int64()
    kp = _kp()
    rc = _native.LIB.fmgp_precompute(X.ctypes.data, Y.ctypes.data, 10, 2, 1, C.byref(kp), 3, S.ctypes.data,
                                     Cm.ctypes.data, C.byref(f))
    assert rc == _native.FMGP_ECUDA
    assert b"no CPU fallback" in _native.LIB.fmgp_last_error()
    import paper_2205_10879_b200 as fm
    with pytest.raises(fm.CudaError):
        fm.precompute(fm.TrainingSet(X, Y, 0.0), fm.FittedParams(fm.KernelParams(1, 0.5, 1.5, 0.1)),
                      fm.NeighborIndex.build(X), 3)


def test_product_never_imports_the_oracle():
    # build.py may *build* the checker (the driver's build() contract); nothing else may touch it.
    pkg = REPO / "paper_2205_10879_b200"
    for p in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cpp")) + list(pkg.rglob("*.h*")):
        if p.name == "build.py":
            continue
        text = p.read_text(errors="ignore")
        assert "fmgp_oracle" not in text and "from oracle" not in text and "import oracle" not in text, p
