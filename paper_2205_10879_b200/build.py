"""Build every native artefact in-tree (no JIT cache), for sm_100a only.

    python -m paper_2205_10879_b200.build            # product + oracle checker
    python -m paper_2205_10879_b200.build --product  # product only

Outputs (git-ignored, but they travel to the GPU box with the snapshot):
    paper_2205_10879_b200/lib/libfmgp_b200.so      CUDA kernels + C ABI (include/fmgp_b200.h)
    paper_2205_10879_b200/lib/libfmgp_datagen.so   seeded host workload generators
    paper_2205_10879_b200/lib/libfastmuygps_b200.so the C++ facade (reference headers)
    oracle/build/libfmgp_oracle.so                 C restatement (checker only)
    oracle/_ref/*                                  reference TUs, when /root/reference exists
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
LIB = PKG / "lib"
CSRC = PKG / "csrc"
CPP = PKG / "cpp"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_SOURCES = ["knn.cu", "knn_grid.cu", "knn_tc.cu", "solve.cu", "solve_big.cu", "solve_tc.cu", "solve_reg.cu", "solve_2d.cu", "solve_dm.cu", "solve_cta.cu", "predict.cu", "misc.cu", "capi.cu", "muygps.cu", "group.cu", "graph.cu"]
FACADE_SOURCES = ["facade_kernel.cpp", "facade_linalg.cpp", "facade_nn_index.cpp", "facade_fast_predict.cpp",
                  "facade_dataset.cpp", "facade_muygps.cpp"]


def _run(cmd: list[str], cwd: Path | None = None) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=cwd)


def _stale(out: Path, deps: list[Path]) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(p.stat().st_mtime > t for p in deps)


def build_cuda(force: bool = False, defines: list[str] | None = None, out: Path | None = None) -> Path:
    """Compile each CUDA TU to an object in parallel (build/obj), then link the
    shared library. `defines` (-DNAME=V) and `out` are for kernel A/B variants."""
    out = out or LIB / "libfmgp_b200.so"
    defines = defines or []
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [REPO / "include" / "fmgp_b200.h", Path(__file__)]
    deps = [CSRC / s for s in CUDA_SOURCES] + headers
    if not (force or _stale(out, deps)):
        return out
    LIB.mkdir(exist_ok=True)
    out.parent.mkdir(parents=True, exist_ok=True)
    tag = "_".join(d.lstrip("-D").replace("=", "") for d in defines) or "default"
    objdir = REPO / "build" / "obj" / tag
    objdir.mkdir(parents=True, exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-O3", *defines]
    jobs = []
    for s in CUDA_SOURCES:
        obj = objdir / (Path(s).stem + ".o")
        if force or _stale(obj, [CSRC / s] + headers):
            jobs.append([NVCC, *flags, "-c", "-o", str(obj), str(CSRC / s)])
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4) or 1) as ex:
        list(ex.map(_run, jobs))
    _run([NVCC, *ARCH, "-shared", "-o", str(out), *[str(objdir / (Path(s).stem + ".o")) for s in CUDA_SOURCES], "-ldl"])
    return out


def build_datagen(force: bool = False) -> Path:
    out = LIB / "libfmgp_datagen.so"
    src = PKG / "datagen" / "datagen.cpp"
    if force or _stale(out, [src]):
        LIB.mkdir(exist_ok=True)
        _run([CXX, "-std=c++20", "-O2", "-fPIC", "-shared", "-o", str(out), str(src)])
    return out


def build_facade(force: bool = False) -> Path | None:
    srcs = [CPP / "src" / s for s in FACADE_SOURCES]
    if not all(s.exists() for s in srcs):
        return None
    out = LIB / "libfastmuygps_b200.so"
    deps = srcs + list((CPP / "include" / "fastmuygps").glob("*.hpp")) + list((CPP / "src").glob("*.hpp"))
    deps += [LIB / "libfmgp_b200.so", Path(__file__)]
    if force or _stale(out, deps):
        _run([CXX, "-std=c++20", "-O2", "-fPIC", "-shared", f"-I{CPP / 'include'}", f"-I{CPP / 'shim'}",
              f"-I{REPO / 'include'}", "-o", str(out), *[str(s) for s in srcs],
              f"-L{LIB}", "-lfmgp_b200", "-lz", "-Wl,-rpath,$ORIGIN"])
    return out


def build_test_tools() -> None:
    """tests/cpp/facade_tool: the repo's own driver of the C++ facade (test infrastructure)."""
    _run(["make", "-s", "-C", str(REPO / "tests" / "cpp"), "tool"])


def build_oracle() -> None:
    """The checker: C restatement always; reference TUs when the reference is mounted."""
    _run(["make", "-s", "-C", str(REPO / "oracle")])
    if Path("/root/reference/proj/core/src/fast_predict.cpp").exists():
        _run(["make", "-s", "-C", str(REPO / "oracle"), "ref"])
        # the reference's own test sources compiled against the facade (drop-in check)
        _run(["make", "-s", "-C", str(REPO / "tests" / "cpp")])


def build(product_only: bool = False, force: bool = False) -> None:
    if shutil.which(NVCC) is None and not Path(NVCC).exists():
        raise RuntimeError(f"nvcc not found at {NVCC}; the B200 path cannot be built")
    build_cuda(force)
    build_datagen(force)
    build_facade(force)
    if not product_only:
        build_test_tools()
        build_oracle()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--product", action="store_true")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    build(product_only=a.product, force=a.force)
    sys.exit(0)
