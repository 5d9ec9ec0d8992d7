"""Run one stage of the path once on cuda:0 (for ncu captures):
    python profiles/tools/run_stage.py --cfg 2 --n 200000 --stage precompute|predict|knn|knnrows [--rows R]"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=2)
    ap.add_argument("--n", type=int, default=200000)
    ap.add_argument("--nt", type=int, default=200000)
    ap.add_argument("--stage", default="precompute")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--rows", type=int, default=0, help="knnrows: neighbour rows [0, rows) against all n points")
    a = ap.parse_args()
    import torch
    import paper_2205_10879_b200 as fm
    from paper_2205_10879_b200 import _native as N, datagen
    ds = datagen.generate(a.cfg, a.n, a.nt)
    i = ds.info
    X = torch.from_numpy(ds.X).cuda()
    Y = torch.from_numpy(ds.Y).cuda()
    Z = torch.from_numpy(ds.Z).cuda()
    fit = fm.FittedParams(fm.KernelParams(i.sigma, i.rho, i.nu, i.tau), fm.KernelKind(i.kind))
    S = torch.empty((a.n, i.k), dtype=torch.int32, device="cuda")
    Cm = torch.empty((a.n, i.k, i.m), dtype=torch.float64, device="cuda")
    out = torch.empty((a.nt, i.m), dtype=torch.float64, device="cuda")
    for _ in range(a.reps):
        if a.stage in ("precompute", "predict"):
            fm.precompute_device(X, Y, fit, i.k, 0, a.n, S, Cm)
        if a.stage == "predict":
            fm.predict_device(X, S, Cm, fit, ds.mean_offset, Z, out)
        if a.stage == "knn":
            s = torch.cuda.current_stream()
            N.check(N.LIB.fmgp_query_knn_device(C.c_void_p(X.data_ptr()), a.n, i.d, C.c_void_p(X.data_ptr()), a.n,
                                                i.k - 1, 0, C.c_void_p(S.data_ptr()), None, C.c_void_p(s.cuda_stream)))
        if a.stage == "knnrows":
            s = torch.cuda.current_stream()
            N.check(N.LIB.fmgp_knn_rows_device(C.c_void_p(X.data_ptr()), a.n, i.d, i.k, 0, a.rows or a.n,
                                               C.c_void_p(S.data_ptr()), C.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
