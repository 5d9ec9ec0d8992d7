"""Helper for tests/test_gpu_knn.py: run the GPU kNN through the C ABI in a
fresh process (so FMGP_KNN=brute can select the brute-force path) for every
case in the input file and save the results.
Usage: python knn_dump.py in.npz out.npz   (cases c0_P, c0_k, [c0_Q], c1_...)"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2205_10879_b200 import _native as N  # noqa: E402


def one(P, k, Q, res, tag):
    import torch
    n, d = P.shape
    dP = torch.from_numpy(P).cuda()
    idx = torch.empty((n, k), dtype=torch.int32, device="cuda")
    dsq = torch.empty((n, k), dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()
    # self mode through the device entry point (precompute's exclusion by index)
    N.check(N.LIB.fmgp_query_knn_device(C.c_void_p(dP.data_ptr()), n, d, C.c_void_p(dP.data_ptr()), n, k, 0,
                                        C.c_void_p(idx.data_ptr()), C.c_void_p(dsq.data_ptr()),
                                        C.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    res[f"{tag}_self_idx"] = idx.cpu().numpy()
    res[f"{tag}_self_dsq"] = dsq.cpu().numpy()
    if Q is not None:
        qi = np.empty((Q.shape[0], k), np.int32)
        qd = np.empty((Q.shape[0], k))
        N.check(N.LIB.fmgp_query_knn(P.ctypes.data, n, d, Q.ctypes.data, Q.shape[0], k, None, qi.ctypes.data,
                                     qd.ctypes.data))
        res[f"{tag}_ext_idx"], res[f"{tag}_ext_d"] = qi, qd
        nn = np.empty(Q.shape[0], np.int32)
        N.check(N.LIB.fmgp_nearest(P.ctypes.data, n, d, Q.ctypes.data, Q.shape[0], nn.ctypes.data))
        res[f"{tag}_nn"] = nn


def main(inp, outp):
    z = np.load(inp)
    res = {}
    for c in range(int(z["ncases"])):
        P = np.ascontiguousarray(z[f"c{c}_P"])
        Q = np.ascontiguousarray(z[f"c{c}_Q"]) if f"c{c}_Q" in z else None
        one(P, int(z[f"c{c}_k"]), Q, res, f"c{c}")
    np.savez(outp, **res)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
