"""Helper for tests/test_gpu_fulltable.py: one full-size neighbour search of a
BASELINE config through the C ABI in a fresh process (so FMGP_KNN=brute can
select the fp64 brute-force kernel), saved as .npy files.
Usage: python fulltable_dump.py <cfg> self|nn <out prefix>
  self: precompute's S rows for every training row (k-1 neighbours, self
        excluded by index) and their dist_sq keys
  nn:   the 1-NN of every test point (nearest_training_point)"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main(cfg, what, out):
    import torch
    from paper_2205_10879_b200 import _native as N, datagen
    info = datagen.config_info(cfg)
    ds = datagen.generate(cfg, info.n, info.n_test if what == "nn" else 1)
    n, d = ds.X.shape
    X = torch.from_numpy(ds.X).cuda()
    s = torch.cuda.current_stream()
    if what == "self":
        kk = info.k - 1
        idx = torch.empty((n, kk), dtype=torch.int32, device="cuda")
        dsq = torch.empty((n, kk), dtype=torch.float64, device="cuda")
        N.check(N.LIB.fmgp_query_knn_device(C.c_void_p(X.data_ptr()), n, d, C.c_void_p(X.data_ptr()), n, kk, 0,
                                            C.c_void_p(idx.data_ptr()), C.c_void_p(dsq.data_ptr()),
                                            C.c_void_p(s.cuda_stream)))
        torch.cuda.synchronize()
        np.save(out + "_idx.npy", idx.cpu().numpy())
        np.save(out + "_dsq.npy", dsq.cpu().numpy())
    else:
        Z = torch.from_numpy(ds.Z).cuda()
        nn = torch.empty(ds.Z.shape[0], dtype=torch.int32, device="cuda")
        N.check(N.LIB.fmgp_nearest_device(C.c_void_p(X.data_ptr()), n, d, C.c_void_p(Z.data_ptr()), ds.Z.shape[0],
                                          C.c_void_p(nn.data_ptr()), C.c_void_p(s.cuda_stream)))
        torch.cuda.synchronize()
        np.save(out + "_nn.npy", nn.cpu().numpy())


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2], sys.argv[3])
