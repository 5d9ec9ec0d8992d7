"""MuyGPs widening measured on cfg2 data (d=2, n=1e6,
Matern nu=1.5): LOOCV loss evaluations/s for batches of b points with k
neighbours (one Nelder-Mead step of `train`), and muygps_predict test-pts/s.
GPU (host-synchronous C ABI, wall clock incl. the b-prediction read-back)
next to the reference's own muygps.cpp (oracle/_ref; loocv_loss and
muygps_predict are single-threaded in the reference). One JSON line each.
    python profiles/tools/muygps_bench.py"""
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))


def main():
    import paper_2205_10879_b200 as fm
    from paper_2205_10879_b200 import datagen
    from oracle.oracle import Reference, Port
    ref = Reference()
    port = Port()
    ds = datagen.generate(2, 1_000_000, 100_000)
    i = ds.info
    X, Y = ds.X, ds.Y.reshape(-1)
    kind = fm.KernelKind(i.kind)
    p = fm.KernelParams(i.sigma, i.rho, i.nu, i.tau)
    tr = fm.TrainingSet(X, Y, 0.0)
    for b, k in [(500, 50), (5000, 50), (50000, 50)]:
        batch = fm.BatchSpec.sample(X.shape[0], b, 7)
        ix = fm.NeighborIndex.build(X)
        nbr, dist = ix.query_knn_batch(X[batch.indices], k, exclude=np.asarray(batch.indices))
        lists = [fm.NeighborList(list(a), list(c)) for a, c in zip(nbr, dist)]
        sess = fm.LoocvSession(tr, batch, lists)
        sess.loss(kind, p)
        reps = 20
        t = time.perf_counter()
        for _ in range(reps):
            loss = sess.loss(kind, p)
        gpu = (time.perf_counter() - t) / reps
        nb = min(b, 500)  # the reference on a bounded sub-batch
        t = time.perf_counter()
        loss_r = ref.loocv_loss(X, Y, batch.indices[:nb], nbr[:nb], dist[:nb], i.kind, i.sigma, i.rho, i.nu, i.tau)
        cpu = (time.perf_counter() - t) * b / nb
        print(json.dumps({"what": "loocv_loss evaluation", "b": b, "k": k, "gpu_s": gpu, "gpu_evals_per_s": 1 / gpu,
                          "reference_s_per_eval": cpu, "reference_threads": 1, "loss": loss}), flush=True)
    Z = ds.Z
    fit = fm.FittedParams(p, kind)
    fm.muygps_predict(tr, Z[:1000], fit, fm.NeighborIndex.build(X), 50)
    t = time.perf_counter()
    out = fm.muygps_predict(tr, Z, fit, fm.NeighborIndex.build(X), 50)
    gpu = time.perf_counter() - t
    t = time.perf_counter()
    want = ref.muygps_predict(X, Y, 0.0, Z[:200], 50, i.kind, i.sigma, i.rho, i.nu, i.tau)
    cpu = (time.perf_counter() - t) / 200
    err = float(np.max(np.abs(out[:200] - want) / (1 + np.abs(want))))
    print(json.dumps({"what": "muygps_predict", "n_test": Z.shape[0], "k": 50,
                      "gpu_test_pts_per_s": Z.shape[0] / gpu, "reference_test_pts_per_s": 1 / cpu,
                      "reference_threads": 1, "max_mean_rel_err_vs_reference": err}), flush=True)


if __name__ == "__main__":
    main()
