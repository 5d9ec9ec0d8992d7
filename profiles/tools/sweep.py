"""Time every BASELINE config at full size on cuda:0 (one JSON line each):
precompute (kNN + solve) and predict with CUDA events, inputs resident in HBM.
    python profiles/tools/sweep.py [--configs 1,2,3,4,5] [--reps 2]"""
import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import torch
    import paper_2205_10879_b200 as fm
    from paper_2205_10879_b200 import _native as N, datagen
    from bench import ClockSampler  # nvidia-smi clocks + throttle reasons during the timed calls
    s = torch.cuda.current_stream()
    for cfg in [int(c) for c in a.configs.split(",")]:
        t0 = time.time()
        ds = datagen.generate(cfg)
        gen_s = time.time() - t0
        i = ds.info
        X = torch.from_numpy(ds.X).cuda()
        Y = torch.from_numpy(ds.Y).cuda()
        Z = torch.from_numpy(ds.Z).cuda()
        fit = fm.FittedParams(fm.KernelParams(i.sigma, i.rho, i.nu, i.tau), fm.KernelKind(i.kind))
        S = torch.empty((i.n, i.k), dtype=torch.int32, device="cuda")
        Cm = torch.empty((i.n, i.k, i.m), dtype=torch.float64, device="cuda")
        out = torch.empty((i.n_test, i.m), dtype=torch.float64, device="cuda")
        idx = torch.empty((i.n, i.k - 1), dtype=torch.int32, device="cuda")

        def ev(fn):
            times = []
            for r in range(a.reps + 1):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(s)
                fn()
                e1.record(s)
                e1.synchronize()
                if r > 0:
                    times.append(e0.elapsed_time(e1))
            return min(times)

        with ClockSampler(torch.cuda.current_device()) as clk:
            pre = ev(lambda: fm.precompute_device(X, Y, fit, i.k, 0, i.n, S, Cm, s))
            knn = ev(lambda: N.check(N.LIB.fmgp_query_knn_device(C.c_void_p(X.data_ptr()), i.n, i.d,
                                                                  C.c_void_p(X.data_ptr()), i.n, i.k - 1, 0,
                                                                  C.c_void_p(idx.data_ptr()), None,
                                                                  C.c_void_p(s.cuda_stream))))
            pred = ev(lambda: fm.predict_device(X, S, Cm, fit, ds.mean_offset, Z, out, None, s))
        line = {"cfg": cfg, "d": i.d, "n_train": i.n, "n_test": i.n_test, "k": i.k, "m": i.m,
                "precompute_ms": pre, "knn_ms": knn, "solve_ms": pre - knn, "predict_ms": pred,
                "precompute_train_pts_per_s": i.n / (pre / 1e3), "predict_test_pts_per_s": i.n_test / (pred / 1e3),
                "gen_s": gen_s, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
        del X, Y, Z, S, Cm, out, idx
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
