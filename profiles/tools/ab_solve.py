"""A/B of the fused-solve variants on one GPU, same data, same process:
the default solve vs FMGP_SOLVE_DM=1 (DMMA-blocked) — time (CUDA events,
fmgp_solve_rows_device on the full row set of the config) and agreement of C.
    python profiles/tools/ab_solve.py [--configs 5,2] [--rows N] [--reps 3]"""
import argparse
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="5,2")
    ap.add_argument("--rows", type=int, default=0, help="solve only the first N rows (0: all)")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--variants", default="reg,dm")
    a = ap.parse_args()
    import torch
    import paper_2205_10879_b200 as fm
    from paper_2205_10879_b200 import _native as N, datagen
    from bench import ClockSampler
    s = torch.cuda.current_stream()
    for cfg in [int(c) for c in a.configs.split(",")]:
        ds = datagen.generate(cfg)
        i = ds.info
        X = torch.from_numpy(ds.X).cuda()
        Y = torch.from_numpy(ds.Y).cuda()
        fit = fm.FittedParams(fm.KernelParams(i.sigma, i.rho, i.nu, i.tau), fm.KernelKind(i.kind))
        n = i.n if a.rows <= 0 else min(a.rows, i.n)
        S = torch.empty((n, i.k), dtype=torch.int32, device="cuda")
        N.check(N.LIB.fmgp_knn_rows_device(C.c_void_p(X.data_ptr()), i.n, i.d, i.k, 0, n, C.c_void_p(S.data_ptr()),
                                           C.c_void_p(s.cuda_stream)))
        kp = fit.theta_hat.c(fit.kind)
        res = {}
        outs = {}
        for var in a.variants.split(","):
            if "=" in var:  # NAME=VALUE: a runtime switch of the default solve (e.g. FMGP_CTA_SLICE=0)
                name, value = var.split("=", 1)
                os.environ[name] = value
            else:
                os.environ["FMGP_SOLVE_DM"] = "1" if var == "dm" else "0"
                os.environ["FMGP_SOLVE_2D"] = "1" if var == "2d" else "0"
            Cm = torch.empty((n, i.k, i.m), dtype=torch.float64, device="cuda")
            failed = C.c_int64(-1)

            def run():
                N.check(N.LIB.fmgp_solve_rows_device(C.c_void_p(X.data_ptr()), C.c_void_p(Y.data_ptr()), i.n, i.d,
                                                     i.m, C.byref(kp), i.k, C.c_void_p(S.data_ptr()), n, 0,
                                                     C.c_void_p(Cm.data_ptr()), None, C.byref(failed),
                                                     C.c_void_p(s.cuda_stream)), failed.value)
            times = []
            with ClockSampler(torch.cuda.current_device()) as clk:
                for r in range(a.reps + 1):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    run()
                    e1.record(s)
                    e1.synchronize()
                    if r > 0:
                        times.append(e0.elapsed_time(e1))
            res[var] = {"ms": min(times), "all_ms": times, "clocks": clk.summary()}
            outs[var] = Cm
        ref = outs[a.variants.split(",")[0]]
        scale = ref.abs().amax(dim=1, keepdim=True).clamp_min(1e-300)
        for var, Cm in outs.items():
            rel = ((Cm - ref).abs() / scale).amax(dim=1).flatten()
            res[var]["max_rel_vs_first"] = float(rel.max())
            res[var]["rows_rel_gt_1e-9"] = int((rel > 1e-9).sum())
            res[var]["nonfinite"] = int((~torch.isfinite(Cm)).sum())
        print(json.dumps({"cfg": cfg, "rows": n, "k": i.k, "d": i.d, **res}), flush=True)
        del outs, S, X, Y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
