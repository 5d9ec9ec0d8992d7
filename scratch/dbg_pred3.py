import numpy as np, ctypes as C, sys, torch, subprocess, os
if len(sys.argv) > 1:
    sys.path.insert(0, '.')
    import paper_2205_10879_b200 as fm
    from paper_2205_10879_b200 import _native as N
    mode, nz = sys.argv[1], int(sys.argv[2])
    rng = np.random.default_rng(5)
    n, k = 30000, 30
    X = rng.random((n, 3)); Y = rng.standard_normal(n)
    p = fm.KernelParams(1.0, 0.2, 2.5, 0.05)
    model = fm.precompute(fm.TrainingSet(X, Y, 0.25), fm.FittedParams(p, fm.KernelKind.Matern), fm.NeighborIndex.build(X), k)
    Z = rng.random((nz, 3))
    Z[nz - 7, 1] = {"nan": np.nan, "inf": np.inf, "big": 1e200, "ok": 0.5}[mode]
    h = model.handle()
    Zd = torch.from_numpy(Z).cuda(); out = torch.empty(nz, dtype=torch.float64, device="cuda"); nn = torch.empty(nz, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    rc = N.LIB.fmgp_model_predict_device(h, C.c_void_p(Zd.data_ptr()), nz, C.c_void_p(out.data_ptr()), C.c_void_p(nn.data_ptr()), C.c_void_p(s.cuda_stream))
    try:
        torch.cuda.synchronize()
        print(mode, nz, "rc", rc, out[nz-7].item(), nn[nz-7].item())
    except Exception as e:
        print(mode, nz, "FAULT", str(e)[:80])
else:
    for mode in ("ok", "nan", "inf", "big"):
        for nz in (1000, 100000):
            r = subprocess.run([sys.executable, __file__, mode, str(nz)], capture_output=True, text=True)
            print(r.stdout.strip()[-200:] or r.stderr.strip()[-200:])
