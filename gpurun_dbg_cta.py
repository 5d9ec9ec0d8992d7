import ctypes as C, os, sys, json
sys.path.insert(0, '.')
import torch
import paper_2205_10879_b200 as fm
from paper_2205_10879_b200 import _native as N, datagen
s = torch.cuda.current_stream()
ds = datagen.generate(4); i = ds.info
X = torch.from_numpy(ds.X).cuda(); Y = torch.from_numpy(ds.Y).cuda()
fit = fm.FittedParams(fm.KernelParams(i.sigma, i.rho, i.nu, i.tau), fm.KernelKind(i.kind))
n = 400000
S = torch.empty((n, i.k), dtype=torch.int32, device="cuda")
N.check(N.LIB.fmgp_knn_rows_device(C.c_void_p(X.data_ptr()), i.n, i.d, i.k, 0, n, C.c_void_p(S.data_ptr()), C.c_void_p(s.cuda_stream)))
kp = fit.theta_hat.c(fit.kind)
def run(var):
    os.environ["FMGP_CTA_SLICE"] = var
    Cm = torch.empty((n, i.k, i.m), dtype=torch.float64, device="cuda")
    failed = C.c_int64(-1)
    N.check(N.LIB.fmgp_solve_rows_device(C.c_void_p(X.data_ptr()), C.c_void_p(Y.data_ptr()), i.n, i.d, i.m, C.byref(kp), i.k,
            C.c_void_p(S.data_ptr()), n, 0, C.c_void_p(Cm.data_ptr()), None, C.byref(failed), C.c_void_p(s.cuda_stream)), failed.value)
    torch.cuda.synchronize()
    return Cm
ref = run("0")
scale = ref.abs().amax(dim=1, keepdim=True).clamp_min(1e-300)
for var in ["0", "8", "8", "8", "24", "24", "24", "16", "12", "40", "48"]:
    Cm = run(var)
    rel = ((Cm - ref).abs() / scale).amax(dim=1).flatten()
    bad = torch.nonzero(rel > 1e-9).flatten().tolist()
    print(var, "max", float(rel.max()), "bad rows", bad[:10], flush=True)
    for b in bad[:3]:
        dcol = ((Cm[b] - ref[b]).abs() / scale[b]).flatten()
        print("   row", b, "ncols>1e-9:", int((dcol > 1e-9).sum()), "first cols", torch.nonzero(dcol > 1e-9).flatten().tolist()[:12], "S row head", S[b, :6].tolist(), flush=True)
