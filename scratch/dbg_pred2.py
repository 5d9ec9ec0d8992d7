import numpy as np, ctypes as C, sys, torch
sys.path.insert(0, '.')
import paper_2205_10879_b200 as fm
from paper_2205_10879_b200 import _native as N
rng = np.random.default_rng(5)
n, k, nz = 30000, 30, 100000
X = rng.random((n, 3)); Y = rng.standard_normal(n)
p = fm.KernelParams(1.0, 0.2, 2.5, 0.05)
model = fm.precompute(fm.TrainingSet(X, Y, 0.25), fm.FittedParams(p, fm.KernelKind.Matern), fm.NeighborIndex.build(X), k)
Z = rng.random((nz, 3)) * 1.2 - 0.1
Z[nz - 7, 1] = np.nan
h = model.handle()
Zd = torch.from_numpy(Z).cuda(); out = torch.empty(nz, dtype=torch.float64, device="cuda"); nn = torch.empty(nz, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()
rc = N.LIB.fmgp_model_predict_device(h, C.c_void_p(Zd.data_ptr()), nz, C.c_void_p(out.data_ptr()), C.c_void_p(nn.data_ptr()), C.c_void_p(s.cuda_stream))
torch.cuda.synchronize()
print("rc", rc, out[nz-7].item(), nn[nz-7].item())
