import numpy as np, ctypes as C, sys
sys.path.insert(0, '.')
import paper_2205_10879_b200 as fm
from paper_2205_10879_b200 import _native as N
rng = np.random.default_rng(5)
n, k, nz = 30000, 30, 600000
X = rng.random((n, 3)); Y = rng.standard_normal(n)
p = fm.KernelParams(1.0, 0.2, 2.5, 0.05)
model = fm.precompute(fm.TrainingSet(X, Y, 0.25), fm.FittedParams(p, fm.KernelKind.Matern), fm.NeighborIndex.build(X), k)
Z = rng.random((nz, 3)) * 1.2 - 0.1
h = model.handle()
out = np.empty(nz); nn = np.empty(nz, dtype=np.int32)
Zb = Z.copy(); Zb[nz - 7, 1] = np.nan
rc = N.LIB.fmgp_model_predict(h, Zb.ctypes.data, nz, out.ctypes.data, nn.ctypes.data)
print("rc", rc, N.LIB.fmgp_last_error(), out[nz-7], nn[nz-7], np.isnan(out).sum())
