"""GPU: the tcgen05 (tensor-core) exact kNN used for d >= 4 (kk <= 99).

1. Plumbing: the filter value D~ = n^_q - 2 (q^.p^ - n^_p/2) of the first
   128x256 tile (the point norm enters the GEMM through three fp16 split
   columns), produced by TMA -> tcgen05.mma -> TMEM -> tcgen05.ld, equals
   n^_q + n^_p - 2 q^.p^ computed on the host from the same fp16-rounded
   operands (to fp32 accumulation accuracy).
2. Exactness: indices and keys equal the oracle's for several d (one and many
   64-wide k-blocks, ragged tails), k up to 100, ties/duplicates and row shards.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def host_filter_tile(Q, P):
    # prep of knn_tc.cu: s = 2^e with max|x^| <= 2^14 and max ||p^||^2 <= 2^16;
    # the GEMM folds -n^_p/2 in through three fp16 columns, so the device value
    # is D~ = n^_q - 2 (q^.p^ - n^_p/2)
    mu = P.mean(axis=0)
    maxabs = max(np.abs(P - mu).max(), np.abs(Q - mu).max())
    maxn2 = ((P - mu) ** 2).sum(1).max()
    s = min(2.0 ** np.floor(np.log2(16384.0 / maxabs)), 2.0 ** np.floor(0.5 * np.log2(65536.0 / maxn2)))
    qh = ((Q[:128] - mu) * s).astype(np.float16).astype(np.float64)
    ph = ((P[:256] - mu) * s).astype(np.float16).astype(np.float64)
    nq = (qh ** 2).sum(1)
    npn = (ph ** 2).sum(1)
    return nq[:, None] + npn[None, :] - 2.0 * qh @ ph.T, nq, npn


@pytest.mark.parametrize("d", [4, 40, 64, 65, 200])
def test_tc_tile_matches_host(fm, d):
    from paper_2205_10879_b200 import _native as N
    rng = np.random.default_rng(d)
    P = rng.standard_normal((700, d))
    Q = rng.standard_normal((300, d))
    G = np.zeros((128, 256), dtype=np.float32)
    N.check(N.LIB.fmgp_debug_tc_tile(Q.ctypes.data, 300, P.ctypes.data, 700, d, G.ctypes.data))
    ref, nq, npn = host_filter_tile(Q, P)
    w = 128  # the kernel's point tile is 128 wide; the rest of the 128x256 buffer stays zero
    scale = (nq[:, None] + npn[None, :])[:, :w]
    err = np.abs(G[:, :w] - ref[:, :w]) / scale
    assert np.all(G[:, w:] == 0)
    assert err.max() < 1e-5, err.max()


@pytest.mark.parametrize("d,n,k", [(4, 3000, 10), (5, 2000, 50), (8, 2000, 33), (40, 3000, 99), (64, 1500, 30),
                                   (65, 1500, 30), (130, 1000, 64), (784, 800, 29)])
def test_tc_knn_matches_oracle(fm, port, d, n, k):
    rng = np.random.default_rng(d * 7 + k)
    X = rng.standard_normal((n, d))
    X[5] = X[3]            # exact duplicate
    X[n - 1] = X[n - 2]
    index = fm.NeighborIndex.build(X)
    Q = np.concatenate([rng.standard_normal((40, d)), X[:10]])
    idx, dist = index.query_knn_batch(Q, k)
    for r in range(Q.shape[0]):
        oi, od = port.query_knn(X, Q[r], k)
        assert idx[r].tolist() == oi.tolist(), (d, k, r)
        assert np.array_equal(dist[r], np.sqrt(od))


def test_tc_self_mode_rows_and_shards(fm, port):
    # precompute's self-excluded neighbours, full table and a row shard (device entry points)
    import torch
    from paper_2205_10879_b200 import _native as N
    rng = np.random.default_rng(3)
    n, d, k = 2500, 24, 40
    X = np.round(rng.standard_normal((n, d)) * 4) / 4  # coarse lattice: ties
    dX = torch.from_numpy(X).cuda()
    for b, e in ((0, n), (700, 1900)):
        idx = torch.empty((e - b, k), dtype=torch.int32, device="cuda")
        N.check(N.LIB.fmgp_query_knn_device(C.c_void_p(dX.data_ptr()), n, d, C.c_void_p(dX[b:].data_ptr()), e - b,
                                            k, b, C.c_void_p(idx.data_ptr()), None,
                                            C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        torch.cuda.synchronize()
        got = idx.cpu().numpy()
        for r in range(0, e - b, 97):
            oi, _ = port.query_knn(X, X[b + r], k, b + r)
            assert got[r].tolist() == oi.tolist(), (b, r)


def test_tc_overflow_falls_back_exactly(fm, port):
    # Many exact duplicates at the same distance overflow the candidate window
    # (capacity kk + 29): those queries are redone by the exact brute force.
    rng = np.random.default_rng(9)
    base = rng.standard_normal((20, 6))
    X = np.repeat(base, 100, axis=0)  # 100 copies of 20 points
    index = fm.NeighborIndex.build(X)
    Q = np.concatenate([base[:5] + 1e-3, rng.standard_normal((5, 6))])
    idx, dist = index.query_knn_batch(Q, 50)
    for r in range(Q.shape[0]):
        oi, od = port.query_knn(X, Q[r], 50)
        assert idx[r].tolist() == oi.tolist()
