"""GPU: the ApproxGraph index (IndexMode::ApproxGraph) —
graph.cu's navigable-small-world graph, built on the GPU and searched with
the reference's graph search (nn_index.cpp:83-237, :288-341, :351-366).

What the reference pins for this mode (tests/test_nn_index.cpp:86-147) is
checked here the same way: recall@10 >= 0.95 against brute force, far fewer
distance evaluations than a scan with sub-linear growth, exactly k results on
tiny sets, and serialization round trips. The levels, maximum level and entry
point are the reference's generator's (nn_index.cpp:83-88, :171-176, :231-234),
checked against a Python restatement of it."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def ref_levels(n, max_degree, seed):
    """assign_level (nn_index.cpp:83-88) over the splitmix64 stream (:44-49)."""
    M = (1 << 64) - 1
    state = (seed ^ 0xA02BDBF7BB3C0A7) & M
    ml = 1.0 / math.log(float(max_degree))
    out = np.empty(n, dtype=np.int32)
    for i in range(n):
        state = (state + 0x9E3779B97F4A7C15) & M
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        z ^= z >> 31
        u = (z >> 11) * 2.0 ** -53 + 2.0 ** -54
        out[i] = int(-math.log(u) * ml)
    return out


def brute_knn(X, q, k):
    d = ((X - q) ** 2).sum(axis=1)
    return np.lexsort((np.arange(len(X)), d))[:k]


def test_levels_entry_and_layers_follow_the_reference_generator(fm):
    rng = np.random.default_rng(1)
    X = rng.random((3000, 5))
    p = fm.GraphParams(max_degree=8, seed=77)
    ix = fm.NeighborIndex.build(X, fm.IndexMode.ApproxGraph, p)
    entry, max_level, levels, counts, ids = ix.graph_arrays()
    lv = ref_levels(3000, 8, 77)
    assert np.array_equal(levels, lv)
    assert max_level == lv.max() and entry == int(np.flatnonzero(lv == lv.max())[0])
    # layer 0: every node linked to its 2M exact nearest (self excluded), ascending (dist, index)
    off = np.concatenate([[0], np.cumsum(counts.astype(np.int64))])
    rec = np.concatenate([[0], np.cumsum(levels.astype(np.int64) + 1)])
    for i in range(0, 3000, 97):
        r0 = rec[i]
        l0 = ids[off[r0]:off[r0 + 1]]
        d = ((X - X[i]) ** 2).sum(axis=1)
        d[i] = np.inf
        assert np.array_equal(l0, np.lexsort((np.arange(3000), d))[:16])
        for L in range(1, levels[i] + 1):  # upper layers: the M nearest among the layer's nodes
            ln = ids[off[r0 + L]:off[r0 + L + 1]]
            assert np.all(levels[ln] >= L) and len(ln) <= 8


def test_graph_recall_at_10(fm):
    rng = np.random.default_rng(3)
    X = rng.random((2000, 8))
    ix = fm.NeighborIndex.build(X, fm.IndexMode.ApproxGraph)
    Q = np.random.default_rng(4).random((100, 8))
    idx, dist = ix.query_knn_batch(Q, 10)
    hits = sum(len(set(idx[r]) & set(brute_knn(X, Q[r], 10))) for r in range(100))
    assert hits / 1000 >= 0.95
    # distances are sqrt(dist_sq) of the returned points, ascending
    assert np.allclose(dist, np.sqrt(((X[idx] - Q[:, None, :]) ** 2).sum(axis=2)), rtol=0, atol=1e-15)
    assert np.all(np.diff(dist, axis=1) >= 0)


def test_graph_queries_cost_far_fewer_evaluations_than_a_scan(fm):
    def mean_evals(n):
        X = np.random.default_rng(7).random((n, 8))
        ix = fm.NeighborIndex.build(X, fm.IndexMode.ApproxGraph)
        Q = np.random.default_rng(8).random((50, 8))
        ix.query_knn_batch(Q, 10)
        return ix.dist_evals / 50

    small, large = mean_evals(4000), mean_evals(16000)
    print("mean distance evaluations per query:", small, large)
    assert small < 4000 * 0.5
    assert large / small < 2.5


def test_exclusion_tiny_sets_and_nearest(fm):
    X = np.random.default_rng(9).random((5, 3))
    ix = fm.NeighborIndex.build(X, fm.IndexMode.ApproxGraph)
    nl = ix.query_knn(X[2], 4, 2)
    assert len(nl.indices) == 4 and 2 not in nl.indices and len(set(nl.indices)) == 4
    Y = np.random.default_rng(10).random((4000, 3))
    g = fm.NeighborIndex.build(Y, fm.IndexMode.ApproxGraph)
    Z = np.random.default_rng(11).random((500, 3))
    ex = fm.NeighborIndex.build(Y)
    assert np.mean(g.nearest_batch(Z) == ex.nearest_batch(Z)) >= 0.99
    # self-exclusion as precompute uses it: the k nearest others of a stored point
    rows = np.arange(0, 4000, 37)
    gi, _ = g.query_knn_batch(Y[rows], 8, rows.astype(np.int32))
    assert not np.any(gi == rows[:, None])


def test_serialized_graph_round_trips(fm):
    X = np.random.default_rng(10).random((800, 6))
    p = fm.GraphParams(seed=3)
    ix = fm.NeighborIndex.build(X, fm.IndexMode.ApproxGraph, p)
    arrs = ix.graph_arrays()
    copy = fm.NeighborIndex.from_graph_arrays(X, p, *arrs)
    a2 = copy.graph_arrays()
    for u, v in zip(arrs[2:], a2[2:]):
        assert np.array_equal(u, v)
    Q = np.random.default_rng(11).random((20, 6))
    ia, da = ix.query_knn_batch(Q, 15)
    ib, db = copy.query_knn_batch(Q, 15)
    assert np.array_equal(ia, ib) and np.array_equal(da, db)
