"""GPU parity on WHOLE BASELINE tables (configs 2-5 at their full sizes):
every neighbour row of the production search (cell grid for d <= 3, tcgen05
filter + fp64 recheck for d >= 4, including its overflow-redo path) and every
test point's 1-NN, compared with the fp64 brute-force kernel (FMGP_KNN=brute,
itself pinned to the oracle and the reference in test_gpu_knn.py /
test_gpu_parity.py): indices and dist_sq keys bit-exact. The brute-force runs
take up to a few minutes each on a B200 (cfg4: 4e12 pairs of 40-d keys)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent


def _dump(cfg, what, prefix, brute):
    env = dict(os.environ)
    env.pop("FMGP_KNN", None)
    if brute:
        env["FMGP_KNN"] = "brute"
    r = subprocess.run([sys.executable, str(HERE / "fulltable_dump.py"), str(cfg), what, str(prefix)], env=env,
                       capture_output=True, text=True, timeout=3000)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_every_neighbour_row_matches_brute_force(fm, tmp_path, cfg):
    _dump(cfg, "self", tmp_path / "prod", False)
    _dump(cfg, "self", tmp_path / "brute", True)
    a_i, b_i = np.load(tmp_path / "prod_idx.npy"), np.load(tmp_path / "brute_idx.npy")
    bad = np.flatnonzero(np.any(a_i != b_i, axis=1))
    assert bad.size == 0, f"cfg{cfg}: {bad.size} of {a_i.shape[0]} rows differ, first {bad[:10].tolist()}"
    a_d, b_d = np.load(tmp_path / "prod_dsq.npy"), np.load(tmp_path / "brute_dsq.npy")
    assert np.array_equal(a_d.view(np.int64), b_d.view(np.int64)), f"cfg{cfg}: dist_sq keys differ"


@pytest.mark.parametrize("cfg", [2, 3, 4, 5])
def test_every_test_point_nearest_matches_brute_force(fm, tmp_path, cfg):
    _dump(cfg, "nn", tmp_path / "prod", False)
    _dump(cfg, "nn", tmp_path / "brute", True)
    a, b = np.load(tmp_path / "prod_nn.npy"), np.load(tmp_path / "brute_nn.npy")
    bad = np.flatnonzero(a != b)
    assert bad.size == 0, f"cfg{cfg}: {bad.size} of {a.size} test points differ, first {bad[:10].tolist()}"
