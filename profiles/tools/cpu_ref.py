"""The reference's own CPU implementation (oracle/_ref, all host threads) on a
bounded random row sample of every BASELINE config (precompute train-pts/s),
the same procedure as bench.py's cpu_baseline leg. One JSON line per config.
    python profiles/tools/cpu_ref.py [--configs 1,2,3,4,5] [--budget 10]"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--budget", type=float, default=10.0)
    a = ap.parse_args()
    from oracle.oracle import best_available, host_threads
    from paper_2205_10879_b200 import datagen
    import bench
    orc = best_available()
    thr = host_threads()
    for cfg in (int(c) for c in a.configs.split(",")):
        info = datagen.config_info(cfg)
        ds = datagen.generate(cfg, info.n, 16)
        nrows, kp = bench.rows_sample_rate(orc, ds, info, thr, a.budget, cfg)
        rows = np.sort(np.random.default_rng(cfg).choice(info.n, size=nrows, replace=False)).astype(np.int64)
        t = time.perf_counter()
        orc.precompute_rows(ds.X, ds.Y, *kp, info.k, rows, threads=thr)
        dt = time.perf_counter() - t
        print(json.dumps({"cfg": cfg, "kind": orc.kind, "threads": thr, "rows": nrows, "seconds": dt,
                          "precompute_train_pts_per_s": nrows / dt}), flush=True)


if __name__ == "__main__":
    main()
