"""FastMuyGPs B200 benchmark — precompute train-pts/s (+ predict test-pts/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl b200|reference]

A step is one pass of the hot path over one batch: the precompute of all
n_train rows of the BASELINE config (exact kNN -> kernel matrices ->
jitter-Cholesky -> coefficient table C), sharded by rows over the ranks with
the S/C shards all-gathered over NCCL when N > 1. The predict stage (1-NN ->
cross-covariance -> dot) over all n_test points is timed the same way and
reported under "predict". Inputs are resident in HBM when the timed region
starts (`value`); `e2e` is the same metric through the host-buffer C ABI
(fmgp_precompute) with pinned host buffers, H2D/D2H inside the timed region.

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events
on the launching stream; L2 is flushed (256 MiB write) between timed steps,
outside the events; barrier + synchronize around the timed region; the max
over ranks is reported. Data: seeded synthetic inputs with the config's
shapes and distributions; the paper's datasets are not
available.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--n", type=int, default=None, help="override n_train (debug only; not a bench line)")
    ap.add_argument("--nt", type=int, default=None, help="override n_test (debug only)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text()), "measured"
        except Exception:
            pass
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def fp64_peak():
    """FP64 peak measured on this box by profiles/tools (DADD/DMUL op rate), if recorded."""
    p = REPO / "profiles" / "fp64_peak.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            return None
    return None


# ---------------------------------------------------------------------------- reference arm

def run_reference(args, cfg_info, ds):
    """--impl reference: the reference's own CPU implementation (oracle/_ref when
    it was compiled from /root/reference, else the C port), all host threads,
    on a bounded row sample per step. Rank 0 only."""
    from oracle.oracle import best_available, host_threads
    ws, rank, _ = dist_env()
    if rank != 0:
        return None
    orc = best_available()
    thr = host_threads()
    info = cfg_info
    kp = (info.kind, info.sigma, info.rho, info.nu, info.tau)
    # Size the per-step sample: ~10 s of wall per step in total over W+K steps budget.
    probe = np.arange(0, min(info.n, 2 * thr), dtype=np.int64)
    t = time.perf_counter()
    orc.precompute_rows(ds.X, ds.Y, *kp, info.k, probe, threads=thr)
    per_row = (time.perf_counter() - t) / probe.size
    total_steps = args.steps + args.warmup
    rows_per_step = int(max(thr, min(info.n, (150.0 / total_steps) / max(per_row, 1e-9))))
    rng = np.random.default_rng(0)
    times = []
    for s in range(total_steps):
        rows = np.sort(rng.choice(info.n, size=rows_per_step, replace=False)).astype(np.int64)
        t = time.perf_counter()
        orc.precompute_rows(ds.X, ds.Y, *kp, info.k, rows, threads=thr)
        dt = time.perf_counter() - t
        if s >= args.warmup:
            times.append(dt)
    total = sum(times)
    value = rows_per_step * len(times) / total
    return {
        "metric": "precompute train-pts/s", "value": value, "unit": "train-pts/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg{info.cfg}", "d": info.d, "n_train": info.n, "k": info.k, "m": info.m,
                   "sample_rows_per_step": rows_per_step},
        "cpu_baseline": {"value": value, "unit": "train-pts/s", "cores": thr, "kind": orc.kind,
                         "sample": f"{rows_per_step} random training rows of cfg{info.cfg} per step (kNN against "
                                   f"all {info.n} points + local solve), {thr} threads"},
        "e2e": {"value": value, "unit": "train-pts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def cpu_baseline(info, ds, budget_s=12.0):
    """The reference CPU implementation on a bounded sample of the same workload (rank 0, N=1)."""
    from oracle.oracle import best_available, host_threads
    orc = best_available()
    thr = host_threads()
    kp = (info.kind, info.sigma, info.rho, info.nu, info.tau)
    probe = np.arange(0, min(info.n, 2 * thr), dtype=np.int64)
    t = time.perf_counter()
    orc.precompute_rows(ds.X, ds.Y, *kp, info.k, probe, threads=thr)
    per_row = (time.perf_counter() - t) / probe.size
    nrows = int(max(thr, min(info.n, budget_s / max(per_row, 1e-9))))
    rows = np.sort(np.random.default_rng(1).choice(info.n, size=nrows, replace=False)).astype(np.int64)
    t = time.perf_counter()
    orc.precompute_rows(ds.X, ds.Y, *kp, info.k, rows, threads=thr)
    dt = time.perf_counter() - t
    return {"value": nrows / dt, "unit": "train-pts/s", "cores": thr, "kind": orc.kind,
            "sample": f"{nrows} random training rows of cfg{info.cfg} (full-n kNN + solve each), {thr} threads, "
                      f"{dt:.1f} s"}


# ---------------------------------------------------------------------------- B200 arm

def main():
    args = parse()
    ws, rank, local = dist_env()
    from paper_2205_10879_b200 import datagen
    info = datagen.config_info(args.config)
    n = args.n or info.n
    nt = args.nt or info.n_test

    if args.impl == "reference":
        if rank != 0:
            return 0
        ds = datagen.generate(args.config, n, min(nt, 1000))
        info.n = n
        line = run_reference(args, info, ds)
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2205_10879_b200 as fm
    from paper_2205_10879_b200 import _native as N
    dev = torch.device("cuda", local)

    ds = datagen.generate(args.config, n, nt)
    X = torch.from_numpy(ds.X).to(dev)
    Y = torch.from_numpy(ds.Y).to(dev)
    Z = torch.from_numpy(ds.Z).to(dev)
    k, m = info.k, info.m
    fit = fm.FittedParams(fm.KernelParams(info.sigma, info.rho, info.nu, info.tau), fm.KernelKind(info.kind))

    # row / test shards (contiguous, rank-ordered)
    def shard(total):
        per = (total + ws - 1) // ws
        b = min(total, rank * per)
        return b, min(total, b + per), per

    rb, re_, per = shard(n)
    zb, ze, zper = shard(nt)
    S_full = torch.empty((per * ws, k), dtype=torch.int32, device=dev)
    C_full = torch.empty((per * ws, k, m), dtype=torch.float64, device=dev)
    S_loc = S_full[rank * per: rank * per + per]
    C_loc = C_full[rank * per: rank * per + per]
    out = torch.empty((zper, m), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def precompute_step():
        fm.precompute_device(X, Y, fit, k, rb, re_, S_loc, C_loc, stream)
        if ws > 1:
            dist.all_gather_into_tensor(S_full, S_loc.contiguous())
            dist.all_gather_into_tensor(C_full, C_loc.contiguous())

    S_all = S_full[:n]
    C_all = C_full[:n]

    def predict_step():
        fm.predict_device(X, S_all, C_all.reshape(n, k, m), fit, ds.mean_offset, Z[zb:ze], out[: ze - zb], None,
                          stream)

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        ms = []
        for _ in range(steps):
            flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        t = torch.tensor([sum(ms)], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()) / steps, ms

    with ClockSampler(local) as clk:
        pre_ms, pre_all = timed(precompute_step, args.steps, args.warmup)
        pred_ms, pred_all = timed(predict_step, args.steps, args.warmup)
    clocks = clk.summary()

    # per-kernel share: time the kNN scan alone inside the same process (events)
    knn_ms = None
    if ws == 1:
        idx_tmp = torch.empty((n, k - 1), dtype=torch.int32, device=dev)
        import ctypes
        def knn_only():
            rc = N.LIB.fmgp_query_knn_device(ctypes.c_void_p(X.data_ptr()), n, info.d, ctypes.c_void_p(X.data_ptr()),
                                             n, k - 1, 0, ctypes.c_void_p(idx_tmp.data_ptr()), None,
                                             ctypes.c_void_p(stream.cuda_stream))
            N.check(rc)
        knn_ms, _ = timed(knn_only, max(1, min(3, args.steps)), 1)
        del idx_tmp

    value = n / (pre_ms / 1e3)
    pred_value = nt / (pred_ms / 1e3)

    e2e = None
    if not args.no_e2e and ws == 1:
        Xh = torch.from_numpy(ds.X).pin_memory()
        Yh = torch.from_numpy(ds.Y).pin_memory()
        Sh = torch.empty((n, k), dtype=torch.int32).pin_memory()
        Ch = torch.empty((n, k, m), dtype=torch.float64).pin_memory()
        kp = fit.theta_hat.c(fit.kind)
        failed = C.c_int64(-1)

        def e2e_step():
            rc = N.LIB.fmgp_precompute(C.c_void_p(Xh.data_ptr()), C.c_void_p(Yh.data_ptr()), n, info.d, m,
                                       C.byref(kp), k, C.c_void_p(Sh.data_ptr()), C.c_void_p(Ch.data_ptr()),
                                       C.byref(failed))
            N.check(rc, failed.value)

        for _ in range(args.warmup):
            e2e_step()
        ts = []
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            t = time.perf_counter()
            e2e_step()
            ts.append(time.perf_counter() - t)
        e2e = {"value": n / (sum(ts) / len(ts)), "unit": "train-pts/s",
               "h2d_bytes_per_step": int(Xh.numel() * 8 + Yh.numel() * 8),
               "d2h_bytes_per_step": int(Sh.numel() * 4 + Ch.numel() * 8),
               "api": "fmgp_precompute (include/fmgp_b200.h), pinned host buffers"}

    # roofline of the dominant kernel (exact kNN scan, FP64 pipe)
    pairs = float(n) * float(n)
    fp64_ops = pairs * (3 * info.d - 1)
    fpk = fp64_peak()
    roof = None
    if knn_ms is not None:
        achieved = fp64_ops / (knn_ms / 1e3) / 1e12
        peak = fpk["fp64_tops_nonfma"] if fpk else None
        roof = {"bound": "fp64", "kernel": "knn_scan_reg", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s", "frac": (achieved / peak) if peak else None,
                "traffic": None, "work": f"{pairs:.3g} (query, point) pairs x {3 * info.d - 1} fp64 ops",
                "kernel_ms": knn_ms, "share_of_step": knn_ms / pre_ms,
                "peak_source": "profiles/fp64_peak.json (DADD/DMUL rate measured on B200)" if fpk else "unmeasured"}

    line = {
        "metric": "precompute train-pts/s", "value": value, "unit": "train-pts/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": pre_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg{info.cfg}", "d": info.d, "n_train": n, "n_test": nt, "k": k, "m": m,
                   "kernel": "RBF" if info.kind == 1 else f"Matern nu={info.nu}", "parallelism": f"rows{ws}",
                   "l2": "flushed (256 MiB write) between timed steps"},
        "predict": {"metric": "predict test-pts/s", "value": pred_value, "unit": "test-pts/s", "ms_per_step": pred_ms},
        "e2e": e2e,
        "roofline": roof,
        "clocks": clocks,
        "gpu_launches": None,
        "step_ms": {"precompute": pre_all, "predict": pred_all},
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(info, ds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
