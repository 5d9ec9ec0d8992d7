"""FastMuyGPs B200 benchmark — precompute train-pts/s (+ predict test-pts/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

A step is one pass of the hot path over one batch: the precompute of all
n_train rows of the BASELINE config (exact kNN -> kernel matrices ->
jitter-Cholesky -> coefficient table C). Rows are sharded contiguously over
the ranks (paper_2205_10879_b200/parallel.py) and the S / C shards are
all-gathered over NCCL when N > 1, so every rank ends the step with the whole
model. The predict stage (1-NN -> cross-covariance -> dot) over all n_test
points, sharded the same way, is timed identically and reported under
"predict". `value` has the inputs resident in HBM; `e2e` is the same metric
through the host-buffer C ABI (fmgp_precompute, include/fmgp_b200.h) with
pinned host buffers and H2D/D2H inside the timed region.

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events
on the launching stream; L2 is flushed (256 MiB write) between timed steps,
outside the events; barrier + synchronize around the timed region; the max
over ranks is reported. Data: seeded synthetic inputs with the config's
shapes and distributions; the paper's datasets are not in
the image.
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
    ap.add_argument("--n", type=int, default=None, help="override n_train (debug; not a bench line)")
    ap.add_argument("--nt", type=int, default=None, help="override n_test (debug)")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


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

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(s[0]) for s in self.samples) if v is not None]
        mx = [v for v in (num(s[1]) for s in self.samples) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and
                          s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def load_json(path: Path):
    try:
        return json.loads(path.read_text())
    except Exception:
        return None


def peaks():
    mp = load_json(REPO / "MEASURED_PEAKS.json")
    hbm = (mp or {}).get("hbm_gbs")
    return {"hbm_gbs": hbm or 6650.0, "hbm_src": "measured (MEASURED_PEAKS.json)" if hbm else "fallback",
            "fp64": load_json(REPO / "profiles" / "fp64_peak.json")}


# ---------------------------------------------------------------------------- reference arm

def rows_sample_rate(orc, ds, info, thr, budget_s, seed):
    kp = (info.kind, info.sigma, info.rho, info.nu, info.tau)
    probe = np.arange(0, min(info.n, 8 * thr), dtype=np.int64)
    orc.precompute_rows(ds.X, ds.Y, *kp, info.k, probe[:thr], threads=thr)  # warm (index build, pages)
    t = time.perf_counter()
    orc.precompute_rows(ds.X, ds.Y, *kp, info.k, probe, threads=thr)
    per_row = (time.perf_counter() - t) / probe.size
    nrows = int(max(thr, min(info.n, budget_s / max(per_row, 1e-9))))
    return nrows, kp


def run_reference(args, info, ds):
    """--impl reference: the reference's own CPU implementation (oracle/_ref when
    it was compiled from /root/reference, else the C port), all host threads, on
    a bounded random row sample per step. Rank 0 only."""
    from oracle.oracle import best_available, host_threads
    orc = best_available()
    thr = host_threads()
    total_steps = args.steps + args.warmup
    nrows, kp = rows_sample_rate(orc, ds, info, thr, 150.0 / total_steps, 0)
    rng = np.random.default_rng(0)
    times = []
    for s in range(total_steps):
        rows = np.sort(rng.choice(info.n, size=nrows, replace=False)).astype(np.int64)
        t = time.perf_counter()
        orc.precompute_rows(ds.X, ds.Y, *kp, info.k, rows, threads=thr)
        if s >= args.warmup:
            times.append(time.perf_counter() - t)
    value = nrows * len(times) / sum(times)
    return {
        "metric": "precompute train-pts/s", "value": value, "unit": "train-pts/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg{info.cfg}", "d": info.d, "n_train": info.n, "k": info.k, "m": info.m,
                   "sample_rows_per_step": nrows},
        "cpu_baseline": {"value": value, "unit": "train-pts/s", "cores": thr, "kind": orc.kind,
                         "sample": f"{nrows} random training rows of cfg{info.cfg} per step (exact kNN against "
                                   f"all {info.n} points + local solve each), {thr} threads"},
        "e2e": {"value": value, "unit": "train-pts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def cpu_baseline(info, ds, budget_s=12.0):
    """The reference CPU implementation on a bounded sample of the same workload (rank 0, N=1)."""
    from oracle.oracle import best_available, host_threads
    orc = best_available()
    thr = host_threads()
    nrows, kp = rows_sample_rate(orc, ds, info, thr, budget_s, 1)
    rows = np.sort(np.random.default_rng(1).choice(info.n, size=nrows, replace=False)).astype(np.int64)
    t = time.perf_counter()
    orc.precompute_rows(ds.X, ds.Y, *kp, info.k, rows, threads=thr)
    dt = time.perf_counter() - t
    return {"value": nrows / dt, "unit": "train-pts/s", "cores": thr, "kind": orc.kind,
            "sample": f"{nrows} random training rows of cfg{info.cfg} (exact kNN against all {info.n} points + "
                      f"local solve each), {thr} threads, {dt:.1f} s"}


# ---------------------------------------------------------------------------- B200 arm

def solve_flops_per_row(info):
    """F = k^3/3 + 2 k^2 m + 3 d k(k-1)/2 fp64 flops per training row."""
    k, m, d = info.k, info.m, info.d
    return k ** 3 / 3 + 2 * k * k * m + 3 * d * k * (k - 1) / 2


def predict_bytes_per_point(info):
    """4k + 8km + 8kd + 8d + 8m HBM bytes per test point."""
    k, m, d = info.k, info.m, info.d
    return 4 * k + 8 * k * m + 8 * k * d + 8 * d + 8 * m


def main():
    args = parse()
    ws, rank, local = dist_env()
    from paper_2205_10879_b200 import datagen
    info = datagen.config_info(args.config)
    if args.n:
        info.n = args.n
    if args.nt:
        info.n_test = args.nt
    n, nt = info.n, info.n_test

    if args.impl == "reference":
        if rank != 0:
            return 0
        ds = datagen.generate(args.config, n, min(nt, 1000))
        print(json.dumps(run_reference(args, info, ds)), flush=True)
        return 0

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2205_10879_b200 as fm
    from paper_2205_10879_b200 import _native as N
    from paper_2205_10879_b200.parallel import overlapped_precompute, sharded_precompute, sharded_predict
    dev = torch.device("cuda", local)

    ds = datagen.generate(args.config, n, nt)
    X = torch.from_numpy(ds.X).to(dev)
    Y = torch.from_numpy(ds.Y).to(dev)
    Z = torch.from_numpy(ds.Z).to(dev)
    k, m, d = info.k, info.m, info.d
    fit = fm.FittedParams(fm.KernelParams(info.sigma, info.rho, info.nu, info.tau), fm.KernelKind(info.kind))
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    state = {}

    def shard(b, e):
        S = torch.empty((e - b, k), dtype=torch.int32, device=dev)
        Cm = torch.empty((e - b, k, m), dtype=torch.float64, device=dev)
        fm.precompute_device(X, Y, fit, k, b, e, S, Cm, stream)
        return S, Cm

    kp_c = fit.theta_hat.c(fit.kind)
    fail_word = torch.full((1,), -1, dtype=torch.int64, device=dev)  # UINT64_MAX: no failed row

    def knn_rows(b, e):  # K1 for rows [b, e): precompute's S rows
        S = torch.empty((e - b, k), dtype=torch.int32, device=dev)
        N.check(N.LIB.fmgp_knn_rows_device(C.c_void_p(X.data_ptr()), n, d, k, b, e, C.c_void_p(S.data_ptr()),
                                           C.c_void_p(stream.cuda_stream)))
        return S

    def solve_rows(S_rows, row_begin, C_out):  # K2 for a chunk, asynchronous (failures -> fail_word)
        N.check(N.LIB.fmgp_solve_rows_device(C.c_void_p(X.data_ptr()), C.c_void_p(Y.data_ptr()), n, d, m,
                                             C.byref(kp_c), k, C.c_void_p(S_rows.data_ptr()), S_rows.shape[0],
                                             row_begin, C.c_void_p(C_out.data_ptr()),
                                             C.c_void_p(fail_word.data_ptr()), None, C.c_void_p(stream.cuda_stream)))

    def precompute_step():
        if ws == 1:
            state["S"], state["C"] = sharded_precompute(n, shard)
        else:  # K1 per shard; S and each C chunk all-gathered while the next chunk is solved
            state["S"], state["C"] = overlapped_precompute(n, k, m, knn_rows, solve_rows, nchunks=4, device=dev)

    def predict_step():
        def pshard(b, e):
            out = torch.empty((e - b, m), dtype=torch.float64, device=dev)
            fm.predict_device(X, state["S"], state["C"], fit, ds.mean_offset, Z[b:e], out, None, stream)
            return out
        state["P"] = sharded_predict(nt, pshard)

    def timed(fn, steps, warmup, stage_events=False):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        ms = []
        if stage_events:  # kernel-stage CUDA events on the launch stream, inside the timed region
            N.LIB.fmgp_stage_times(None, None, None)
            N.LIB.fmgp_set_stage_timing(1)
        l0 = N.LIB.fmgp_launch_count()
        for _ in range(steps):
            flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        launches = N.LIB.fmgp_launch_count() - l0
        if stage_events:
            N.LIB.fmgp_set_stage_timing(0)
            a, b, c = C.c_double(0), C.c_double(0), C.c_int64(0)
            N.check(N.LIB.fmgp_stage_times(C.byref(a), C.byref(b), C.byref(c)))
            state["stage"] = {"knn_ms_per_launch": a.value / max(c.value, 1),
                              "solve_ms_per_launch": b.value / max(c.value, 1), "launches": c.value}
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        t = torch.tensor([sum(ms)], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()) / steps, ms, launches

    with ClockSampler(local) as clk:
        pre_ms, pre_all, pre_launch = timed(precompute_step, args.steps, args.warmup, stage_events=True)
        pred_ms, pred_all, pred_launch = timed(predict_step, args.steps, args.warmup)
    clocks = clk.summary()
    if int(fail_word.item()) != -1:
        raise RuntimeError(f"precompute: Cholesky factorization failed in row {int(fail_word.item()) & ((1 << 64) - 1)}")
    stage = state.get("stage", {})
    knn_ms = stage.get("knn_ms_per_launch")
    solve_ms = stage.get("solve_ms_per_launch")

    value = n / (pre_ms / 1e3)
    pred_value = nt / (pred_ms / 1e3)

    # e2e: the reference-facing host-buffer call, pinned buffers, copies inside the
    # timing. One process per GPU: each rank passes the full X, Y and receives its
    # row shard of S and C (fmgp_precompute_rows; = fmgp_precompute at N=1); the
    # step time is the max over ranks.
    e2e = None
    if not args.no_e2e:
        from paper_2205_10879_b200.parallel import shard_bounds
        rb, re_, _ = shard_bounds(n, ws, rank)
        Xh = torch.from_numpy(ds.X).pin_memory()
        Yh = torch.from_numpy(ds.Y).pin_memory()
        Sh = torch.empty((re_ - rb, k), dtype=torch.int32).pin_memory()
        Ch = torch.empty((re_ - rb, k, m), dtype=torch.float64).pin_memory()
        kp = fit.theta_hat.c(fit.kind)
        failed = C.c_int64(-1)

        def e2e_step():
            N.check(N.LIB.fmgp_precompute_rows(C.c_void_p(Xh.data_ptr()), C.c_void_p(Yh.data_ptr()), n, d, m,
                                               C.byref(kp), k, rb, re_, C.c_void_p(Sh.data_ptr()),
                                               C.c_void_p(Ch.data_ptr()), C.byref(failed)), failed.value)

        for _ in range(args.warmup):
            e2e_step()
        ts = []
        for _ in range(args.steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            if ws > 1:
                dist.barrier()
            t = time.perf_counter()
            e2e_step()
            ts.append(time.perf_counter() - t)
        tt = torch.tensor([sum(ts) / len(ts)], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": n / float(tt.item()), "unit": "train-pts/s",
               "h2d_bytes_per_step": int(Xh.numel() * 8 + Yh.numel() * 8),
               "d2h_bytes_per_step": int(Sh.numel() * 4 + Ch.numel() * 8),
               "api": "fmgp_precompute_rows (include/fmgp_b200.h; = fmgp_precompute at N=1), pinned host "
                      "buffers, per rank: full X/Y in, its row shard of S/C out; max over ranks"}

    # roofline of the dominant kernel of the step: algorithmic work per launch /
    # that kernel's average launch duration (CUDA events on its stream, above)
    pk = peaks()
    fp64 = pk["fp64"] or {}
    traffic = load_json(REPO / "profiles" / "r01" / "traffic.json") or {}
    roof = None
    if solve_ms is not None and knn_ms is not None:
        rows_per_rank = (n + ws - 1) // ws
        if solve_ms >= knn_ms:
            flops = solve_flops_per_row(info) * rows_per_rank
            achieved = flops / (solve_ms / 1e3) / 1e12
            peak = fp64.get("fp64_dfma_tflops")
            tr = traffic.get(f"cfg{info.cfg}", {}).get("solve")
            roof = {"bound": "fp64", "kernel": "fused solve (gather / kernel build / jitter-Cholesky / solve, "
                    "FP64 pipe)", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak if peak else None,
                    "traffic": tr["dram_bytes_per_launch"] * rows_per_rank / tr["rows"] if tr else None,
                    "traffic_source": tr.get("source") if tr else None,
                    "work": f"{solve_flops_per_row(info):.0f} fp64 flops per training row (SURVEY 8(d): k^3/3 + "
                            f"2k^2m + 3d k(k-1)/2; kernel evaluations not counted) x {rows_per_rank} rows",
                    "kernel_ms": solve_ms, "share_of_step": solve_ms / pre_ms,
                    "peak_source": "profiles/fp64_peak.json: measured DFMA rate on this B200 (neither HBM nor the "
                                   "tensor pipe bounds an fp64 Cholesky; MEASURED_PEAKS.json has no fp64 figure)"}
        else:
            tr = traffic.get(f"cfg{info.cfg}", {}).get("knn")
            roof = {"bound": "fp64", "kernel": "kNN stage", "achieved": None,
                    "peak": fp64.get("fp64_tops_nonfma"), "unit": "TFLOP/s", "frac": None,
                    "traffic": tr["dram_bytes_per_launch"] if tr else None,
                    "kernel_ms": knn_ms, "share_of_step": knn_ms / pre_ms}
    tr_pred = traffic.get(f"cfg{info.cfg}", {}).get("predict")
    pred_traffic = tr_pred["dram_bytes_per_launch"] * ((nt + ws - 1) // ws) / tr_pred["points"] if tr_pred else None
    pred_bytes = predict_bytes_per_point(info) * ((nt + ws - 1) // ws)
    pred_gbs = pred_bytes / (pred_ms / 1e3) / 1e9

    line = {
        "metric": "precompute train-pts/s", "value": value, "unit": "train-pts/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": pre_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg{info.cfg}", "d": d, "n_train": n, "n_test": nt, "k": k, "m": m,
                   "kernel": "RBF" if info.kind == 1 else f"Matern nu={info.nu}", "parallelism": f"rows{ws}",
                   "l2": "flushed (256 MiB write) between timed steps"},
        "predict": {"metric": "predict test-pts/s", "value": pred_value, "unit": "test-pts/s", "ms_per_step": pred_ms,
                    "roofline": {"bound": "hbm", "achieved": pred_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                                 "frac": pred_gbs / pk["hbm_gbs"], "peak_source": pk["hbm_src"],
                                 "work": f"{predict_bytes_per_point(info)} B per test point (SURVEY §8(d)); the "
                                         "stage also runs the grid 1-NN", "traffic": pred_traffic},
                    "gpu_launches": pred_launch},
        "stages_ms": {"knn": knn_ms, "solve": solve_ms, "precompute": pre_ms, "predict": pred_ms},
        "e2e": e2e,
        "roofline": roof,
        "clocks": clocks,
        "gpu_launches": pre_launch,
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
