"""FastMuyGPs B200 benchmark — precompute train-pts/s and predict test-pts/s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl b200|reference]

`--gpus N` with N > 1 outside torchrun re-launches itself under
`python -m torch.distributed.run --nproc-per-node N` (one process per GPU);
under torchrun (WORLD_SIZE set) it runs as one rank.

Workload: BASELINE.json configs[4] ("cfg5": d = 3, n_train = n_test = 8e6,
k = 50, Matern nu = 2.5, fp64), the config the 1/2/4/8-GPU metric is quoted
on and the largest one; it fits one B200. Other configs (`--config 1..4`)
are parity-test cases and A/B runs, not bench lines.

A precompute step is one pass of the hot path over all n_train rows (exact
kNN -> kernel matrices -> jitter-Cholesky -> coefficient table C) through the
C ABI's group call (fmgp_group_precompute_device, include/fmgp_b200.h): rows
dealt block-cyclically over the ranks, S and C all-gathered in place over
NVLink (NCCL from C++) while the next round is solved, so every rank ends the
step holding the whole model. A predict step is the 1-NN -> cross-covariance
-> dot pass over all n_test points, test points split contiguously over the
ranks, through the device-resident model handle (fmgp_model_predict_device).
`value` / `predict.value` have the inputs resident in HBM; `e2e` (and
`predict.e2e`) is the same metric through the host-buffer C ABI with pinned
host buffers, host<->device copies inside the timed region: fmgp_precompute
at N = 1 (the call the C++ facade's precompute makes), fmgp_group_precompute
at N > 1; fmgp_model_predict for predict.

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events
on the launching stream; L2 is flushed (256 MiB write) between timed steps,
outside the events; barrier + synchronize around the timed region; the max
over ranks is reported. Before the warm-up the process idles for --settle
seconds (default 20, reported as config.settle_s): run within seconds of a
CPU-heavy process exiting (the reference arm), two or three of the first
steps show 5-15 ms host-side stalls (profiles/r02/README.md), gone after 30 s. Data: seeded synthetic inputs with the config's
shapes and distributions; the paper's datasets are not in
the image. The CPU baselines are the reference's own TUs (oracle/_ref) on
bounded samples of the same workload, on the box's host cores (rank 0, N=1).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
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
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--settle", type=float, default=20.0,
                    help="seconds to idle before the warm-up (outside every timed region): for ~30 s after a CPU-heavy "
                         "process such as the reference arm exits, a few steps show 5-15 ms host-side stalls")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--n", type=int, default=None, help="override n_train (debug; not a bench line)")
    ap.add_argument("--nt", type=int, default=None, help="override n_test (debug)")
    ap.add_argument("--probe-launch", action="store_true",
                    help="launcher check: every rank joins a gloo group, rank 0 prints the rank count and exits")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def relaunch_under_torchrun(args) -> int:
    """`--gpus N` outside torchrun: one process per GPU via torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


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
            self._stop.wait(float(os.environ.get("FMGP_BENCH_SMI_INTERVAL", "0.2")))

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


def hbm_peak():
    mp = load_json(REPO / "MEASURED_PEAKS.json")
    hbm = (mp or {}).get("hbm_gbs")
    if hbm:
        return hbm, "measured (MEASURED_PEAKS.json, driver-written)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def solve_flops_per_row(info):
    """F = k^3/3 + 2 k^2 m + 3 d k(k-1)/2 fp64 flops per training row."""
    k, m, d = info.k, info.m, info.d
    return k ** 3 / 3 + 2 * k * k * m + 3 * d * k * (k - 1) / 2


def predict_bytes_per_point(info):
    """4k + 8km + 8kd + 8d + 8m HBM bytes per test point."""
    k, m, d = info.k, info.m, info.d
    return 4 * k + 8 * k * m + 8 * k * d + 8 * d + 8 * m


# ---------------------------------------------------------------------------- CPU reference legs

def rows_sample_rate(orc, ds, info, thr, budget_s):
    kp = (info.kind, info.sigma, info.rho, info.nu, info.tau)
    probe = np.arange(0, min(info.n, 8 * thr), dtype=np.int64)
    orc.precompute_rows(ds.X, ds.Y, *kp, info.k, probe[:thr], threads=thr)  # warm (index build, pages)
    t = time.perf_counter()
    orc.precompute_rows(ds.X, ds.Y, *kp, info.k, probe, threads=thr)
    per_row = (time.perf_counter() - t) / probe.size
    nrows = int(max(thr, min(info.n, budget_s / max(per_row, 1e-9))))
    return nrows, kp


def cpu_precompute_baseline(orc, info, ds, thr, budget_s, seed):
    """The reference's precompute body (fast_predict.cpp:89-107) on a random row sample, all host threads."""
    nrows, kp = rows_sample_rate(orc, ds, info, thr, budget_s)
    rows = np.sort(np.random.default_rng(seed).choice(info.n, size=nrows, replace=False)).astype(np.int64)
    t = time.perf_counter()
    orc.precompute_rows(ds.X, ds.Y, *kp, info.k, rows, threads=thr)
    dt = time.perf_counter() - t
    return {"value": nrows / dt, "unit": "train-pts/s", "cores": thr, "kind": orc.kind,
            "sample": f"{nrows} random training rows of cfg{info.cfg} (exact kNN against all {info.n} points + "
                      f"local solve each), {thr} threads, {dt:.1f} s"}


def cpu_predict_baseline(orc, info, X, S, Cm, mean_offset, Z, thr, budget_s, table_note):
    """The reference's predict on a bounded sample of the test points: fast_predict_batch single-threaded
    (fast_predict.cpp:146-156, as the reference runs it) and, labelled, fast_predict_one over `thr` host
    threads (concurrent callers on a shared model, fast_predict.hpp:20-24)."""
    kp = (info.kind, info.sigma, info.rho, info.nu, info.tau)
    ss = orc.predict_session(X, S, Cm, *kp, mean_offset)
    try:
        t = time.perf_counter()
        ss.run(Z[:2], 1)
        per = max((time.perf_counter() - t) / 2, 1e-7)
        n1 = int(max(2, min(Z.shape[0], budget_s / 2 / per)))
        t = time.perf_counter()
        ss.run(Z[:n1], 1)
        v1 = n1 / (time.perf_counter() - t)
        nt = int(max(thr, min(Z.shape[0], budget_s / 2 * v1 * thr)))
        t = time.perf_counter()
        ss.run(Z[:nt], thr)
        dtt = time.perf_counter() - t
    finally:
        ss.close()
    return {"value": nt / dtt, "unit": "test-pts/s", "cores": thr, "kind": orc.kind,
            "sample": f"first {nt} test points of cfg{info.cfg}, fast_predict_one on {thr} host threads "
                      f"(1-NN scan of all {info.n} training points + k-term dot each); {table_note}",
            "single_thread": {"value": v1, "unit": "test-pts/s", "cores": 1,
                              "sample": f"first {n1} test points, fast_predict_batch (the reference's own "
                                        "single-threaded batch loop)"}}


def synthetic_table(n, k, m, seed):
    """A model table with the reference's layout (S[i,0] = i, then k-1 distinct other indices; C a random
    k x m block repeated) for timing the reference's predict where no precomputed model exists: its per-point
    cost is the 1-NN scan plus k kernel terms, independent of the table's values."""
    S = np.empty((n, k), dtype=np.int32)
    i = np.arange(n, dtype=np.int32)
    S[:, 0] = i
    stride = max(1, n // max(k, 1))
    for j in range(1, k):
        S[:, j] = (i + np.int32(j * stride)) % np.int32(n)
    blk = np.random.default_rng(seed).standard_normal((1, k, m))
    Cm = np.broadcast_to(blk, (n, k, m))
    return S, Cm


def run_reference(args, info):
    """--impl reference: the reference's own CPU implementation (oracle/_ref, the reference's TUs compiled
    from /root/reference), all host threads, bounded samples per step. Rank 0 only."""
    from paper_2205_10879_b200 import datagen
    from oracle.oracle import best_available, host_threads
    orc = best_available()
    thr = host_threads()
    ds = datagen.generate(args.config, info.n, min(info.n_test, 20000))
    total = args.steps + args.warmup
    nrows, kp = rows_sample_rate(orc, ds, info, thr, 100.0 / total)
    rng = np.random.default_rng(0)
    times = []
    for s in range(total):
        rows = np.sort(rng.choice(info.n, size=nrows, replace=False)).astype(np.int64)
        t = time.perf_counter()
        orc.precompute_rows(ds.X, ds.Y, *kp, info.k, rows, threads=thr)
        if s >= args.warmup:
            times.append(time.perf_counter() - t)
    value = nrows * len(times) / sum(times)
    S, Cm = synthetic_table(info.n, info.k, info.m, 1)
    pred = cpu_predict_baseline(orc, info, ds.X, S, Cm, ds.mean_offset, ds.Z, thr, 40.0,
                                "table: the reference's layout with synthetic values (no reference-built model "
                                "of this size exists; the per-point cost does not depend on the values)")
    return {
        "metric": "precompute train-pts/s", "value": value, "unit": "train-pts/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg{info.cfg}", "d": info.d, "n_train": info.n, "n_test": info.n_test,
                   "k": info.k, "m": info.m, "sample_rows_per_step": nrows},
        "cpu_baseline": {"value": value, "unit": "train-pts/s", "cores": thr, "kind": orc.kind,
                         "sample": f"{nrows} random training rows of cfg{info.cfg} per step (exact kNN against "
                                   f"all {info.n} points + local solve each), {thr} threads"},
        "e2e": {"value": value, "unit": "train-pts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "predict": {"metric": "predict test-pts/s", "value": pred["value"], "unit": "test-pts/s",
                    "cpu_baseline": pred,
                    "e2e": {"value": pred["value"], "unit": "test-pts/s", "h2d_bytes_per_step": 0,
                            "d2h_bytes_per_step": 0}},
    }


# ---------------------------------------------------------------------------- B200 arm

def main():
    args = parse()
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch_under_torchrun(args)

    if args.probe_launch:  # launcher check (CPU): the ranks really start and meet
        import torch
        import torch.distributed as dist
        if ws > 1:
            dist.init_process_group("gloo")
        t = torch.ones(1)
        if ws > 1:
            dist.all_reduce(t)
        if rank == 0:
            print(json.dumps({"probe": "launch", "n_ranks": int(t.item()), "world_size": ws, "n_gpus": args.gpus}),
                  flush=True)
        if ws > 1:
            dist.destroy_process_group()
        return 0

    from paper_2205_10879_b200 import datagen
    info = datagen.config_info(args.config)
    if args.n:
        info.n = args.n
    if args.nt:
        info.n_test = args.nt
    n, nt = info.n, info.n_test

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, info)), flush=True)
        return 0

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if ws > 1:  # control plane only (id exchange, barriers, max over ranks); the data path is NCCL from C++
        dist.init_process_group("gloo")
    from paper_2205_10879_b200 import _native as N
    from paper_2205_10879_b200.parallel import shard_bounds
    dev = torch.device("cuda", local)
    k, m, d = info.k, info.m, info.d
    kp = N.KernelParamsC(info.kind, info.sigma, info.rho, info.nu, info.tau)
    mo = np.ascontiguousarray(np.broadcast_to(np.asarray(0.0), (m,)), dtype=np.float64)

    # the rank group (NCCL communicator from a unique id rank 0 draws)
    uid = (C.c_uint8 * 128)()
    if ws > 1:
        if rank == 0:
            N.check(N.LIB.fmgp_group_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        C.memmove(uid, obj[0], 128)
    group = C.c_void_p()
    N.check(N.LIB.fmgp_group_create_rank(uid if ws > 1 else None, ws, rank, local, C.byref(group)))

    ds = datagen.generate(args.config, n, nt)
    mo = np.ascontiguousarray(np.asarray(ds.mean_offset, dtype=np.float64).reshape(-1))
    X = torch.from_numpy(ds.X).to(dev)
    Y = torch.from_numpy(ds.Y).to(dev)
    Z = torch.from_numpy(ds.Z).to(dev)
    S_all = torch.empty((n, k), dtype=torch.int32, device=dev)
    C_all = torch.empty((n, k, m), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    state = {}
    failed = C.c_int64(-1)

    def sync_all():
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64)
        if ws > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def precompute_step():
        N.check(N.LIB.fmgp_group_precompute_device(group, C.c_void_p(X.data_ptr()), C.c_void_p(Y.data_ptr()), n, d,
                                                   m, C.byref(kp), k, C.c_void_p(S_all.data_ptr()),
                                                   C.c_void_p(C_all.data_ptr()), C.byref(failed),
                                                   C.c_void_p(stream.cuda_stream)), failed.value)

    pb, pe, _ = shard_bounds(nt, ws, rank)
    P_out = torch.empty((max(pe - pb, 1), m), dtype=torch.float64, device=dev)

    def predict_step():
        N.check(N.LIB.fmgp_model_predict_device(state["model"], C.c_void_p(Z[pb:pe].data_ptr()), pe - pb,
                                                C.c_void_p(P_out.data_ptr()), None, C.c_void_p(stream.cuda_stream)))

    def timed(fn, steps, warmup, stage_events=False):
        for _ in range(warmup):
            fn()
        sync_all()
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
            state["stage"] = {"knn_ms": a.value / max(c.value, 1), "solve_ms": b.value / max(c.value, 1)}
        sync_all()
        return max_over_ranks(sum(ms) / steps), ms, launches

    # FP64 roofline denominators measured on this GPU in this run
    dfma, dmma = C.c_double(0), C.c_double(0)
    N.check(N.LIB.fmgp_diag_fp64_peak(C.byref(dfma), C.byref(dmma)))

    if args.settle > 0:  # see --settle; nothing is timed before or during this wait
        time.sleep(args.settle)
        sync_all()
    with ClockSampler(local) as clk:
        pre_ms, pre_all, pre_launch = timed(precompute_step, args.steps, args.warmup, stage_events=True)
        model = C.c_void_p()  # the device-resident model over this rank's full (all-gathered) S, C
        N.check(N.LIB.fmgp_model_wrap_device(C.c_void_p(X.data_ptr()), C.c_void_p(S_all.data_ptr()),
                                             C.c_void_p(C_all.data_ptr()), n, d, k, m, C.byref(kp),
                                             mo.ctypes.data_as(C.c_void_p), C.byref(model)))
        state["model"] = model
        pred_ms, pred_all, pred_launch = timed(predict_step, args.steps, args.warmup)
    clocks = clk.summary()
    stage = state.get("stage", {})
    knn_ms, solve_ms = stage.get("knn_ms"), stage.get("solve_ms")
    value = n / (pre_ms / 1e3)
    pred_value = nt / (pred_ms / 1e3)

    # ---- e2e: host buffers through the C ABI, copies inside the timed region
    e2e = pred_e2e = None
    cpu_model = None
    if not args.no_e2e:
        Xh = torch.from_numpy(ds.X).pin_memory()
        Yh = torch.from_numpy(ds.Y).pin_memory()
        Sh = torch.empty((n, k), dtype=torch.int32).pin_memory()
        Ch = torch.empty((n, k, m), dtype=torch.float64).pin_memory()
        own = [(0, n)]
        if ws > 1:
            nb = C.c_int64(0)
            N.check(N.LIB.fmgp_group_rows(n, ws, rank, C.byref(nb), None))
            rg = np.zeros(2 * max(nb.value, 1), dtype=np.int64)
            N.check(N.LIB.fmgp_group_rows(n, ws, rank, C.byref(nb), rg.ctypes.data_as(C.c_void_p)))
            own = [(int(rg[2 * i]), int(rg[2 * i + 1])) for i in range(nb.value)]
        own_rows = sum(e - b for b, e in own)

        def e2e_step():
            if ws == 1:
                N.check(N.LIB.fmgp_precompute(C.c_void_p(Xh.data_ptr()), C.c_void_p(Yh.data_ptr()), n, d, m,
                                              C.byref(kp), k, C.c_void_p(Sh.data_ptr()), C.c_void_p(Ch.data_ptr()),
                                              C.byref(failed)), failed.value)
            else:
                N.check(N.LIB.fmgp_group_precompute(group, C.c_void_p(Xh.data_ptr()), C.c_void_p(Yh.data_ptr()), n,
                                                    d, m, C.byref(kp), k, mo.ctypes.data_as(C.c_void_p),
                                                    C.c_void_p(Sh.data_ptr()), C.c_void_p(Ch.data_ptr()),
                                                    C.byref(failed), None), failed.value)

        def host_timed(fn):
            for _ in range(args.warmup):
                fn()
            ts = []
            for _ in range(args.steps):
                flush.fill_(1.0)
                sync_all()
                t = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - t)
            return max_over_ranks(sum(ts) / len(ts))

        t_e2e = host_timed(e2e_step)
        e2e = {"value": n / t_e2e, "unit": "train-pts/s", "h2d_bytes_per_step": int(Xh.numel() * 8 + Yh.numel() * 8),
               "d2h_bytes_per_step": int(own_rows * k * 4 + own_rows * k * m * 8),
               "api": ("fmgp_precompute (the C++ facade's precompute)" if ws == 1 else
                       "fmgp_group_precompute (rank group: full X/Y in per rank, the rank's row blocks of S/C out, "
                       "every rank's device ends with the full all-gathered model)") +
                      ", pinned host buffers, max over ranks"}

        # predict through the host-buffer model handle (fmgp_model_predict): the model is built once from
        # the precompute (untimed; the reference's PrecomputedModel is likewise built before predicting)
        hmodel = C.c_void_p()
        N.check(N.LIB.fmgp_group_precompute(group, C.c_void_p(Xh.data_ptr()), C.c_void_p(Yh.data_ptr()), n, d, m,
                                            C.byref(kp), k, mo.ctypes.data_as(C.c_void_p),
                                            C.c_void_p(Sh.data_ptr()), C.c_void_p(Ch.data_ptr()), C.byref(failed),
                                            C.byref(hmodel)), failed.value)
        Zh = torch.from_numpy(np.ascontiguousarray(ds.Z[pb:pe])).pin_memory()
        Oh = torch.empty((max(pe - pb, 1), m), dtype=torch.float64).pin_memory()

        def pred_e2e_step():
            N.check(N.LIB.fmgp_model_predict(hmodel, C.c_void_p(Zh.data_ptr()), pe - pb, C.c_void_p(Oh.data_ptr()),
                                             None))

        t_pe = host_timed(pred_e2e_step)
        pred_e2e = {"value": nt / t_pe, "unit": "test-pts/s", "h2d_bytes_per_step": int((pe - pb) * d * 8),
                    "d2h_bytes_per_step": int((pe - pb) * m * 8),
                    "api": "fmgp_model_predict (the facade's fast_predict_batch) on a model handle, pinned host "
                           "buffers, this rank's test shard, max over ranks"}
        if ws == 1:
            cpu_model = (Sh.numpy(), Ch.numpy())
        N.LIB.fmgp_model_destroy(hmodel)

    # ---- rooflines: algorithmic work per launch / that kernel's average launch time (CUDA events)
    hbm, hbm_src = hbm_peak()
    # measured DRAM traffic of the same kernels (committed ncu capture of this command), scaled to the step
    tr = load_json(REPO / "profiles" / "r02" / "traffic.json") or {}
    tr_solve = tr.get("solve_cfg5") if info.cfg == 5 else None
    tr_pred = tr.get("predict_cfg5") if info.cfg == 5 else None
    rows_per_rank = (n + ws - 1) // ws
    roof = None
    if solve_ms is not None and knn_ms is not None:
        if solve_ms >= knn_ms:
            flops = solve_flops_per_row(info) * rows_per_rank
            achieved = flops / (solve_ms / 1e3) / 1e12
            roof = {"bound": "fp64", "kernel": "fused solve (gather / kernel build / jitter-Cholesky / solve)",
                    "achieved": achieved, "peak": dfma.value, "unit": "TFLOP/s", "frac": achieved / dfma.value,
                    "traffic": ((tr_solve["dram_read_bytes"] + tr_solve["dram_write_bytes"]) / tr_solve["rows_per_launch"]
                                * rows_per_rank) if tr_solve else None,
                    "traffic_unit": "DRAM bytes for the step's rows (ncu per-launch bytes scaled by rows)",
                    "traffic_source": f"profiles/r02/traffic.json ({tr_solve.get('kernel')})" if tr_solve else None,
                    "fp64_pipe_active_pct_ncu": tr_solve.get("fp64_pipe_active_pct") if tr_solve else None,
                    "work": f"{solve_flops_per_row(info):.0f} fp64 flops per training row (SURVEY 8(d): k^3/3 + "
                            f"2k^2m + 3d k(k-1)/2; the k(k-1)/2 kernel evaluations are not counted) x {rows_per_rank} "
                            "rows per rank",
                    "kernel_ms": solve_ms, "share_of_step": solve_ms / pre_ms,
                    "peak_source": "DFMA rate measured in this run on this GPU (fmgp_diag_fp64_peak); "
                                   f"DMMA {dmma.value:.1f} TFLOP/s",
                    "hbm_gbs": (4 * k + 8 * k * d + 8 * k * m + 8 * k * m) * rows_per_rank / (solve_ms / 1e3) / 1e9}
        else:
            roof = {"bound": "alu", "kernel": "kNN stage", "achieved": None, "peak": None, "unit": None, "frac": None,
                    "kernel_ms": knn_ms, "share_of_step": knn_ms / pre_ms, "traffic": None}
    pred_pts = pe - pb
    pred_gbs = predict_bytes_per_point(info) * pred_pts / (pred_ms / 1e3) / 1e9

    line = {
        "metric": "precompute train-pts/s", "value": value, "unit": "train-pts/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": pre_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg{info.cfg}", "d": d, "n_train": n, "n_test": nt, "k": k, "m": m,
                   "kernel": "RBF" if info.kind == 1 else f"Matern nu={info.nu}",
                   "parallelism": f"rows block-cyclic over {ws} GPU(s), S/C all-gathered (NCCL, C++)",
                   "l2": "flushed (256 MiB write) between timed steps",
                   "settle_s": args.settle},
        "predict": {"metric": "predict test-pts/s", "value": pred_value, "unit": "test-pts/s", "ms_per_step": pred_ms,
                    "roofline": {"bound": "hbm", "achieved": pred_gbs, "peak": hbm, "unit": "GB/s",
                                 "frac": pred_gbs / hbm, "peak_source": hbm_src,
                                 "work": f"{predict_bytes_per_point(info)} B per test point (SURVEY 8(d)) x "
                                         f"{pred_pts} points per rank; the stage also runs the grid 1-NN walk",
                                 "traffic": ((tr_pred["dram_read_bytes"] + tr_pred["dram_write_bytes"])
                                             / tr_pred["points_per_launch"] * pred_pts) if tr_pred else None,
                                 "traffic_source": "profiles/r02/traffic.json" if tr_pred else None},
                    "e2e": pred_e2e, "gpu_launches": pred_launch},
        "stages_ms": {"knn": knn_ms, "solve": solve_ms, "precompute": pre_ms, "predict": pred_ms},
        "e2e": e2e,
        "roofline": roof,
        "clocks": clocks,
        "gpu_launches": pre_launch,
        "fp64_peak_tflops": {"dfma": dfma.value, "dmma": dmma.value},
        "step_ms": {"precompute": pre_all, "predict": pred_all},
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        from oracle.oracle import best_available, host_threads
        orc = best_available()
        thr = host_threads()
        line["cpu_baseline"] = cpu_precompute_baseline(orc, info, ds, thr, 12.0, 1)
        if cpu_model is None:
            cpu_model = (S_all.cpu().numpy(), C_all.cpu().numpy())
        line["predict"]["cpu_baseline"] = cpu_predict_baseline(
            orc, info, ds.X, cpu_model[0], cpu_model[1], ds.mean_offset, ds.Z, thr, 24.0,
            "model: this run's precomputed S and C")
    N.LIB.fmgp_model_destroy(state["model"])
    N.LIB.fmgp_group_destroy(group)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
