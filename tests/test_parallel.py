"""CPU, world_size 2 over gloo: the multi-GPU host logic (row shards ->
all-gather) assembles the same S and C as a single rank, bit-exactly. The
per-shard compute is the oracle here (stand-in for fmgp_precompute_device)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Port
        from paper_2205_10879_b200 import datagen
        from paper_2205_10879_b200.parallel import sharded_precompute, sharded_predict
        orc = Port()
        ds = datagen.generate(5, 301, 37)
        i = ds.info
        kp = (i.kind, i.sigma, i.rho, i.nu, i.tau)
        k = 9

        def shard(b, e):
            S, C = orc.precompute_rows(ds.X, ds.Y, *kp, k, np.arange(b, e))
            return torch.from_numpy(S), torch.from_numpy(C)

        S, C = sharded_precompute(ds.X.shape[0], shard)

        def pshard(b, e):
            out, _ = orc.predict(ds.X, S.numpy(), C.numpy(), *kp, ds.mean_offset, ds.Z[b:e])
            return torch.from_numpy(out)

        P = sharded_predict(ds.Z.shape[0], pshard, gather=True)
        if rank == 0:
            q.put((S.numpy(), C.numpy(), P.numpy()))
    finally:
        dist.destroy_process_group()


def test_shard_bounds_cover_rows_once():
    from paper_2205_10879_b200.parallel import shard_bounds
    for total in (1, 7, 100, 301):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                b, e, per = shard_bounds(total, world, r)
                assert e - b <= per
                seen.extend(range(b, e))
            assert seen == list(range(total))


def test_two_rank_gloo_sharding_is_bit_identical_to_one_rank():
    from oracle.oracle import Port
    from paper_2205_10879_b200 import datagen
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    S2, C2, P2 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    orc = Port()
    ds = datagen.generate(5, 301, 37)
    i = ds.info
    S1, C1 = orc.precompute_rows(ds.X, ds.Y, i.kind, i.sigma, i.rho, i.nu, i.tau, 9)
    P1, _ = orc.predict(ds.X, S1, C1, i.kind, i.sigma, i.rho, i.nu, i.tau, ds.mean_offset, ds.Z)
    assert np.array_equal(S1, S2) and np.array_equal(C1, C2) and np.array_equal(P1, P2)


def _overlap_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import Port
        from paper_2205_10879_b200 import datagen
        from paper_2205_10879_b200.parallel import overlapped_precompute
        orc = Port()
        ds = datagen.generate(5, 301, 7)
        i = ds.info
        kp = (i.kind, i.sigma, i.rho, i.nu, i.tau)
        k = 9

        def knn_rows(b, e):  # K1 stand-in: the oracle's S rows
            S, _ = orc.precompute_rows(ds.X, ds.Y, *kp, k, np.arange(b, e))
            return torch.from_numpy(S)

        def solve_rows(S_rows, row_begin, C_out):  # K2 stand-in: the oracle's C rows for those rows
            rows = np.arange(row_begin, row_begin + S_rows.shape[0])
            S, C = orc.precompute_rows(ds.X, ds.Y, *kp, k, rows)
            assert np.array_equal(S, S_rows.numpy())  # the chunk got its own rows' S
            C_out.copy_(torch.from_numpy(C))

        S, C = overlapped_precompute(ds.X.shape[0], k, 1, knn_rows, solve_rows, nchunks=3)
        if rank == 0:
            q.put((S.numpy(), C.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_overlapped_gather_is_bit_identical_to_one_rank(world):
    # K1 per shard, S gathered on a side stream, K2 in chunks with each chunk's C
    # gathered while the next is solved: same tables as a single rank
    from oracle.oracle import Port
    from paper_2205_10879_b200 import datagen
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overlap_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    S2, C2 = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ds = datagen.generate(5, 301, 7)
    i = ds.info
    S1, C1 = Port().precompute_rows(ds.X, ds.Y, i.kind, i.sigma, i.rho, i.nu, i.tau, 9)
    assert np.array_equal(S1, S2) and np.array_equal(C1, C2)


@pytest.mark.parametrize("n", [1, 5, 301, 1000, 8_000_000])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_cyclic_layout_matches_the_c_abi(n, world):
    # the Python mirror and csrc/group.cu deal the same blocks (fmgp_group_rows
    # needs no device), and every row is owned exactly once
    import ctypes as C
    from paper_2205_10879_b200 import _native as N
    from paper_2205_10879_b200.parallel import cyclic_blocks
    _, rounds = cyclic_blocks(n, world)
    owned = np.zeros(n, dtype=np.int64)
    for r in range(world):
        mine = [blk[r] for blk in rounds if blk[r][1] > blk[r][0]]
        nb = C.c_int64(-1)
        assert N.LIB.fmgp_group_rows(n, world, r, C.byref(nb), None) == 0
        rg = np.zeros(2 * max(nb.value, 1), dtype=np.int64)
        assert N.LIB.fmgp_group_rows(n, world, r, C.byref(nb), rg.ctypes.data_as(C.c_void_p)) == 0
        assert [(int(rg[2 * i]), int(rg[2 * i + 1])) for i in range(nb.value)] == mine
        for b, e in mine:
            owned[b:e] += 1
    assert (owned == 1).all()


def test_bench_gpus_flag_launches_that_many_ranks():
    # `python bench.py --gpus 2` (the driver's form, no torchrun) re-launches
    # itself with one process per GPU; the probe makes every rank join a gloo
    # group and rank 0 report the count
    import json
    import subprocess
    import sys
    from pathlib import Path
    repo = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(repo / "bench.py"), "--gpus", "2", "--probe-launch"],
                         capture_output=True, text=True, timeout=300, cwd=repo)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_ranks"] == 2 and line["world_size"] == 2
