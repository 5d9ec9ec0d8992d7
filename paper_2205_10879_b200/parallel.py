"""Multi-GPU sharding of the path: one process per GPU.

The product's multi-GPU precompute is the C ABI's device group
(csrc/group.cu: fmgp_group_create_rank / fmgp_group_precompute[_device]),
which bench.py drives: X and Y replicated on every rank, training rows (the
kNN / solve queries) dealt block-cyclically, S and C all-gathered in place
over NVLink by NCCL from C++, each round's exchange overlapped with the next
round's solve. This module is the same host logic over torch.distributed
(`overlapped_precompute`, `cyclic_blocks`), so the layout and the exchange
order are testable on CPU with a gloo process group (tests/test_parallel.py),
plus the plain contiguous-shard helpers. Every row's arithmetic is
independent of the layout, so S and C are bit-identical for any world size.
Predict: test points are split contiguously; no collective is needed (each
rank holds the full replicated model after the gather).

The per-shard compute is injected, so CPU tests pass the oracle while a GPU
caller passes the fmgp_*_device launchers.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def shard_bounds(total: int, world: int, rank: int) -> tuple[int, int, int]:
    """Contiguous shard [begin, end) of `total` rows for `rank`, and the padded per-rank size."""
    per = (total + world - 1) // world
    begin = min(total, rank * per)
    end = min(total, begin + per)
    return begin, end, per


def _all_gather_rows(local: torch.Tensor, per: int, group=None) -> torch.Tensor:
    """Gather equally padded row shards (rank order) into one tensor of world*per rows."""
    world = dist.get_world_size(group)
    if local.shape[0] < per:
        pad = torch.zeros((per - local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        local = torch.cat([local, pad], 0)
    local = local.contiguous()
    out = torch.empty((world * per,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local, group=group)
    else:
        parts = list(out.chunk(world, 0))
        dist.all_gather(parts, local, group=group)
        out = torch.cat(parts, 0)
    return out


def sharded_precompute(n: int, compute_shard: Callable[[int, int], tuple[torch.Tensor, torch.Tensor]],
                       group=None) -> tuple[torch.Tensor, torch.Tensor]:
    """Run compute_shard(begin, end) -> (S rows, C rows) on this rank's rows and
    all-gather the full (S n x k, C n x k x m) on every rank."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    b, e, per = shard_bounds(n, world, rank)
    S_loc, C_loc = compute_shard(b, e)
    if world == 1:
        return S_loc, C_loc
    S = _all_gather_rows(S_loc, per, group)[:n]
    C = _all_gather_rows(C_loc, per, group)[:n]
    return S, C


def cyclic_blocks(n: int, world: int, rounds: int = 4) -> tuple[int, list[list[tuple[int, int]]]]:
    """The block-cyclic row layout of the C ABI's device groups (csrc/group.cu,
    fmgp_group_rows): blocks of pc = ceil(n / (world * rounds)) rows dealt
    round-robin; round c is rows [c*world*pc, (c+1)*world*pc) and member r owns
    its block c*world + r. Returns pc and, per round, every member's [b, e)."""
    if world == 1:
        rounds = 1  # nothing to exchange: one round (as csrc/group.cu)
    pc = max(1, -(-n // (world * rounds)))
    out = []
    c = 0
    while c * world * pc < n:
        out.append([(min(n, (c * world + r) * pc), min(n, (c * world + r) * pc + pc)) for r in range(world)])
        c += 1
    return pc, out


class _Side:
    """A side stream for collectives on CUDA tensors; a no-op on CPU (gloo tests)."""

    def __init__(self, device: torch.device):
        self.cuda = device.type == "cuda"
        self.main = torch.cuda.current_stream(device) if self.cuda else None
        self.side = torch.cuda.Stream(device) if self.cuda else None

    def after_main(self):
        """Context: work issued inside runs on the side stream, after everything issued so far on main."""
        if not self.cuda:
            return _Null()
        self.side.wait_stream(self.main)
        return torch.cuda.stream(self.side)

    def join(self):
        if self.cuda:
            self.main.wait_stream(self.side)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def _exchange_round(buf: torch.Tensor, blocks: list[tuple[int, int]], rank: int, group=None) -> None:
    """Every member's block of one round into every member's `buf`, in place.
    A full round (equal blocks, contiguous) is one all-gather whose send buffer
    is this rank's block of the receive buffer; a short last round is one
    broadcast per member."""
    world = len(blocks)
    sizes = {e - b for b, e in blocks}
    if len(sizes) == 1 and blocks[-1][1] - blocks[0][0] == world * (blocks[0][1] - blocks[0][0]):
        b0, e_last = blocks[0][0], blocks[-1][1]
        region = buf[b0:e_last]
        mine = buf[blocks[rank][0]:blocks[rank][1]]
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(region, mine, group=group)
        else:
            parts = [buf[b:e] for b, e in blocks]
            tmp = [torch.empty_like(mine) for _ in parts]
            dist.all_gather(tmp, mine.contiguous(), group=group)
            for p_, t in zip(parts, tmp):
                p_.copy_(t)
        return
    for q, (b, e) in enumerate(blocks):
        if e > b:
            view = buf[b:e]
            if view.is_contiguous():
                dist.broadcast(view, src=q, group=group)
            else:
                t = view.contiguous()
                dist.broadcast(t, src=q, group=group)
                view.copy_(t)


def overlapped_precompute(n: int, k: int, m: int, knn_rows: Callable[[int, int], torch.Tensor],
                          solve_rows: Callable[[torch.Tensor, int, torch.Tensor], None], nchunks: int = 4,
                          group=None, device: torch.device | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """The device-group precompute of csrc/group.cu, host logic in Python:
    block-cyclic rows (cyclic_blocks); K1 for this rank's blocks
    (knn_rows(b, e) -> S rows), S exchanged in place per round on a side
    stream; then per round K2 of this rank's block (solve_rows(S_rows,
    row_begin, C_rows) writes C rows, stream-ordered) followed by that round's
    in-place C exchange on the side stream, overlapping the next round's solve.
    No staging copies. Every rank returns the full S (n x k) and C (n x k x m),
    bit-identical to a single rank (rows are independent)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    _, rounds = cyclic_blocks(n, world, nchunks)
    dev = device
    S_all = C_all = None
    for blocks in rounds:
        b, e = blocks[rank]
        if e > b:
            S_loc = knn_rows(b, e)
            if S_all is None:
                dev = S_loc.device if device is None else device
                S_all = torch.empty((n, k), dtype=torch.int32, device=dev)
            S_all[b:e] = S_loc
    if S_all is None:  # a rank without rows (n < world)
        dev = torch.device("cpu") if device is None else device
        S_all = torch.empty((n, k), dtype=torch.int32, device=dev)
    C_all = torch.empty((n, k, m), dtype=torch.float64, device=dev)
    if world == 1:
        for blocks in rounds:
            b, e = blocks[0]
            solve_rows(S_all[b:e], b, C_all[b:e])
        return S_all, C_all
    side = _Side(dev)
    with side.after_main():
        for blocks in rounds:
            _exchange_round(S_all, blocks, rank, group)
    for blocks in rounds:
        b, e = blocks[rank]
        if e > b:
            solve_rows(S_all[b:e], b, C_all[b:e])
        with side.after_main():
            _exchange_round(C_all, blocks, rank, group)
    side.join()
    return S_all, C_all


def sharded_predict(nz: int, predict_shard: Callable[[int, int], torch.Tensor], gather: bool = False,
                    group=None) -> torch.Tensor:
    """Each rank predicts its contiguous test shard; optionally gather all means."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    b, e, per = shard_bounds(nz, world, rank)
    out = predict_shard(b, e)
    if not gather or world == 1:
        return out
    return _all_gather_rows(out, per, group)[:nz]
