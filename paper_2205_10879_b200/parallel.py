"""Multi-GPU sharding of the path: one process per GPU.

* Precompute: X and Y are replicated on every rank; training rows (the kNN /
  solve queries) are split into contiguous, rank-ordered shards; each rank
  computes its S and C rows against the full X, then the shards are
  all-gathered (NCCL over NVLink on B200s; gloo in the CPU tests). Every row's
  arithmetic is independent of the shard layout, so S and C are bit-identical
  for any world size.
* Predict: test points are split the same way; no collective is needed (each
  rank holds the full replicated model after the gather).

The per-shard compute is injected (`compute_shard`), so the host-side logic
is testable on CPU with a gloo process group; the product passes the
fmgp_precompute_device launcher.
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


def overlapped_precompute(n: int, k: int, m: int, knn_rows: Callable[[int, int], torch.Tensor],
                          solve_rows: Callable[[torch.Tensor, int, torch.Tensor], None], nchunks: int = 4,
                          group=None, device: torch.device | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """sharded_precompute with the exchange overlapped: K1 for this rank's rows
    (knn_rows(b, e) -> S rows), the S all-gather then runs on a side stream
    while K2 solves the shard in `nchunks` chunks (solve_rows(S_rows, row_begin,
    C_rows) writes C rows, stream-ordered); each chunk's C all-gather is issued
    on the side stream as soon as the chunk is solved, so it overlaps the next
    chunk's solve. Every rank returns the full S (n x k) and C (n x k x m),
    bit-identical to sharded_precompute (rows are independent)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    b, e, per = shard_bounds(n, world, rank)
    rows = e - b
    S_loc = knn_rows(b, e)
    dev = S_loc.device if device is None else device
    if world == 1:
        C_loc = torch.empty((rows, k, m), dtype=torch.float64, device=dev)
        solve_rows(S_loc, b, C_loc)
        return S_loc, C_loc
    side = _Side(dev)
    S_pad = torch.zeros((per, k), dtype=torch.int32, device=dev)
    S_pad[:rows] = S_loc
    S_all = torch.empty((world * per, k), dtype=torch.int32, device=dev)
    with side.after_main():
        _all_gather_into(S_all, S_pad, group)
    C_pad = torch.zeros((per, k, m), dtype=torch.float64, device=dev)
    C_all = torch.empty((world, per, k, m), dtype=torch.float64, device=dev)
    pc = (per + nchunks - 1) // nchunks
    staging = []
    for lo in range(0, per, pc):
        hi = min(per, lo + pc)
        r_lo, r_hi = min(rows, lo), min(rows, hi)
        if r_hi > r_lo:
            solve_rows(S_loc[r_lo:r_hi], b + r_lo, C_pad[r_lo:r_hi])
        g = torch.empty((world * (hi - lo), k, m), dtype=torch.float64, device=dev)
        staging.append(g)
        with side.after_main():
            _all_gather_into(g, C_pad[lo:hi], group)
            C_all[:, lo:hi].copy_(g.view(world, hi - lo, k, m))
    side.join()
    return S_all[:n], C_all.view(world * per, k, m)[:n]


def _all_gather_into(out: torch.Tensor, local: torch.Tensor, group=None) -> None:
    """out (world * rows, ...) <- the ranks' `local` (rows, ...) in rank order."""
    local = local.contiguous()
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, local, group=group)
    else:
        parts = list(out.chunk(dist.get_world_size(group), 0))
        tmp = [torch.empty_like(local) for _ in parts]
        dist.all_gather(tmp, local, group=group)
        for p_, t in zip(parts, tmp):
            p_.copy_(t)


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
