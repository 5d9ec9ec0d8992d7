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
