"""Multi-GPU driver: independent (batch, window, head) problems sharded over ranks.

QFlash problems are independent (Algorithm 1's outer loops; windows
folded into the batch axis), so the hot path shards with NO collective: rank r
of `world` takes the contiguous problem range qflash_partition(P, world, r) --
a pointer offset into the [P, N, d] tensors -- and runs the same C-ABI call
with the same per-tensor scales.  The only collectives are
outside the hot path:
  * gather_problems: one all_gather of the int8 outputs, for verification;
  * allreduce_amax: when several ranks quantize shards of ONE logical tensor,
    a 4-byte MAX all-reduce keeps the per-tensor scale identical to 1 GPU.
Process groups come from torch.distributed (NCCL on GPUs; gloo in CPU tests).
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from .api import qflash_partition


def problem_range(num_problems: int, world: int, rank: int) -> tuple[int, int]:
    """(begin, count) of this rank's contiguous problem slab (C-ABI qflash_partition)."""
    return qflash_partition(num_problems, world, rank)


def local_slab(t: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """The rank's [count, N, d] view of a [P, N, d] tensor (no copy)."""
    b, c = problem_range(t.shape[0], world, rank)
    return t.narrow(0, b, c)


def gather_problems(local: torch.Tensor, num_problems: int, group=None) -> torch.Tensor:
    """all_gather the ranks' output slabs into the full [P, N, d] tensor on every rank
    (verification only; uneven slabs are padded to the largest count)."""
    world = dist.get_world_size(group)
    counts = [problem_range(num_problems, world, r)[1] for r in range(world)]
    cmax = max(counts) if counts else 0
    pad = torch.zeros((cmax,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)


def allreduce_amax(amax: torch.Tensor, group=None) -> torch.Tensor:
    """MAX all-reduce of a per-tensor amax so sharded quantization uses the
    single-GPU scale s = amax / 127 (Eq. 2)."""
    dist.all_reduce(amax, op=dist.ReduceOp.MAX, group=group)
    return amax


def run_sharded(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                attention_fn: Callable[[torch.Tensor, torch.Tensor, torch.Tensor], torch.Tensor],
                group=None, verify_gather: bool = True):
    """Run `attention_fn` on this rank's slab of the [P, N, d] int8 inputs.

    attention_fn(q_slab, k_slab, v_slab) -> out_slab (e.g. a closure over
    qflash_attention_int8 with the shared scales).  Returns (local_out,
    full_out_or_None); the gather is the verification collective only."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    P = q.shape[0]
    qs, ks, vs = (local_slab(t, world, rank) for t in (q, k, v))
    out = attention_fn(qs, ks, vs)
    full = gather_problems(out, P, group) if (verify_gather and world > 1) else None
    return out, full
