"""Data parallelism for the F-Hash train step.

Samples are independent, so the global batch is split evenly over the
ranks; tables and MLP are replicated.  The loss carries 1/N_global
(fh_train_fwd_bwd, R12), so the SUM of the ranks' gradients is exactly the
gradient of the global batch: the one exchange step is an all-reduce (SUM)
of the trainer's flat fp32 grad buffer over the process group (NCCL over
NVLink/NVSwitch on the GPU box; gloo in the CPU tests), between
`fwd_bwd` and `apply`.  Identical initial parameters + identical summed
grads + deterministic Adam keep the replicas bit-identical.
"""
from __future__ import annotations

from typing import Optional, Tuple


def shard(n_global: int, rank: int, world: int) -> Tuple[int, int]:
    """(start, count) of rank's slice of a global batch: even split, the
    first n_global % world ranks take one extra sample."""
    if world < 1 or not (0 <= rank < world) or n_global < 0:
        raise ValueError("bad shard arguments")
    base, rem = divmod(n_global, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def allreduce_grads(grads, group=None) -> None:
    """In-place SUM all-reduce of a flat gradient tensor (no-op when the
    default process group is not initialised or has one rank)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=group)


def dp_train_step(trainer, coords, target, n_global: int, group=None, stream=None):
    """One data-parallel step on this rank's shard: local forward+backward
    (loss scaled by 1/n_global), all-reduce of the flat grads, Adam."""
    loss = trainer.fwd_bwd(coords, target, n_global, stream=stream)
    allreduce_grads(trainer.grads, group)
    trainer.apply(stream=stream)
    return loss


def replicas_identical(tensor, group=None) -> bool:
    """True when `tensor` is bit-identical on every rank (compares a 64-bit
    checksum of its bytes gathered from all ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return True
    raw = tensor.detach().contiguous().view(torch.uint8)
    pad = (-raw.numel()) % 8
    if pad:
        raw = torch.cat([raw, torch.zeros(pad, dtype=torch.uint8, device=raw.device)])
    words = raw.view(torch.int64)
    w = torch.arange(1, words.numel() + 1, device=words.device, dtype=torch.int64)
    chk = torch.stack([(words * w).sum(), words.sum(), torch.tensor(words.numel(), device=words.device)])
    allc = [torch.empty_like(chk) for _ in range(dist.get_world_size(group))]
    dist.all_gather(allc, chk, group=group)
    return all(torch.equal(allc[0], c) for c in allc[1:])
