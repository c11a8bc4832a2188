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


class ShardedDP:
    """Reduce-scatter -> sharded Adam -> all-gather (ZeRO-1 style) for the
    table parameters; the small MLP segment is all-reduced and updated on
    every rank.  Same mathematics as dp_train_step; per step it moves
    (W-1)/W of the fp32 table grads plus (W-1)/W of the fp16 shadow instead
    of 2(W-1)/W of the fp32 grads, and each rank runs Adam over 1/W of the
    table.  Needs a trainer built with world=W and
    an fp16 table shadow.  The fp32 masters / moments of a rank are only
    current inside its shard; the replicated state is the fp16 shadow."""

    def __init__(self, trainer, group=None):
        import torch
        import torch.distributed as dist
        self.tr = trainer
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        if trainer.world != self.world:
            raise ValueError(f"trainer padded for world={trainer.world}, group has {self.world} ranks")
        if trainer.shadow_flat is None:
            raise ValueError("sharded DP needs an fp16 table shadow (the replicated state)")
        self.chunk = trainer.nt_pad // self.world
        self.begin = min(self.rank * self.chunk, trainer.n_table)
        self.end = min(self.begin + self.chunk, trainer.n_table)
        self.shard = torch.empty(self.chunk, dtype=torch.float32, device=trainer.grads.device)
        self._inplace_ok = (not dist.is_initialized()) or dist.get_backend(group) == "nccl"

    def reduce(self):
        import torch.distributed as dist
        tr = self.tr
        if self.world == 1:
            self.shard.copy_(tr.grads[:self.chunk])
            return
        dist.reduce_scatter_tensor(self.shard, tr.grads[:tr.nt_pad], op=dist.ReduceOp.SUM, group=self.group)
        dist.all_reduce(tr.mlp_grad, op=dist.ReduceOp.SUM, group=self.group)

    def apply(self, stream=None):
        self.tr.apply_sharded(self.begin, self.end, self.shard, stream=stream)

    def gather(self):
        import torch.distributed as dist
        if self.world == 1:
            return
        flat = self.tr.shadow_flat
        lo = self.rank * self.chunk
        mine = flat[lo:lo + self.chunk]
        if not self._inplace_ok:
            mine = mine.clone()          # gloo: no aliasing of input and output
        dist.all_gather_into_tensor(flat, mine, group=self.group)

    def step(self, coords, target, n_global: int, stream=None):
        loss = self.tr.fwd_bwd(coords, target, n_global, stream=stream)
        self.reduce()
        self.apply(stream=stream)
        self.gather()
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
