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

from typing import Tuple


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


def overlap_plan(launch_ranges, world: int, rank: int):
    """Partition of the table gradient for OverlappedShardedDP.

    launch_ranges: per backward launch, the flat element ranges it finalises
    (Trainer.bwd_launch_ranges).  Each range [b, e) splits into a MAIN part
    [a, a + m) -- a = b rounded up to 4, m the largest multiple of 4 W that
    fits -- reduce-scattered in W equal chunks of m / W (a multiple of 4, so
    every chunk is 16-byte aligned for the vectorised Adam), and at most
    3 + 4 W - 1 TAIL elements, all-reduced and updated on every rank.
    Returns (mains, tails): mains = [(launch, a, m)], tails = [(b, e)]."""
    mains, tails = [], []
    q = 4 * world
    for li, rngs in enumerate(launch_ranges):
        for b, e in rngs:
            a = min((b + 3) // 4 * 4, e)
            m = (e - a) // q * q
            if a > b:
                tails.append((b, a))
            if m > 0:
                mains.append((li, a, m))
            if a + m < e:
                tails.append((a + m, e))
    return mains, tails


class OverlappedShardedDP:
    """ShardedDP with the reduction overlapped with the backward (SURVEY.md
    §8(e) item 2).  fh_train_fwd_bwd records one CUDA event after each
    backward launch (a level group whose gradients are then final); a
    communication stream waits for each event and reduce-scatters that
    group's gradients while the later groups' backward still runs.  Each
    rank then runs ONE Adam launch over its chunks of every group plus the
    (tiny, replicated) tails (fh_train_apply_ranges) and all-gathers the
    fp16 shadow of its chunks.  Same mathematics as ShardedDP / the
    single-process step: every table element is in exactly one main chunk
    or tail, see overlap_plan.  Works on CPU tensors too (gloo, no streams),
    which is how the CPU tests exercise the partition."""

    def __init__(self, trainer, group=None, force_collectives: bool = False):
        import torch
        import torch.distributed as dist
        self.tr = trainer
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        # force_collectives: run the collective path even on a 1-rank group
        # (tests the stream / event plumbing with NCCL on one GPU)
        self.force = force_collectives and dist.is_initialized()
        if trainer.shadow_flat is None:
            raise ValueError("sharded DP needs an fp16 table shadow (the replicated state)")
        self.launches = trainer.bwd_launch_ranges()
        self.mains, self.tails = overlap_plan(self.launches, self.world, self.rank)
        dev = trainer.grads.device
        self.cuda = dev.type == "cuda"
        self.chunks = [m // self.world for (_, _, m) in self.mains]
        self.shard = torch.empty(max(1, sum(self.chunks)), dtype=torch.float32, device=dev)
        self.shard_views, off = [], 0
        for c in self.chunks:
            self.shard_views.append(self.shard[off:off + c])
            off += c
        idx = [i for (b, e) in self.tails for i in range(b, e)]
        self.n_tail = len(idx)
        self.tail_idx = torch.tensor(idx, dtype=torch.int64, device=dev)
        n_mlp = trainer.mlp_grad.numel()
        self.tail_buf = torch.empty(self.n_tail + n_mlp, dtype=torch.float32, device=dev)
        self.tail_views, off = [], 0
        for b, e in self.tails:
            self.tail_views.append(self.tail_buf[off:off + e - b])
            off += e - b
        # Adam ranges: this rank's chunk of every main part, then the tails
        self.ranges = [(a + self.rank * c, a + (self.rank + 1) * c) for (_, a, m), c in zip(self.mains, self.chunks)]
        self.ranges += list(self.tails)
        if len(self.ranges) > 63:
            raise ValueError(f"{len(self.ranges)} Adam ranges (max 63)")
        self._inplace_ok = (not dist.is_initialized()) or dist.get_backend(group) == "nccl"
        self.events = []
        if self.cuda:
            self.comm = torch.cuda.Stream(device=dev)
            self.events = [torch.cuda.Event() for _ in self.launches]
            for ev in self.events:   # create the CUDA events before handing them over
                ev.record()
            trainer.set_bwd_events(self.events)

    def _by_launch(self):
        out = [[] for _ in self.launches]
        for k, (li, a, m) in enumerate(self.mains):
            out[li].append(k)
        return out

    def step(self, coords, target, n_global: int, stream=None):
        loss = self.tr.fwd_bwd(coords, target, n_global, stream=stream)
        self.reduce_and_apply(stream=stream)
        return loss

    def reduce_and_apply(self, stream=None):
        """Everything after fwd_bwd: the per-launch reduce-scatters (queued
        behind the backward launches' events), the tails + MLP all-reduce,
        one Adam over the owned ranges, the shadow all-gathers."""
        import contextlib
        import torch
        import torch.distributed as dist
        tr = self.tr
        grads = tr.grads
        if self.world == 1 and not self.force:
            grad_views = [grads[a:a + m] for (_, a, m) in self.mains] + [grads[b:e] for b, e in self.tails]
            tr.apply_ranges(self.ranges, grad_views, stream=stream)
            return
        cur = torch.cuda.current_stream() if self.cuda else None
        ctx = torch.cuda.stream(self.comm) if self.cuda else contextlib.nullcontext()
        with ctx:
            for li, ks in enumerate(self._by_launch()):
                if self.cuda:
                    self.comm.wait_event(self.events[li])   # launch li's gradients are final
                for k in ks:
                    _, a, m = self.mains[k]
                    dist.reduce_scatter_tensor(self.shard_views[k], grads[a:a + m], op=dist.ReduceOp.SUM,
                                               group=self.group)
            if self.cuda:
                self.comm.wait_stream(cur)                  # MLP grads and tails: whole step done
            if self.n_tail:
                torch.index_select(grads, 0, self.tail_idx, out=self.tail_buf[:self.n_tail])
            self.tail_buf[self.n_tail:].copy_(tr.mlp_grad)
            dist.all_reduce(self.tail_buf, op=dist.ReduceOp.SUM, group=self.group)
            tr.mlp_grad.copy_(self.tail_buf[self.n_tail:])
        if self.cuda:
            cur.wait_stream(self.comm)
        tr.apply_ranges(self.ranges, self.shard_views + self.tail_views, stream=stream)
        flat = tr.shadow_flat
        for (_, a, m), c in zip(self.mains, self.chunks):
            mine = flat[a + self.rank * c: a + (self.rank + 1) * c]
            if not self._inplace_ok:
                mine = mine.clone()          # gloo: no aliasing of input and output
            dist.all_gather_into_tensor(flat[a:a + m], mine, group=self.group)


def symm_alloc(n: int, dtype, device):
    """Trainer(alloc=...) hook: grads / shadow in torch symmetric memory, so
    every rank can map every other rank's buffers (PeerShardedDP)."""
    import torch.distributed._symmetric_memory as sm
    return sm.empty(n, dtype=dtype, device=device)


class PeerShardedDP:
    """The reduction fused with the optimiser over peer memory (SURVEY.md
    §8(e) item 3, with NVLink peer pointers of torch symmetric memory in
    place of an NVLS multicast object).  Per backward level group, once
    every rank has finished it (a symmetric-memory barrier on the
    communication stream, queued behind the group's event), ONE kernel
    (fh_train_apply_peers) sums this rank's chunk of the group over all
    ranks' gradient buffers, runs Adam, and stores the fp16 shadow into every
    rank's shadow buffer -- reduce-scatter, Adam and all-gather in one pass,
    overlapped with the later groups' backward.  The tails of overlap_plan
    and the MLP are summed and updated redundantly on every rank at the end;
    a last barrier precedes the next step's fwd_bwd, which overwrites the
    local gradients.  The trainer must
    be built with alloc=dp.symm_alloc."""

    def __init__(self, trainer, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as sm
        self.tr = trainer
        if trainer.shadow_flat is None:
            raise ValueError("PeerShardedDP needs an fp16 table shadow")
        grp = group or dist.group.WORLD
        name = grp.group_name
        self.hg = sm.rendezvous(trainer.grads, name)
        self.hs = sm.rendezvous(trainer.shadow_flat, name)
        self.world, self.rank = self.hg.world_size, self.hg.rank
        if self.world > 8:
            raise ValueError("PeerShardedDP supports up to 8 ranks")
        og, osh = int(getattr(self.hg, "offset", 0)), int(getattr(self.hs, "offset", 0))
        self.pg = [int(p) + og for p in self.hg.buffer_ptrs]
        self.ps = [int(p) + osh for p in self.hs.buffer_ptrs]
        self.pm = [p + trainer.nt_pad * 4 for p in self.pg]
        self.launches = trainer.bwd_launch_ranges()
        self.mains, self.tails = overlap_plan(self.launches, self.world, self.rank)
        self.by_launch = [[] for _ in self.launches]
        for (li, a, m) in self.mains:
            c = m // self.world
            self.by_launch[li].append((a + self.rank * c, a + (self.rank + 1) * c))
        self.comm = torch.cuda.Stream(device=trainer.grads.device)
        self.events = [torch.cuda.Event() for _ in self.launches]
        for ev in self.events:
            ev.record()
        trainer.set_bwd_events(self.events)

    def step(self, coords, target, n_global: int, stream=None):
        loss = self.tr.fwd_bwd(coords, target, n_global, stream=stream)
        self.reduce_and_apply(stream=stream)
        return loss

    def reduce_and_apply(self, stream=None):
        import torch
        tr = self.tr
        cur = torch.cuda.current_stream() if stream is None else stream
        first = True
        with torch.cuda.stream(self.comm):
            for li, ranges in enumerate(self.by_launch):
                self.comm.wait_event(self.events[li])   # this rank's group li is final
                self.hg.barrier(channel=0)              # ... and every other rank's
                if ranges:
                    tr.apply_peers(self.pg, self.ps, self.pm, ranges, [1] * len(ranges), False, first,
                                   stream=self.comm)
                    first = False
            self.comm.wait_stream(cur)                  # the whole local step (tails, MLP grads)
            self.hg.barrier(channel=0)
            tr.apply_peers(self.pg, self.ps, self.pm, self.tails, [0] * len(self.tails), True, first,
                           stream=self.comm)
            self.hg.barrier(channel=0)                  # every rank done reading gradients: the next
                                                        # fwd_bwd (queued behind it) may overwrite them
        cur.wait_stream(self.comm)


class MulticastShardedDP(PeerShardedDP):
    """SURVEY.md §8(e) item 3 as written: the same schedule as PeerShardedDP,
    with the gradient sum and the shadow broadcast done by the NVSwitch
    through an NVLS multicast object bound to every rank's grad and shadow
    buffers (fh_train_apply_multicast: multimem.ld_reduce, Adam in
    registers, multimem.st).  By default the multicast addresses and the
    cross-rank barrier come from torch symmetric memory (Trainer built with
    alloc=dp.symm_alloc, on a system with multicast support); `mc` =
    (grad, shadow) multicast addresses and `barrier` override them (tests:
    a one-device multicast object, no peers)."""

    def __init__(self, trainer, group=None, mc=None, barrier=None):
        import torch
        self.tr = trainer
        if trainer.shadow_flat is None:
            raise ValueError("MulticastShardedDP needs an fp16 table shadow")
        if mc is None:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as sm
            grp = group or dist.group.WORLD
            self.hg = sm.rendezvous(trainer.grads, grp.group_name)
            self.hs = sm.rendezvous(trainer.shadow_flat, grp.group_name)
            mg, ms = int(self.hg.multicast_ptr), int(self.hs.multicast_ptr)
            if not mg or not ms:
                raise ValueError("torch symmetric memory has no multicast object on this system")
            mc = (mg + int(getattr(self.hg, "offset", 0)), ms + int(getattr(self.hs, "offset", 0)))
            self.world, self.rank = self.hg.world_size, self.hg.rank
            self._barrier = barrier or (lambda: self.hg.barrier(channel=0))
        else:
            import torch.distributed as dist
            self.world = dist.get_world_size(group) if dist.is_initialized() else 1
            self.rank = dist.get_rank(group) if dist.is_initialized() else 0
            self._barrier = barrier or (lambda: None)
        self.mg, self.ms = mc
        self.mm = self.mg + trainer.nt_pad * 4
        self.launches = trainer.bwd_launch_ranges()
        self.mains, self.tails = overlap_plan(self.launches, self.world, self.rank)
        self.by_launch = [[] for _ in self.launches]
        for (li, a, m) in self.mains:
            c = m // self.world
            self.by_launch[li].append((a + self.rank * c, a + (self.rank + 1) * c))
        self.comm = torch.cuda.Stream(device=trainer.grads.device)
        self.events = [torch.cuda.Event() for _ in self.launches]
        for ev in self.events:
            ev.record()
        trainer.set_bwd_events(self.events)

    def reduce_and_apply(self, stream=None):
        import torch
        tr = self.tr
        cur = torch.cuda.current_stream() if stream is None else stream
        first = True
        with torch.cuda.stream(self.comm):
            for li, ranges in enumerate(self.by_launch):
                self.comm.wait_event(self.events[li])   # this rank's group li is final
                self._barrier()                         # ... and every other rank's
                if ranges:
                    tr.apply_multicast(self.mg, self.ms, self.mm, ranges, [1] * len(ranges), False, first,
                                       stream=self.comm)
                    first = False
            self.comm.wait_stream(cur)
            self._barrier()
            tr.apply_multicast(self.mg, self.ms, self.mm, self.tails, [0] * len(self.tails), True, first,
                               stream=self.comm)
            self._barrier()                             # gradients read by every rank: the next
                                                        # fwd_bwd may overwrite them
        cur.wait_stream(self.comm)


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
