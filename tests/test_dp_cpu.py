"""Multi-process data-parallel host logic on CPU (gloo, world size 2).

The GPU box in this run has one GPU, so the N>1 path is covered here: each
rank computes its shard's gradients with the oracle (as a stand-in for the
per-rank kernels), the product's all-reduce helper sums them, and the result
must equal the single-process gradient of the global batch (the 1/N_global
scaling of R12 makes the split exact).  Also: even sharding and the
replica-identity check."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_03836_b200 import dp


def test_shard_even_split():
    for n in (0, 1, 7, 1000, 2 ** 24):
        for w in (1, 2, 3, 8):
            parts = [dp.shard(n, r, w) for r in range(w)]
            assert sum(c for _, c in parts) == n
            assert parts[0][0] == 0
            for (s0, c0), (s1, _) in zip(parts, parts[1:]):
                assert s1 == s0 + c0
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    with pytest.raises(ValueError):
        dp.shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import workloads as W
        from oracle import train as T
        g = W.rng(0)
        layers = W.draw_mlp(g, W.MLPConfig((16, 64, 64, 1)))
        n_global = 1001
        x = g.standard_normal((n_global, 16))
        t = g.random(n_global)
        s, c = dp.shard(n_global, rank, world)
        y, cache = T.mlp_forward(x[s:s + c], layers, emulate_bf16=False)
        _, dy = T.mse_loss(y, t[s:s + c], n_global)
        grads, _ = T.mlp_backward(dy, layers, cache, emulate_bf16=False)
        flat = torch.from_numpy(np.concatenate([np.concatenate([a.ravel(), b.ravel()]) for a, b in grads]))
        dp.allreduce_grads(flat)
        out[rank] = flat.numpy().copy()
        # replicas: identical tensors compare equal, perturbed ones do not
        same = torch.arange(10, dtype=torch.float32)
        diff = same + (rank * 1e-3)
        out[f"same{rank}"] = dp.replicas_identical(same)
        out[f"diff{rank}"] = dp.replicas_identical(diff)
    finally:
        dist.destroy_process_group()


class _MockTrainer:
    """CPU stand-in with the attributes dp.ShardedDP uses; fwd_bwd writes a
    deterministic per-(rank, step) gradient (overwriting, as
    fh_train_fwd_bwd does), apply_sharded runs the oracle's Adam on the given
    range (the GPU kernels are tested in test_train_gpu)."""

    def __init__(self, n_table, n_mlp, world, rank):
        from oracle import train as T
        self.T = T
        q = 4 * world
        self.n_table, self.world, self.rank = n_table, world, rank
        self.nt_pad = (n_table + q - 1) // q * q
        self.grads = torch.zeros(self.nt_pad + n_mlp)
        self.mlp_grad = self.grads[self.nt_pad:]
        g = np.random.default_rng(99)
        self.p = g.uniform(-1e-4, 1e-4, n_table)
        self.pm = g.uniform(-0.1, 0.1, n_mlp)
        self.m, self.v = np.zeros(n_table), np.zeros(n_table)
        self.mm, self.mv = np.zeros(n_mlp), np.zeros(n_mlp)
        self.shadow_flat = torch.zeros(self.nt_pad, dtype=torch.float16)
        self.shadow_flat[:n_table] = torch.from_numpy(self.p).half()
        self.step_no = 0

    @staticmethod
    def local_grad(rank, step, n):
        return np.random.default_rng(1000 * step + rank).standard_normal(n).astype(np.float32)

    def fwd_bwd(self, coords, target, n_global, stream=None):
        nm = self.mlp_grad.numel()
        g = torch.from_numpy(self.local_grad(self.rank, self.step_no, self.n_table + nm))
        self.grads[:self.n_table] = g[:self.n_table]
        self.mlp_grad.copy_(g[self.n_table:])

    def apply_sharded(self, begin, end, shard, stream=None):
        self.step_no += 1
        s = self.step_no
        g = shard.numpy()[:end - begin].astype(np.float64)
        self.p[begin:end], self.m[begin:end], self.v[begin:end] = self.T.adam_step(
            self.p[begin:end], g, self.m[begin:end], self.v[begin:end], s)
        self.pm, self.mm, self.mv = self.T.adam_step(self.pm, self.mlp_grad.numpy().astype(np.float64),
                                                     self.mm, self.mv, s)
        self.shadow_flat[begin:end] = torch.from_numpy(self.p[begin:end]).half()


def _sharded_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = _MockTrainer(1001, 37, world, rank)
        sdp = dp.ShardedDP(tr)
        for _ in range(3):
            sdp.step(None, None, 1)
        out[f"shadow{rank}"] = tr.shadow_flat[:tr.n_table].float().numpy().copy()
        out[f"mlp{rank}"] = tr.pm.copy()
        out[f"same{rank}"] = dp.replicas_identical(tr.shadow_flat)
    finally:
        dist.destroy_process_group()


def test_sharded_adam_equals_replicated_adam():
    """Reduce-scatter + sharded Adam + all-gather gives every rank the same
    fp16 shadow as a single process running Adam on the summed gradients."""
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_sharded_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    ref = _MockTrainer(1001, 37, 1, 0)
    from oracle import train as T
    for s in range(1, 4):
        g = sum(_MockTrainer.local_grad(r, s - 1, 1001 + 37).astype(np.float32)
                for r in range(world)).astype(np.float64)
        ref.p, ref.m, ref.v = T.adam_step(ref.p, g[:1001], ref.m, ref.v, s)
        ref.pm, ref.mm, ref.mv = T.adam_step(ref.pm, g[1001:], ref.mm, ref.mv, s)
    exp = torch.from_numpy(ref.p).half().float().numpy()
    for r in range(world):
        assert np.array_equal(res[f"shadow{r}"], exp)
        assert np.allclose(res[f"mlp{r}"], ref.pm, rtol=0, atol=1e-12)
        assert res[f"same{r}"]


def test_allreduce_of_shard_grads_equals_global_grad():
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    import workloads as W
    from oracle import train as T
    g = W.rng(0)
    layers = W.draw_mlp(g, W.MLPConfig((16, 64, 64, 1)))
    x = g.standard_normal((1001, 16))
    t = g.random(1001)
    y, cache = T.mlp_forward(x, layers, emulate_bf16=False)
    _, dy = T.mse_loss(y, t, 1001)
    grads, _ = T.mlp_backward(dy, layers, cache, emulate_bf16=False)
    ref = np.concatenate([np.concatenate([a.ravel(), b.ravel()]) for a, b in grads])
    for r in range(world):
        assert np.allclose(res[r], ref, rtol=1e-10, atol=1e-14)
    assert np.array_equal(res[0], res[1])
    assert res["same0"] and res["same1"]
    assert not res["diff0"] and not res["diff1"]


# ---------------------------------------------- overlapped reduction (§8(e) 2)
def test_overlap_plan_partitions_the_table():
    """Every table element is in exactly one rank's main chunk or in a tail
    (replicated); chunks are 4-aligned and equal across ranks."""
    g = np.random.default_rng(3)
    for trial in range(40):
        n = int(g.integers(1, 5000))
        cuts = sorted(set(int(c) for c in g.integers(0, n, int(g.integers(0, 8))))) + [n]
        rngs, b = [], 0
        for c in cuts:
            if c > b:
                rngs.append((b, c))
            b = c
        launches = [rngs[i::2] for i in range(2)]   # ranges spread over two launches
        for W in (1, 2, 3, 8):
            cover = np.zeros(n, np.int64)
            for r in range(W):
                mains, tails = dp.overlap_plan(launches, W, r)
                for (_, a, m) in mains:
                    assert a % 4 == 0 and m % (4 * W) == 0
                    c = m // W
                    cover[a + r * c:a + (r + 1) * c] += 1
            for (b, e) in tails:
                assert e - b < 4 * W + 4
                cover[b:e] += 1
            assert np.all(cover == 1), (trial, W)


class _MockOverlapTrainer(_MockTrainer):
    """Adds the overlap interface: two backward launches covering the table,
    and apply_ranges running the oracle's Adam on each range."""

    def bwd_launch_ranges(self):
        n = self.n_table
        return [[(0, 301)], [(301, 702), (702, n)]]

    def set_bwd_events(self, events):
        pass

    def apply_ranges(self, ranges, grads, stream=None):
        self.step_no += 1
        s = self.step_no
        for (b, e), g in zip(ranges, grads):
            gg = g.numpy()[:e - b].astype(np.float64)
            self.p[b:e], self.m[b:e], self.v[b:e] = self.T.adam_step(self.p[b:e], gg, self.m[b:e], self.v[b:e], s)
            self.shadow_flat[b:e] = torch.from_numpy(self.p[b:e]).half()
        self.pm, self.mm, self.mv = self.T.adam_step(self.pm, self.mlp_grad.numpy().astype(np.float64),
                                                     self.mm, self.mv, s)


def _overlap_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr = _MockOverlapTrainer(1001, 37, world, rank)
        odp = dp.OverlappedShardedDP(tr)
        for _ in range(3):
            odp.step(None, None, 1)
        out[f"shadow{rank}"] = tr.shadow_flat[:tr.n_table].float().numpy().copy()
        out[f"mlp{rank}"] = tr.pm.copy()
        out[f"same{rank}"] = dp.replicas_identical(tr.shadow_flat)
    finally:
        dist.destroy_process_group()


def test_overlapped_sharded_adam_equals_replicated_adam():
    """Per-launch reduce-scatter + all-reduced tails + one Adam over the
    owned ranges + all-gather gives every rank the single-process result."""
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_overlap_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    ref = _MockTrainer(1001, 37, 1, 0)
    from oracle import train as T
    for s in range(1, 4):
        g = sum(_MockTrainer.local_grad(r, s - 1, 1001 + 37).astype(np.float32)
                for r in range(world)).astype(np.float64)
        ref.p, ref.m, ref.v = T.adam_step(ref.p, g[:1001], ref.m, ref.v, s)
        ref.pm, ref.mm, ref.mv = T.adam_step(ref.pm, g[1001:], ref.mm, ref.mv, s)
    exp = torch.from_numpy(ref.p).half().float().numpy()
    for r in range(world):
        assert np.array_equal(res[f"shadow{r}"], exp)
        assert np.allclose(res[f"mlp{r}"], ref.pm, rtol=0, atol=1e-12)
        assert res[f"same{r}"]
