"""Multi-GPU host logic on CPU: world_size-2 ``gloo`` process groups.

The product path averages the replicas' weights with NCCL every K local images
(BASELINE.json configs[3..4]; reading R11: average weights).  Here the
same ``DistTrainer`` runs over gloo with a CPU stand-in for ``chaos.Net`` that has
the two methods the trainer uses, so sharding, interval boundaries, the number of
collectives and the averaging semantics are checked without a GPU.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1506_09067_b200.dist import DistTrainer, async_targets, batch_part, intervals, n_averages, shard_range


def test_shard_range_partitions_and_aligns():
    for n in (0, 4, 60000, 480000, 1001):
        for world in (1, 2, 3, 4, 8):
            edges = [shard_range(n, r, world) for r in range(world)]
            assert edges[0][0] == 0 and edges[-1][1] == n
            for (a, b), (c, d) in zip(edges, edges[1:]):
                assert b == c and a <= b
            for a, _ in edges:
                assert a % 4 == 0  # 16-B aligned image groups for the bulk copies


def test_intervals_and_average_counts():
    assert intervals(0, 10, 4) == [(0, 4), (4, 8), (8, 10)]
    assert intervals(5, 5, 4) == []
    assert intervals(0, 10, 0) == [(0, 10)]
    # averages per epoch
    assert n_averages(30000, 1024) == 30
    assert n_averages(15000, 1024) == 15
    assert n_averages(7500, 1024) == 8
    assert n_averages(60000, 256) == 235
    assert n_averages(60000, 1024) == 59
    assert n_averages(60000, 8192) == 8


class FakeNet:
    """CPU stand-in for chaos.Net: 'training' adds lr * (rank+1) * sum(images) to every weight;
    the 'gradient' of an image set is (sum of its rows, as a per-weight vector)."""

    def __init__(self, n, rank):
        self.w = torch.arange(n, dtype=torch.float32)
        self.rank = rank
        self.calls = []

    def device_params(self):
        return self.w

    def train_epoch(self, images, labels, lr):
        self.calls.append(int(labels.shape[0]))
        self.w += lr * (self.rank + 1) * float(images.sum())

    def batch_gradient(self, images, labels, grad):
        # a gradient that depends on the weights (like a real one) and on every image
        self.calls.append(int(labels.shape[0]))
        grad.zero_()
        for row in images:
            grad += row.sum() * torch.tanh(self.w)

    def apply_gradient(self, grad, lr):
        self.w -= lr * grad


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, k, lr, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 1000
        lo, hi = shard_range(n, rank, world)
        X = torch.ones(n, 3)
        Y = torch.zeros(n, dtype=torch.int32)
        net = FakeNet(16, rank)
        w0 = net.w.clone()
        tr = DistTrainer(net, rank, world, k)
        tr.epoch(X[lo:hi], Y[lo:hi], lr)
        gathered = [torch.zeros_like(net.w) for _ in range(world)]
        dist.all_gather(gathered, net.w)
        q.put((rank, net.calls, tr.n_collectives, w0.numpy(), net.w.numpy(), [g.numpy() for g in gathered]))
    finally:
        dist.destroy_process_group()


def _run(world, k, lr):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, lr, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def test_gloo_world2_average_every_k():
    world, k, lr = 2, 128, 0.01
    out = _run(world, k, lr)
    for rank, calls, ncoll, w0, w, gathered in out:
        lo, hi = shard_range(1000, rank, world)
        assert sum(calls) == hi - lo
        assert all(c <= k for c in calls)
        assert ncoll == n_averages(hi - lo, k)
        # after the final average every rank holds bitwise-identical parameters
        for g in gathered:
            np.testing.assert_array_equal(g, gathered[0])
    # averaged model = mean of the replicas: each interval of c images (all-ones rows of
    # 3 features) moves rank r by lr*(r+1)*3c, then the average takes the mean over ranks
    w0 = out[0][3]
    expect = w0.astype(np.float64).copy()
    ncalls = [out[r][1] for r in range(world)]
    for i in range(max(len(c) for c in ncalls)):
        delta = np.mean([lr * (r + 1) * 3 * (ncalls[r][i] if i < len(ncalls[r]) else 0) for r in range(world)])
        expect += delta
    np.testing.assert_allclose(out[0][4], expect, rtol=1e-5)


def test_gloo_world2_lr0_leaves_params_unchanged():
    out = _run(2, 256, 0.0)
    for _, _, _, w0, w, _ in out:
        np.testing.assert_array_equal(w, w0)


def test_single_process_skips_collective():
    net = FakeNet(4, 0)
    tr = DistTrainer(net, 0, 1, 8)
    tr.epoch(torch.ones(20, 3), torch.zeros(20, dtype=torch.int32), 0.1)
    assert tr.n_collectives == 0
    assert net.calls == [20]  # one launch over the whole shard


def test_batch_part_partitions_every_batch():
    for nb in (0, 1, 7, 64, 65):
        for world in (1, 2, 3, 8):
            parts = [batch_part(100, nb, r, world) for r in range(world)]
            assert parts[0][0] == 100 and parts[-1][1] == 100 + nb
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c


def _sync_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(0)
        X = torch.rand(37, 5, generator=g, dtype=torch.float64)
        Y = torch.zeros(37, dtype=torch.int32)
        net = FakeNet(16, rank)
        net.w = net.w.double() / 16
        tr = DistTrainer(net, rank, world, 0)
        tr.sync_epoch(X, Y, 0.01, batch=8)
        q.put((rank, net.w.numpy(), tr.n_collectives))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sync_epoch_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sync_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # the same sync SGD in one process: every batch's gradient at the batch-start weights, summed
    g = torch.Generator().manual_seed(0)
    X = torch.rand(37, 5, generator=g, dtype=torch.float64)
    w = torch.arange(16, dtype=torch.float64) / 16
    for b0 in range(0, 37, 8):
        G = torch.zeros(16, dtype=torch.float64)
        for row in X[b0:b0 + 8]:
            G += row.sum() * torch.tanh(w)
        w = w - 0.01 * G
    for rank, wr, ncoll in out:
        assert ncoll == 5  # one all-reduce per batch (37 = 4*8 + 5)
        np.testing.assert_allclose(wr, w.numpy(), rtol=1e-12)
    np.testing.assert_array_equal(out[0][1], out[1][1])  # replicas stay bitwise identical


def test_async_targets():
    assert async_targets(10, 4) == [4, 8]
    assert async_targets(8, 4) == [4]          # the shard end gets the final exact average
    assert async_targets(3, 4) == [] and async_targets(10, 0) == []
    assert len(async_targets(7500, 1024)) + 1 == n_averages(7500, 1024)


class FakeAsyncNet(FakeNet):
    """Stand-in for the asynchronous-averaging API: train_epoch only enqueues (as the real launch
    is asynchronous); progress_wait(t) lets the 'device' train up to image t; avg_apply first lets
    `lag` more images train -- local progress made while the collective ran -- then adds
    avg - snap.  Every image adds lr*(rank+1)*3 to every weight (all-ones rows of 3 features)."""

    stream = None

    def __init__(self, n, rank, lag):
        super().__init__(n, rank)
        self.lag, self.enq, self.done, self.lr = lag, 0, 0, 0.0
        self.residual = []

    def progress_enqueued(self):
        return self.enq

    def train_epoch(self, images, labels, lr):
        assert self.done == self.enq  # the previous epoch completed (final average waited for it)
        self.calls.append(int(labels.shape[0]))
        self.enq += int(labels.shape[0])
        self.lr = lr

    def _advance(self, t):
        t = min(t, self.enq)
        self.w += (t - self.done) * self.lr * (self.rank + 1) * 3
        self.done = max(self.done, t)

    def progress_wait(self, target, stream):
        assert target <= self.enq
        self._advance(target)

    def avg_snapshot(self, snap, stream):
        snap.copy_(self.w)

    def avg_apply(self, avg, snap, stream):
        d0 = self.done
        self._advance(self.done + self.lag)
        self.w += avg - snap
        # weights after the apply minus the average: exactly the local progress since the snapshot
        self.residual.append((self.w - avg).max().item() - (self.done - d0) * self.lr * (self.rank + 1) * 3)

    def sync(self):
        self._advance(self.enq)


def _async_worker(rank, world, port, k, lr, lag, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 1000
        lo, hi = shard_range(n, rank, world)
        X = torch.ones(n, 3)
        Y = torch.zeros(n, dtype=torch.int32)
        net = FakeAsyncNet(16, rank, lag)
        net.w = net.w.double()
        w0 = net.w.clone()
        tr = DistTrainer(net, rank, world, k)
        for _ in range(2):
            tr.epoch_async(X, Y, lr, lo, hi)
        gathered = [torch.zeros_like(net.w) for _ in range(world)]
        dist.all_gather(gathered, net.w)
        q.put((rank, net.calls, tr.n_collectives, w0.numpy(), [g.numpy() for g in gathered], net.residual))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("lag", [0, 37])
def test_gloo_world2_async_average(lag):
    """NEXT-2: in-flight averages keep the local progress made during the collective (the
    sum over ranks is preserved), the final average leaves identical replicas, and the result is
    the mean of the replicas' total progress whatever the timing (additive updates)."""
    world, k, lr = 2, 128, 0.01
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_async_worker, args=(r, world, port, k, lr, lag, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sizes = [shard_range(1000, r, world) for r in range(world)]
    for rank, calls, ncoll, w0, gathered, residual in out:
        lo, hi = sizes[rank]
        assert len(residual) == 2 * len(async_targets(hi - lo, k)) and max(map(abs, residual)) < 1e-9
        assert calls == [hi - lo, hi - lo]  # one launch per epoch, no K-interval split
        assert ncoll == 2 * (len(async_targets(hi - lo, k)) + 1)
        np.testing.assert_array_equal(gathered[1], gathered[0])
    expect = out[0][3] + 2 * np.mean([(hi - lo) * lr * (r + 1) * 3 for r, (lo, hi) in enumerate(sizes)])
    np.testing.assert_allclose(out[0][4][0], expect, rtol=1e-12)


def _uneven_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # shards of 1025 and 1021 images: ceil(n/K) differs per rank at K = 1024
        edges = [(0, 1025), (1025, 2046)]
        lo, hi = edges[rank]
        X = torch.ones(2046, 3)
        Y = torch.zeros(2046, dtype=torch.int32)
        out = []
        for kind in ("interval", "async"):
            net = FakeAsyncNet(8, rank, 5) if kind == "async" else FakeNet(8, rank)
            net.w = net.w.double()
            tr = DistTrainer(net, rank, world, 1024)
            (tr.epoch_async if kind == "async" else tr.epoch)(X, Y, 0.01, lo, hi)
            gathered = [torch.zeros_like(net.w) for _ in range(world)]
            dist.all_gather(gathered, net.w)
            out.append((kind, tr.n_collectives, sum(net.calls), [g.numpy() for g in gathered]))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_uneven_shards_agree_on_collective_count():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_uneven_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (_, a), (_, b) in [(res[0], res[1])]:
        for (kind, nc0, n0, g0), (_, nc1, n1, _) in zip(a, b):
            assert nc0 == nc1, kind  # 2 intervals on both ranks; async: no in-flight average
            assert (n0, n1) == (1025, 1021)
            np.testing.assert_array_equal(g0[0], g0[1])
    assert [o[1] for o in res[0][1]] == [2, 1]


class FakeFusedNet(FakeNet):
    """FakeNet plus the chaos_pavg_* host surface: the exchange buffer's 'IPC handle' names the rank
    that made it; opened peers and armed rounds are recorded (the in-kernel rounds themselves are
    GPU-tested: tests/test_gpu_pavg.py)."""

    def pavg_setup(self, rank, world, k, nslice=0):
        self.setup = (rank, world, k)
        self.opened = {}
        self.armed = []

    def pavg_ipc_handle(self):
        return bytes([self.rank]) + b"h" * 63

    def pavg_open_peer(self, peer, handle):
        assert len(handle) == 64 and peer not in self.opened
        self.opened[peer] = handle[0]

    def pavg_arm(self, rounds):
        self.armed.append(rounds)


def _fused_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # uneven shards (1029 / 1021 / 1000 images at K = 256): every rank arms the rounds of the
        # shortest shard, launches once per epoch and ends with one exact average
        edges = [(0, 1029), (1029, 2050), (2050, 3050)]
        lo, hi = edges[rank]
        X = torch.ones(3050, 3)
        Y = torch.zeros(3050, dtype=torch.int32)
        net = FakeFusedNet(8, rank)
        net.w = net.w.double()
        tr = DistTrainer(net, rank, world, 256)
        with pytest.raises(RuntimeError):
            tr.epoch_fused(X, Y, 0.01, lo, hi)  # setup_fused first
        tr.setup_fused()
        for _ in range(2):
            tr.epoch_fused(X, Y, 0.01, lo, hi)
        gathered = [torch.zeros_like(net.w) for _ in range(world)]
        dist.all_gather(gathered, net.w)
        q.put((rank, net.setup, net.opened, net.armed, net.calls, tr.n_collectives, tr.n_fused_rounds,
               [g.numpy() for g in gathered]))
    finally:
        dist.destroy_process_group()


def test_gloo_world3_fused_averaging_host_logic():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rounds = len(async_targets(1000, 256))
    assert rounds == 3
    sizes = [1029, 1021, 1000]
    for rank, setup, opened, armed, calls, ncoll, nfused, gathered in res:
        assert setup == (rank, world, 256)
        assert opened == {q: q for q in range(world) if q != rank}  # every peer's handle, at its index
        assert armed == [rounds, rounds]
        assert calls == [sizes[rank], sizes[rank]]  # one launch per epoch
        assert ncoll == 2 and nfused == 2 * rounds
        for g in gathered[1:]:
            np.testing.assert_array_equal(g, gathered[0])  # identical after the exact average


class FakeFusedNetNoPeer(FakeFusedNet):
    """Rank 1 cannot map its peers' buffers (no peer access)."""

    def pavg_open_peer(self, peer, handle):
        if self.rank == 1:
            raise RuntimeError("peer access unsupported")
        super().pavg_open_peer(peer, handle)


def _fused_fallback_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        net = FakeFusedNetNoPeer(8, rank)
        tr = DistTrainer(net, rank, world, 256)
        q.put((rank, tr.setup_fused(), getattr(tr, "fused_error", None)))
    finally:
        dist.destroy_process_group()


def test_gloo_world3_fused_setup_agrees_on_failure():
    # one rank failing to map a peer's exchange buffer makes setup_fused return False on EVERY rank
    # (bench.py then falls back to the NCCL averaging everywhere: no rank waits for a missing peer)
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_fallback_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [ok for _, ok, _ in res] == [False, False, False]
    assert res[1][2] is not None and "peer access" in res[1][2]
