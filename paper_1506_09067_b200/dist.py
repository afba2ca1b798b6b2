"""Multi-GPU plumbing (BASELINE.json north_star): one process per
GPU, contiguous data shards, and an allreduce-average of all parameters every K local images
(hogwild replicas); or the deterministic multi-GPU sync mode, one gradient all-reduce per batch.

Each rank trains its replica in hogwild mode on its shard; after every interval of K
images (and at the end of the shard) the replicas are averaged, w <- (1/P) sum_r w_r
(reading R11: average weights, not summed deltas).  The collective is
torch.distributed (NCCL on GPUs; gloo on CPU for the host-logic tests); the averaging
runs on the training stream so the next interval's kernel sees the averaged weights.
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [r*n/P, (r+1)*n/P) of rank r (SURVEY C-10), rounded to multiples of 4
    so every shard start keeps the 16-B image alignment the bulk copies use."""
    def edge(r):
        return (n * r // world) // 4 * 4 if r < world else n
    return edge(rank), edge(rank + 1)


def intervals(lo: int, hi: int, k: int) -> list[tuple[int, int]]:
    """Sync intervals of at most k images over [lo, hi); an average follows each one."""
    if k <= 0:
        return [(lo, hi)] if hi > lo else []
    return [(s, min(s + k, hi)) for s in range(lo, hi, k)]


def n_averages(n_local: int, k: int) -> int:
    return len(intervals(0, n_local, k))


def batch_part(b0: int, nb: int, rank: int, world: int) -> tuple[int, int]:
    """Rank r's contiguous part [s, e) of the global sync batch [b0, b0 + nb) (fixed split)."""
    return b0 + nb * rank // world, b0 + nb * (rank + 1) // world


def sum_(tensor, world: int, group=None, force: bool = False):
    """In-place all-reduce sum (the sync-mode gradient exchange)."""
    import torch.distributed as dist
    if world > 1 or force:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
    return tensor


def average_(tensor, world: int, group=None, force: bool = False):
    """In-place all-reduce average.  NCCL has ReduceOp.AVG; gloo does not (sum, then scale)."""
    import torch.distributed as dist
    if world == 1 and not force:
        return tensor
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(tensor, op=dist.ReduceOp.AVG, group=group)
    else:
        dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
        tensor.div_(world)
    return tensor


class DistTrainer:
    """Trains one replica per rank with periodic averaging (hogwild), or all ranks as one
    deterministic sync-SGD trainer (``sync_epoch``).

    ``net`` needs ``train_epoch(images, labels, lr)`` and ``device_params()`` (the chaos.Net
    API) -- plus ``batch_gradient`` / ``apply_gradient`` for the sync mode; tests substitute a
    CPU stand-in with the same methods."""

    def __init__(self, net, rank: int, world: int, k: int, group=None, force_collective: bool = False):
        """force_collective: run the K-interval schedule and the collectives even with one rank
        (exercises the multi-GPU code path on one GPU)."""
        self.net, self.rank, self.world, self.k, self.group = net, rank, world, k, group
        self.force = force_collective
        self.n_collectives = 0
        self.n_launches = 0

    def epoch(self, images, labels, lr: float, lo: int = 0, hi: int | None = None):
        """One Training phase over this rank's images[lo:hi) (already sharded by the caller)."""
        hi = int(labels.shape[0]) if hi is None else hi
        params = self.net.device_params()
        multi = self.world > 1 or self.force
        for s, e in intervals(lo, hi, self.k if multi else 0):
            self.net.train_epoch(images[s:e], labels[s:e], lr)
            self.n_launches += 1
            if multi:
                average_(params, self.world, self.group, force=self.force)
                self.n_collectives += 1

    def sync_epoch(self, images, labels, lr: float, batch: int, grad=None):
        """Deterministic multi-GPU sync SGD: for every consecutive global
        batch of ``batch`` images, rank r computes the fixed-order gradient sum of its contiguous
        part (``batch_part``), the parts are all-reduced (sum), and every rank applies
        W -= lr * G.  ``images``/``labels`` hold the whole (replicated) training set.  With one
        rank this is exactly chaos_train_epoch(SYNC); with P ranks it is the same update up to
        the summation order, and bitwise reproducible for a fixed P and topology."""
        import torch
        params = self.net.device_params()
        if grad is None:
            grad = torch.zeros_like(params)
        n = int(labels.shape[0])
        for b0 in range(0, n, batch):
            nb = min(batch, n - b0)
            s, e = batch_part(b0, nb, self.rank, self.world)
            self.net.batch_gradient(images[s:e], labels[s:e], grad)
            self.n_launches += 2
            if self.world > 1 or self.force:
                sum_(grad, self.world, self.group, force=self.force)
                self.n_collectives += 1
            self.net.apply_gradient(grad, lr)
        return grad
