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


def async_targets(n_local: int, k: int) -> list[int]:
    """Progress points (images into the shard) of the in-flight averages of ``epoch_async``:
    k, 2k, ... strictly inside the shard; the end of the shard gets the final, exact average."""
    return list(range(k, n_local, k)) if k > 0 else []


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


def check_async_comm(comm: str, net) -> None:
    """The in-flight averages run beside a persistent hogwild launch that holds every other SM:
    all blocks of each collective must be co-resident on the reserved SMs, else one can spin on a
    peer block that is never scheduled.  comm "chaos": chaos_dist_init caps the communicator at
    the reserved SMs (ncclCommInitRankConfig maxCTAs / nvlsCTAs).  comm "torch": NCCL reads
    NCCL_MAX_CTAS / NCCL_NVLS_ENABLE when the process group is created -- they must have been set
    to at most the reserved SMs / 0 (bench.py does); raise otherwise instead of risking a hang."""
    from .chaos import OPT_RESERVE_SMS
    reserve = net.get_option(OPT_RESERVE_SMS)
    if reserve < 1:
        raise RuntimeError("asynchronous averaging needs CHAOS_OPT_RESERVE_SMS >= 1 (SMs for the collectives)")
    if comm == "torch":
        import os
        cap = os.environ.get("NCCL_MAX_CTAS")
        if cap is None or not cap.isdigit() or int(cap) > reserve or os.environ.get("NCCL_NVLS_ENABLE") != "0":
            raise RuntimeError(f"asynchronous averaging over torch.distributed needs NCCL_MAX_CTAS <= {reserve} "
                               "(the reserved SMs) and NCCL_NVLS_ENABLE=0 set before the process group is "
                               "created; or use comm='chaos', whose communicator the library caps itself")


class DistTrainer:
    """Trains one replica per rank with periodic averaging (hogwild), or all ranks as one
    deterministic sync-SGD trainer (``sync_epoch``).

    ``net`` needs ``train_epoch(images, labels, lr)`` and ``device_params()`` (the chaos.Net
    API) -- plus ``batch_gradient`` / ``apply_gradient`` for the sync mode; tests substitute a
    CPU stand-in with the same methods."""

    def __init__(self, net, rank: int, world: int, k: int, group=None, force_collective: bool = False,
                 comm: str = "torch"):
        """force_collective: run the K-interval schedule and the collectives even with one rank
        (exercises the multi-GPU code path on one GPU).  comm: "torch" = torch.distributed
        all-reduces; "chaos" = the library's own NCCL communicator (chaos_dist_*; its unique id
        travels over the torch process group once, here)."""
        self.net, self.rank, self.world, self.k, self.group = net, rank, world, k, group
        self.force = force_collective
        self.comm = comm
        if comm == "chaos" and (world > 1 or force_collective):
            import torch
            import torch.distributed as dist
            uid = net.dist_unique_id() if rank == 0 else bytes(128)
            t = torch.tensor(list(uid), dtype=torch.uint8,
                             device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
            dist.broadcast(t, src=0, group=group)
            net.dist_init(bytes(t.cpu().tolist()), rank, world)
        elif comm not in ("torch", "chaos"):
            raise ValueError(f"comm must be 'torch' or 'chaos', not {comm!r}")
        self.n_collectives = 0
        self.n_launches = 0
        self.n_aux_launches = 0  # epoch_async: progress-wait + apply kernels
        self._agreed_cache = {}

    def _average(self, tensor, stream=None):
        """In-place average over the ranks: torch.distributed (current stream) or chaos_dist_*."""
        if self.comm == "chaos":
            import torch
            if tensor.data_ptr() == self.net.device_params().data_ptr() and stream is None:
                self.net.dist_average()  # the net's stream
            else:
                self.net.dist_average_buffer(tensor, stream if stream is not None else torch.cuda.current_stream())
        else:
            average_(tensor, self.world, self.group, force=self.force)

    def _agreed(self, n_local: int, op: str) -> int:
        """MIN / MAX of the shard length over ranks (cached per length): the number of
        collectives per epoch must be the same on every rank even when shard sizes differ."""
        key = (n_local, op)
        if key not in self._agreed_cache:
            import torch
            import torch.distributed as dist
            on_gpu = dist.get_backend(self.group) == "nccl"
            t = torch.tensor([n_local], dtype=torch.int64, device="cuda" if on_gpu else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MIN if op == "min" else dist.ReduceOp.MAX, group=self.group)
            self._agreed_cache[key] = int(t.item())
        return self._agreed_cache[key]

    def _on_net_stream(self, t):
        """Collectives on the tensors the training kernels write go on the net's stream (a
        Net(stream=s) need not be torch's current stream), so they are ordered after the launches
        and before the next ones."""
        import contextlib

        import torch
        if getattr(t, "is_cuda", False) and getattr(self.net, "stream", None) is not None:
            return torch.cuda.stream(self.net.stream)
        return contextlib.nullcontext()

    def epoch(self, images, labels, lr: float, lo: int = 0, hi: int | None = None):
        """One Training phase over this rank's images[lo:hi) (already sharded by the caller):
        one launch per interval of K images, each followed by a blocking average.  Every rank runs
        ceil(max shard / K) intervals (a shorter shard ends with empty ones) so the collectives
        match."""
        hi = int(labels.shape[0]) if hi is None else hi
        params = self.net.device_params()
        multi = self.world > 1 or self.force
        if not multi or self.k <= 0:
            if hi > lo:
                self.net.train_epoch(images[lo:hi], labels[lo:hi], lr)
                self.n_launches += 1
            if multi:
                with self._on_net_stream(params):
                    self._average(params)
                self.n_collectives += 1
            return
        count = max(1, -(-self._agreed(hi - lo, "max") // self.k))
        for i in range(count):
            s, e = lo + i * self.k, min(lo + (i + 1) * self.k, hi)
            if e > s:
                self.net.train_epoch(images[s:e], labels[s:e], lr)
                self.n_launches += 1
            with self._on_net_stream(params):
                self._average(params)
            self.n_collectives += 1

    def _launch(self, images, labels, lr, lo, hi, host, chunks):
        """Training launch(es) over [lo, hi) on the net's stream.  host = pinned CPU (images,
        labels) of the same rows: the rows are copied into images/labels in `chunks` pieces on a
        copy stream and each piece trains as soon as its own copy has landed (the H2D transfer
        overlaps training -- the end-to-end path; one launch per piece)."""
        if hi <= lo:
            return
        if host is None:
            self.net.train_epoch(images[lo:hi], labels[lo:hi], lr)
            self.n_launches += 1
            return
        if hasattr(self.net, "train_epoch_host_async"):
            # the library's streamed host entry: one launch gated by the landed-images counter
            self.net.train_epoch_host_async(host[0][lo:hi], host[1][lo:hi], lr)
            self.n_launches += 1
            return
        import torch
        ts = self.net.stream
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream()
        cps = self._copy_stream
        cps.wait_stream(ts)  # earlier launches no longer read the buffers being overwritten
        step = max(4, -(-(hi - lo) // chunks) // 4 * 4)
        for s in range(lo, hi, step):
            e = min(s + step, hi)
            with torch.cuda.stream(cps):
                images[s:e].copy_(host[0][s:e], non_blocking=True)
                labels[s:e].copy_(host[1][s:e], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cps)
            ts.wait_event(ev)
            self.net.train_epoch(images[s:e], labels[s:e], lr)
            self.n_launches += 1

    def epoch_async(self, images, labels, lr: float, lo: int = 0, hi: int | None = None, host=None,
                    chunks: int = 8):
        """One Training phase with asynchronous averaging:
        ONE hogwild launch over the whole shard on the net's stream (run with
        CHAOS_OPT_RESERVE_SMS > 0 so the comm kernels find free SMs), and on a second stream, for
        every target t in ``async_targets`` of the shortest shard (the collective count must match on
        every rank): wait until the device progress counter has passed t
        images, snapshot the weights, all-reduce the snapshot (average), add (avg - snapshot) to
        the live weights -- local updates made during the collective are kept (the CHAOS
        "arbitrary order of synchronization", across replicas).  After the launch
        completes, one exact in-place average leaves every rank with identical weights.  Sum over
        ranks of the weights is preserved by every in-flight average (each adds P*avg - sum snap
        = 0), so with additive updates the final weights equal the mean of the replicas' total
        progress, whatever the timing.  No K-interval tail: the kernel never drains mid-shard.
        ``host``/``chunks``: see ``_launch`` (the progress counter spans the chunk launches).
        NCCL's blocks must fit the reserved SMs all at once (set NCCL_MAX_CTAS <= reserved SMs
        before the process group is created; bench.py does), else a collective could wait for a
        block that cannot be scheduled beside the persistent training kernel."""
        import contextlib

        import torch
        hi = int(labels.shape[0]) if hi is None else hi
        net = self.net
        params = net.device_params()
        if not (self.world > 1 or self.force):
            self._launch(images, labels, lr, lo, hi, host, chunks)
            return
        cuda = params.is_cuda
        if cuda:
            check_async_comm(self.comm, net)
        if getattr(self, "_async_bufs", None) is None:
            self._async_bufs = (torch.empty_like(params), torch.empty_like(params),
                                torch.cuda.Stream() if cuda else None)
        snap, avg, cs = self._async_bufs
        ts = net.stream if cuda else None
        scope = torch.cuda.stream(cs) if cuda else contextlib.nullcontext()
        if cuda:
            cs.wait_stream(ts)  # earlier work on the weights precedes this epoch's snapshots
        n_min = self._agreed(hi - lo, "min")  # before the launch: its host sync must not stall the comm stream
        base = net.progress_enqueued()
        self._launch(images, labels, lr, lo, hi, host, chunks)
        with scope:
            for t in async_targets(n_min, self.k):
                net.progress_wait(base + t, cs)
                net.avg_snapshot(snap, cs)
                avg.copy_(snap)
                self._average(avg, cs)
                net.avg_apply(avg, snap, cs)
                self.n_collectives += 1
                self.n_aux_launches += 2
            if cuda:
                cs.wait_stream(ts)  # the launch has completed
            else:
                net.sync()
            self._average(params, cs)
            self.n_collectives += 1
        if cuda:
            ts.wait_stream(cs)

    def setup_fused(self, comm_ctas: int | None = None):
        """Fused in-kernel averaging (fused variant; chaos_pavg_*):
        the persistent hogwild kernel itself averages the replicas through peer memory -- no
        collective launch beside it.  ``comm_ctas`` (default 1 for up to 2 ranks, else 2) extra CTAs
        of the launch run the rounds (8 slices each) while the training CTAs never stall; 0 = the
        training CTAs run them between image groups (148 slices).  Each rank allocates its exchange
        buffer (snapshot ring + flags) and the ranks trade its CUDA IPC handle (an all-gather of 64
        bytes); every rank maps every other rank's buffer (NVLink peer access).  Returns False -- on
        every rank -- if any rank could not map a peer's buffer (then use epoch_async / epoch)."""
        import torch
        import torch.distributed as dist
        if comm_ctas is None:
            comm_ctas = 1 if self.world <= 2 else 2
        if hasattr(self.net, "set_option"):
            from .chaos import OPT_PAVG_COMM_CTAS
            self.net.set_option(OPT_PAVG_COMM_CTAS, comm_ctas)
        self.comm_ctas = comm_ctas
        self.net.pavg_setup(self.rank, self.world, self.k, 8 * comm_ctas if comm_ctas else 0)
        ok = True
        if self.world > 1:
            on_gpu = dist.get_backend(self.group) == "nccl"
            h = torch.tensor(list(self.net.pavg_ipc_handle()), dtype=torch.uint8)
            if on_gpu:
                h = h.cuda()
            hs = [torch.zeros_like(h) for _ in range(self.world)]
            dist.all_gather(hs, h, group=self.group)
            try:
                for q, hq in enumerate(hs):
                    if q != self.rank:
                        self.net.pavg_open_peer(q, bytes(hq.cpu().tolist()))
            except Exception as e:  # e.g. no peer access between the devices
                ok = False
                self.fused_error = f"{type(e).__name__}: {e}"
            # every rank must agree: a kernel waiting for a peer that never averages would hang
            t = torch.tensor([1 if ok else 0], dtype=torch.int64, device="cuda" if on_gpu else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
            ok = bool(t.item())
        self.n_fused_rounds = 0
        self._fused = ok
        return ok

    def epoch_fused(self, images, labels, lr: float, lo: int = 0, hi: int | None = None, host=None,
                    chunks: int = 8):
        """One Training phase with the fused averaging (after ``setup_fused``): ONE hogwild launch
        over the shard with ``len(async_targets(shortest shard, K))`` in-kernel averaging rounds
        armed -- the same count on every rank (a round's CTAs wait for every replica's snapshot of
        their slices) -- then one exact average of the parameters on the net's stream, after which
        the replicas are identical.  ``host``/``chunks``: see ``_launch`` (the host entry is one
        gated launch, so the armed rounds cover the whole shard)."""
        hi = int(labels.shape[0]) if hi is None else hi
        if not (self.world > 1 or self.force):
            self._launch(images, labels, lr, lo, hi, host, chunks)
            return
        if not getattr(self, "_fused", False):
            raise RuntimeError("epoch_fused needs setup_fused() first")
        rounds = len(async_targets(self._agreed(hi - lo, "min"), self.k))
        self.net.pavg_arm(rounds)
        self._launch(images, labels, lr, lo, hi, host, chunks)
        self.n_fused_rounds += rounds
        params = self.net.device_params()
        with self._on_net_stream(params):
            self._average(params)
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
                with self._on_net_stream(grad):
                    sum_(grad, self.world, self.group, force=self.force)
                self.n_collectives += 1
            self.net.apply_gradient(grad, lr)
        return grad
