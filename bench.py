"""Benchmark of the CHAOS hot path on B200 (contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload config3]

Workload (BASELINE.json configs[3]): the large net (conv20 4x4 -> pool2 -> conv60 3x3 -> pool2
floor -> conv100 2x2 -> pool2 -> FC 400->150 -> FC 150->10), hogwild (CHAOS) mode, synthetic
prototype+noise 29x29 fp32 data.  One *step* = one Training phase (epoch) over 60,000 images per
GPU: claim, forward, softmax-CE, back-propagation and the controlled-hogwild update of every
image, plus the NCCL weight average every K=1024 images per GPU when
N > 1 (row a9).  Weak scaling: 60,000 images per GPU per step (N=1: configs[3]; N>1: the
configs[4] generator, seed 2, rank r gets images [60000 r, 60000 (r+1))).  Evaluation (row a8)
is timed separately and reported under "eval".  Inputs (202 MB per GPU) exceed the 126 MB L2.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synthdata as sd  # noqa: E402

PER_GPU = 60000
K_AVG = 1024
METRIC = "training samples/sec (fwd+bwd+update) at 1/2/4/8 B200; % of FP32 roofline"
# FP32 FFMA peak from unit counts and clock: 148 SMs x 128 FFMA/clk x 2 FLOP x 1.965 GHz
N_SM = 148
FP32_PEAK_TFLOPS = N_SM * 128 * 2 * 1.965e9 / 1e12
# algorithmic FLOP per training image: forward of the conv outputs
# the pools use, argmax-only backward (gW and delta_in), 2 FLOP per parameter for the update
ALGO_FLOP = {"tiny": 202_990, "medium": 4_985_880, "large": 5_495_720,
             # Table I large (NEXT-1): 34,286,140 MAC (fwd 22,648,820; bwd 11,637,320) + 2 x 383,160
             "paper_large": 69_338_600,
             # Table I small (NEXT-1): fwd 160,330 MAC (conv 54,080 + 101,250, FC 4,500 + 500), argmax-only
             # bwd 46,020 MAC (conv2 gW + delta_in 2 x 11,250, conv1 gW 13,520, FC 2 x 5,000) + 2 x 6,405
             "paper_small": 425_510}
KERNEL_NET = {"tiny": "TinyNet", "medium": "MediumNet", "large": "LargeNet", "paper_large": "PaperLargeNet",
              "paper_small": "PaperSmallNet"}


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def make_data(world, rank, scaling="weak"):
    if scaling == "strong":
        # configs[3] (the D-5 headline): the 60,000 configs[3] images split into P contiguous shards
        w = sd.WORKLOADS["config3"]
        d = sd.make_dataset(w, PER_GPU, 10000)
        lo, hi = rank * PER_GPU // world, (rank + 1) * PER_GPU // world
        lo, hi = lo // 4 * 4, (hi // 4 * 4 if rank < world - 1 else PER_GPU)  # 16-B aligned image groups
        return w, d.x_train[lo:hi], d.y_train[lo:hi], d.x_test, d.y_test
    if world == 1:
        w = sd.WORKLOADS["config3"]
        d = sd.make_dataset(w, PER_GPU, 10000)
        return w, d.x_train, d.y_train, d.x_test, d.y_test
    w = sd.WORKLOADS["config4"]
    xs, ys = sd.prototype_samples(w.seed, rank * PER_GPU, PER_GPU)
    xt, yt = sd.prototype_samples(w.seed, w.n_train, 10000)
    return w, xs, ys, xt, yt


def host_identity():
    """lscpu model name and the host's logical CPU count (SURVEY D-8)."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.split(":")[0].strip() == "Model name":
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def cpu_baseline(arch, seconds=12.0):
    """The oracle as it stands (double, 1 thread) on a bounded sample of the same workload."""
    from oracle import Oracle
    w = sd.WORKLOADS["config3"]
    o = Oracle(sd.ARCHS[arch])
    p = sd.init_params(w.seed, o.blocks())
    xs, ys = sd.prototype_samples(w.seed, 0, 4000)
    # calibrate on 64 images, then run a sample sized to ~`seconds`
    t = time.perf_counter()
    o.train_sgd(p, xs[:64], ys[:64], w.lr0)
    per = (time.perf_counter() - t) / 64
    n = int(max(64, min(4000, seconds / per)))
    t = time.perf_counter()
    o.train_sgd(p, xs[:n], ys[:n], w.lr0)
    dt = time.perf_counter() - t
    return {"value": n / dt, "unit": "samples/s", "cores": 1, "kind": "oracle",
            "sample": f"sequential SGD (oracle, float64, 1 thread) over the first {n} images of configs[3]",
            **host_identity()}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import Oracle
    w = sd.WORKLOADS["config3"]
    o = Oracle(sd.ARCHS["large"])
    p = sd.init_params(w.seed, o.blocks())
    per_step = args.ref_images
    xs, ys = sd.prototype_samples(w.seed, 0, per_step * (args.warmup + args.steps))
    for s in range(args.warmup):
        p, _ = o.train_sgd(p, xs[s * per_step:(s + 1) * per_step], ys[s * per_step:(s + 1) * per_step], w.lr0)
    t = time.perf_counter()
    for s in range(args.warmup, args.warmup + args.steps):
        p, _ = o.train_sgd(p, xs[s * per_step:(s + 1) * per_step], ys[s * per_step:(s + 1) * per_step], w.lr0)
    dt = time.perf_counter() - t
    v = per_step * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "configs[3] large net, sequential SGD (the oracle) on a bounded sample",
                       "images_per_step": per_step, "arch": "large"},
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": 1, "kind": "oracle",
                             "sample": f"{per_step} images of configs[3] per step, oracle float64, 1 thread",
                             **host_identity()},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--arch", default="large", choices=["tiny", "medium", "large", "paper_small", "paper_large"])
    ap.add_argument("--k", type=int, default=K_AVG)
    ap.add_argument("--ref-images", type=int, default=400)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="hogwild", choices=["hogwild", "sync"],
                    help="hogwild (CHAOS, the headline) or the deterministic sync mode (multi-GPU: one "
                         "gradient all-reduce per global batch, SURVEY NEXT-4)")
    ap.add_argument("--sync-batch", type=int, default=64, help="global batch of --mode sync")
    ap.add_argument("--force-dist", action="store_true",
                    help="run the multi-GPU leg (NCCL process group, configs[4] shards, averaging every K) "
                         "even with one rank -- exercises the N>1 code path on one GPU")
    ap.add_argument("--avg", default="fused", choices=["interval", "async", "fused"],
                    help="multi-GPU hogwild averaging: 'interval' = one launch per K images, then a blocking "
                         "NCCL average; 'async' = one launch per shard with in-flight averages every K images on "
                         "a second stream (SURVEY NEXT-2); 'fused' = the persistent kernel averages the replicas "
                         "itself every K images through peer memory (CUDA IPC / NVLink), no reserved SMs")
    ap.add_argument("--reserve-sms", type=int, default=4, help="--avg async: SMs left to the comm kernels")
    ap.add_argument("--pavg-comm", type=int, default=None,
                    help="--avg fused: comm CTAs per GPU running the in-kernel rounds (default 1 for N <= 2, "
                         "else 2; 0 = the training CTAs run them between image groups)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: 60,000 images per GPU per step (configs[4] shards for N > 1); strong: the "
                         "60,000 configs[3] images split over the N GPUs (SURVEY D-5 headline)")
    ap.add_argument("--comm", default="torch", choices=["torch", "chaos"],
                    help="hogwild averaging collectives: torch.distributed or the library's own NCCL "
                         "communicator (chaos_dist_*)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_1506_09067_b200 import HOGWILD, OPT_RESERVE_SMS, Net
    from paper_1506_09067_b200.dist import DistTrainer

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    distributed = world > 1 or args.force_dist
    if distributed and args.mode == "hogwild" and args.avg in ("async", "fused"):  # fused: for its fallback
        # the averaging collectives run beside a persistent kernel that holds every other SM:
        # NCCL's blocks must all be co-resident on the reserved SMs (a channel block waiting for
        # a peer whose matching block cannot be scheduled would never finish), so cap them, and
        # leave NVLS (which wants many channels) off for this small-message path
        os.environ.setdefault("NCCL_MAX_CTAS", str(max(1, args.reserve_sms)))
        os.environ.setdefault("NCCL_NVLS_ENABLE", "0")
    if distributed:
        if "RANK" not in os.environ:  # --force-dist without a launcher: a one-rank group
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            os.environ.update(RANK="0", WORLD_SIZE="1", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=str(sk.getsockname()[1]))
            sk.close()
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.mode == "sync" and distributed:
        # sync mode: every rank holds the global training set (60,000 per GPU, weak scaling) and
        # computes its contiguous part of every global batch
        wl = sd.WORKLOADS["config4"]
        xs, ys = sd.prototype_samples(wl.seed, 0, PER_GPU * world)
        xt, yt = sd.prototype_samples(wl.seed, wl.n_train, 10000)
        w = wl
    else:
        w, xs, ys, xt, yt = make_data(world if not args.force_dist or args.scaling == "strong" else max(world, 2),
                                      rank, args.scaling)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    net = Net(sd.ARCHS[args.arch], init_seed=w.seed, stream=stream)
    use_async = distributed and args.mode == "hogwild" and args.avg == "async"
    use_fused = distributed and args.mode == "hogwild" and args.avg == "fused"
    if use_async:
        net.set_option(OPT_RESERVE_SMS, args.reserve_sms)
    info = net.launch_info()
    if args.mode == "sync" and args.sync_batch < info["group"] * N_SM:
        info["group"] = 1  # G unset: batches smaller than G x #SMs run one image per CTA (chaos.h)
    X = torch.from_numpy(xs).cuda()
    Y = torch.from_numpy(ys).cuda()
    Xt = torch.from_numpy(xt).cuda()
    Yt = torch.from_numpy(yt).cuda()
    trainer = DistTrainer(net, rank, world, args.k, force_collective=args.force_dist,
                          comm=args.comm if args.mode == "hogwild" else "torch")
    grad_buf = torch.zeros_like(net.device_params()) if args.mode == "sync" else None
    if use_fused and not trainer.setup_fused(args.pavg_comm):
        # a rank could not map a peer's exchange buffer (no peer access): every rank falls back to
        # the in-flight NCCL averaging -- caps set before any collective runs on the communicator
        use_fused, use_async = False, True
        net.set_option(OPT_RESERVE_SMS, args.reserve_sms)
        args.avg = "async (fused unavailable: " + getattr(trainer, "fused_error", "a peer rank") + ")"

    def step(Xs, Ys, lr_s):
        if args.mode == "sync":
            trainer.sync_epoch(Xs, Ys, lr_s, args.sync_batch, grad_buf)
        elif use_fused:
            trainer.epoch_fused(Xs, Ys, lr_s)
        elif use_async:
            trainer.epoch_async(Xs, Ys, lr_s)
        else:
            trainer.epoch(Xs, Ys, lr_s)

    def barrier():
        torch.cuda.synchronize()
        if distributed:
            dist.barrier(device_ids=[local])

    lr = w.lr0
    if distributed and (use_fused or use_async):
        # the in-kernel / in-flight averaging has only ever run on one GPU (replica emulations): if
        # its first step fails on ANY rank (a peer's rounds timing out is latched and raised by
        # sync), every rank drops to the blocking K-interval NCCL averaging -- agreed collectively,
        # before anything is timed -- and the line says so
        bad = 0
        try:
            step(X, Y, lr)
            net.sync()
            if os.environ.get("CHAOS_BENCH_FAIL_WARMUP"):  # test hook: exercise the fallback
                raise RuntimeError("CHAOS_BENCH_FAIL_WARMUP is set")
        except Exception as e:  # noqa: BLE001
            bad = 1
            print(f"[bench] rank {rank}: {args.avg} averaging failed in warm-up: {e}", file=sys.stderr)
        tb = torch.tensor([bad], dtype=torch.int64, device="cuda")
        dist.all_reduce(tb, op=dist.ReduceOp.MAX)
        if int(tb.item()):
            args.avg = f"interval ({args.avg} failed in warm-up on some rank)"
            use_fused = use_async = False
            net.set_option(OPT_RESERVE_SMS, 0)
            trainer._average(net.device_params())  # the same weights on every rank again
    for s in range(args.warmup):
        step(X, Y, lr * 0.9 ** s)
    net.sync()
    barrier()
    clk = ClockSampler(local)
    clk.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = trainer.n_launches + trainer.n_aux_launches
    fused0 = getattr(trainer, "n_fused_rounds", 0)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    barrier()
    t0.record(stream)
    for s in range(args.steps):
        ev[s][0].record(stream)
        step(X, Y, lr * 0.9 ** (args.warmup + s))
        ev[s][1].record(stream)
    t1.record(stream)
    barrier()
    clocks = clk.stop()
    elapsed = t0.elapsed_time(t1) / 1e3
    per_step_ms = [a.elapsed_time(b) for a, b in ev]
    launches = trainer.n_launches + trainer.n_aux_launches - launches0
    fused_rounds = getattr(trainer, "n_fused_rounds", 0) - fused0
    tmax = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
    if distributed:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    elapsed = float(tmax.item())
    per_gpu_images = int(ys.shape[0])
    if distributed:  # every rank's shard length (strong scaling: shards differ by a few images)
        nt = torch.tensor([per_gpu_images], dtype=torch.int64, device="cuda")
        dist.all_reduce(nt)
        images_per_step = int(nt.item())
    else:
        images_per_step = per_gpu_images
    total = images_per_step * args.steps
    value = total / elapsed
    train_loss = net.last_train_loss() if args.mode == "hogwild" else None

    # a8: evaluation on the averaged model (timed separately)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ml, ne = net.evaluate(Xt, Yt)
    e1.record(stream)
    torch.cuda.synchronize()
    eval_ms = e0.elapsed_time(e1)

    # e2e: the same metric end to end with HOST buffers: every step copies its images + labels
    # from pinned host memory (N=1 hogwild: inside the C-ABI call chaos_train_epoch_host; otherwise
    # an explicit H2D copy on the training stream before the step) and reads a result back (the
    # step's mean training loss / the updated parameters' first value), timed with barriers, max
    # over ranks
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(xs).pin_memory()
        Yh = torch.from_numpy(ys).pin_memory()
        host_entry = args.mode == "hogwild" and not distributed
        out_h = torch.zeros(1, dtype=torch.float32).pin_memory()

        def e2e_step(lr_s):
            if host_entry:
                net.train_epoch_host(Xh, Yh, lr_s)
                net.last_train_loss()
            elif use_async or use_fused:
                (trainer.epoch_fused if use_fused else trainer.epoch_async)(X, Y, lr_s, host=(Xh, Yh))
                out_h.copy_(net.device_params()[:1], non_blocking=True)
                torch.cuda.current_stream().synchronize()
            else:
                X.copy_(Xh, non_blocking=True)
                Y.copy_(Yh, non_blocking=True)
                step(X, Y, lr_s)
                out_h.copy_(net.device_params()[:1], non_blocking=True)
                torch.cuda.current_stream().synchronize()
        e2e_step(lr * 0.5)  # warm the staging buffers
        barrier()
        t = time.perf_counter()
        for s in range(args.steps):
            e2e_step(lr * 0.5)
        barrier()
        dt = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device="cuda")
        if distributed:
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e = {"value": images_per_step * args.steps / float(dt.item()), "unit": "samples/s",
               "h2d_bytes_per_step": int(Xh.numel() * 4 + Yh.numel() * 4),
               "d2h_bytes_per_step": 8 if host_entry else 4,
               "path": "chaos_train_epoch_host (C ABI, host buffers)" if host_entry
               else "DistTrainer.epoch_async(host=...) -> chaos_train_epoch_host_async: one launch gated "
                    "by the copy stream's landed-images counter, in-flight averages beside it" if use_async
               else "DistTrainer.epoch_fused(host=...) -> chaos_train_epoch_host_async: one gated launch "
                    "averaging in-kernel through peer memory" if use_fused
               else "pinned H2D copy + step on the training stream"}

    # per-interval all-reduce time (SURVEY D-6): the K-interval average of the parameters alone,
    # device-timed on the training stream (what one interval's blocking collective costs)
    allreduce_ms = None
    if distributed:
        params = net.device_params()
        buf = params.clone()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            trainer._average(buf)
        a0.record(stream)
        for _ in range(20):
            trainer._average(buf)
        a1.record(stream)
        torch.cuda.synchronize()
        allreduce_ms = a0.elapsed_time(a1) / 20

    if rank != 0:
        if distributed:
            dist.destroy_process_group()
        return
    # roofline of the dominant kernel: the persistent worker (one launch per step at N=1)
    kern_s = statistics.median(per_step_ms) / 1e3 if not distributed else elapsed / args.steps
    achieved = ALGO_FLOP[args.arch] * per_gpu_images / kern_s / 1e12
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "latest_traffic.json")
    if os.path.exists(tp):
        try:
            t = json.load(open(tp)).get(args.arch)
            traffic = t["dram_bytes_per_launch"] if t else None
            traffic_src = (f"not measured in this run: dram__bytes_read+write per launch from the committed "
                           f"ncu --set full capture {t.get('source', 'profiles/')}") if t else None
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": ((f"configs[3] {args.arch} net, hogwild (CHAOS), 60,000 images per GPU per step"
                                 if args.scaling == "weak" else
                                 f"configs[3] {args.arch} net, hogwild (CHAOS), 60,000 images split over "
                                 f"{world} GPUs per step (strong scaling)")
                                + ("" if not distributed else f"; {'configs[4] generator, ' if args.scaling == 'weak' else ''}NCCL average every {args.k}"
                                   + (f" images in flight (async, {args.reserve_sms} SMs reserved)" if use_async
                                      else " claimed images in-kernel through peer memory (fused), exact NCCL "
                                           "average at the end of the step" if use_fused
                                      else " images (blocking)")))
                   if args.mode == "hogwild" else
                   (f"configs[3] {args.arch} net, deterministic sync SGD, global batch {args.sync_batch}, "
                    f"60,000 images per GPU per step" + ("" if not distributed else
                                                         "; one NCCL gradient all-reduce per batch")),
                   "arch": args.arch, "mode": args.mode, "images_per_gpu_per_step": per_gpu_images,
                   "images_per_step": images_per_step,
                   "sync_batch": args.sync_batch if args.mode == "sync" else None,
                   "group_G": info["group"], "publish_group": info["group"], "ctas": info["grid"], "threads_per_cta": info["block"],
                   "smem_bytes_per_cta": info["smem_bytes"], "sync_interval_K": args.k if distributed else None,
                   "averaging": (args.avg if distributed and args.mode == "hogwild" else None),
                   "nccl_max_ctas": os.environ.get("NCCL_MAX_CTAS") if use_async else None,
                   "comm": (args.comm if distributed and args.mode == "hogwild" else None),
                   "l2": "inputs (202 MB/GPU) larger than the 126 MB L2", "parallelism": f"dp{world}"},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP32_PEAK_TFLOPS, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": f"chaos_worker<{KERNEL_NET[args.arch]},{info['group']},{info['block']},"
                               f"{'kHogwild' if args.mode == 'hogwild' else 'kSync'}>",
                     "flop_per_image": ALGO_FLOP[args.arch],
                     "peak_source": "148 SM x 128 FFMA/clk x 2 x 1.965 GHz (unit counts x max clock)"},
        "clocks": clocks,
        "gpu_launches": launches,
        "e2e": e2e,
        "eval": {"images": int(Yt.shape[0]), "ms": eval_ms, "samples_per_s": Yt.shape[0] / (eval_ms / 1e3),
                 "test_mean_loss": ml, "test_errors": ne},
        "train_mean_loss_last_step": train_loss,
        "per_step_ms": per_step_ms,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.arch)
    if distributed:
        line["allreduce_ms_per_interval"] = allreduce_ms
        line["eval"]["model"] = "the averaged replicas (identical on every rank after the epoch's final average)"
    if args.force_dist:
        line["config"]["force_dist"] = True
        line["collectives"] = trainer.n_collectives
    if use_fused:
        line["fused_rounds"] = fused_rounds  # in-kernel averaging rounds inside the timed region
        line["config"]["pavg_comm_ctas"] = trainer.comm_ctas
        line["roofline"]["kernel"] = line["roofline"]["kernel"][:-1] + ",PAVG>"
    emit(line)
    if distributed:
        dist.destroy_process_group()


def _json_stdout():
    """The JSON line is the only thing this script writes to stdout: file descriptor 1 is pointed at
    stderr for the run (NCCL prints its version banner to the C-level stdout under NCCL_DEBUG=WARN /
    VERSION), and the line goes to a duplicate of the original stdout."""
    global _OUT
    if "-h" in sys.argv or "--help" in sys.argv:
        return
    sys.stdout.flush()
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


_OUT = None


def emit(line):
    print(json.dumps(line), file=_OUT or sys.stdout, flush=True)


if __name__ == "__main__":
    _json_stdout()
    main()
