"""Per-phase wall time of the hogwild worker (instrumented build, clock64 marks after barriers).

    CHAOS_LIB=paper_1506_09067_b200/libchaos_timing.so python scripts/phase_times.py [arch] [epochs]

Prints, per phase, the cycles per CTA iteration (G images) averaged over CTAs and its share.
The instrumented build adds a few instructions per phase; absolute throughput is read from bench.py.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("CHAOS_LIB", os.path.join(ROOT, "paper_1506_09067_b200", "libchaos_timing.so"))

import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from paper_1506_09067_b200 import Net  # noqa: E402


def main(arch="large", epochs=2, sync_batch=0):
    w = sd.WORKLOADS["config3"]
    xs, ys = sd.prototype_samples(w.seed, 0, 60000)
    X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    net = Net(sd.ARCHS[arch], init_seed=w.seed)
    info = net.launch_info()
    for e in range(epochs):
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st.record()
        if sync_batch:
            from paper_1506_09067_b200 import OPT_SYNC_BATCH, SYNC
            net.set_option(OPT_SYNC_BATCH, sync_batch)
            net.train_epoch(X, Y, w.lr0 * 0.9 ** e, SYNC)
        else:
            net.train_epoch(X, Y, w.lr0 * 0.9 ** e)
        en.record()
        torch.cuda.synchronize()
        ms = st.elapsed_time(en)
    t = net.phase_times()
    iters = 60000 / info["group"]
    # slots 17 / 18 (c3din_warps, c3gw_warps) and 19 time warp groups *inside* other phases:
    # shown, but not part of the sum
    inner = ("c3din_warps", "c3gw_warps", "p19")
    tot = sum(v for k, v in t.items() if k not in inner)
    print(f"{arch}: last epoch {ms:.2f} ms ({60000 / ms * 1e3 / 1e6:.3f} M samples/s, timing build); "
          f"grid {info['grid']}, G {info['group']}; cycles per CTA iteration (all CTAs averaged):")
    for k, v in t.items():
        if v:
            print(f"  {k:12s} {v / iters:10.0f} cyc/iter  {100 * v / tot:5.1f}%" + ("  (inside a phase)" if k in inner else ""))
    print(f"  {'total':12s} {tot / iters:10.0f} cyc/iter  = {tot / 60000:.0f} cycles per image per SM")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "large", int(sys.argv[2]) if len(sys.argv) > 2 else 2,
         int(sys.argv[3]) if len(sys.argv) > 3 else 0)
