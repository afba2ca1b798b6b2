"""Calibrate the paper's performance model (§III-C) on the B200 and report its accuracy alpha
 on held-out worker counts.

    python scripts/perf_model_fit.py [out.json]

1. MemoryContention, measured as the paper does it -- separately: with the
   instrumented build, the per-iteration cycles of the hogwild worker (148 CTAs, every layer
   reduced into the one shared weight store) minus those of the same kernel in sync mode
   (batch 592 = the same 148 CTAs x G; every CTA stores into a private slot), scaled to seconds
   per image per processing unit.
2. Training-phase times T(p) of the product build for p = CTAs x G images in flight,
   CTAs in {1, 2, 4, 8, 16, 37, 74, 148} (OPT_MAX_CTAS), i images per epoch (fewer for small p
   so the run stays short; the model takes i per point).
3. Fit CPI*OperationFactor and Prep on p in FIT, predict HELD, alpha per held-out point.
4. What-if table (Table III analogue): configs[3] and configs[4] epochs, more workers.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FPROP = 3_483_640.0              # forward FLOP per image, large net (eval column)
BPROP = 5_495_720.0 - FPROP      # backward + update FLOP per image
S = 1.965e9                      # SM clock (MEASURED_PEAKS.json sm_max_mhz)
G = 4
CTAS = [1, 2, 4, 8, 16, 37, 74, 148]
FIT = [1, 4, 16, 148]
HELD = [2, 8, 37, 74]


def measure_times():
    import torch

    import synthdata as sd
    from paper_1506_09067_b200 import OPT_MAX_CTAS, Net
    w = sd.WORKLOADS["config3"]
    xs, ys = sd.prototype_samples(w.seed, 0, 60000)
    X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
    out = {}
    for c in CTAS:
        i = 60000 if c >= 16 else 3750 * c
        net = Net(sd.ARCHS["large"], init_seed=w.seed)
        net.set_option(OPT_MAX_CTAS, c)
        net.train_epoch(X[:i], Y[:i], w.lr0)  # warm-up
        torch.cuda.synchronize()
        best = None
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            net.train_epoch(X[:i], Y[:i], w.lr0)
            b.record()
            torch.cuda.synchronize()
            t = a.elapsed_time(b) / 1e3
            best = t if best is None else min(best, t)
        out[c] = {"i": i, "p": c * G, "seconds": best}
        net.close()
    return out


def measure_contention():
    """cycles/iteration hogwild vs sync(592) from the instrumented build (separate process)."""
    code = r'''
import os, sys, json
sys.path.insert(0, %r)
import torch
import synthdata as sd
from paper_1506_09067_b200 import Net, OPT_SYNC_BATCH, SYNC
w = sd.WORKLOADS["config3"]
xs, ys = sd.prototype_samples(w.seed, 0, 60000)
X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
res = {}
for mode in ("hogwild", "sync"):
    net = Net(sd.ARCHS["large"], init_seed=w.seed)
    net.set_option(OPT_SYNC_BATCH, 592)
    for e in range(2):
        net.train_epoch(X, Y, w.lr0, SYNC if mode == "sync" else 0)
    torch.cuda.synchronize()
    t = net.phase_times()
    res[mode] = sum(v for k, v in t.items() if k not in ("c3din_warps", "c3gw_warps", "p19")) / (60000 / 4)
    net.close()
print(json.dumps(res))
''' % ROOT
    env = dict(os.environ, CHAOS_LIB=os.path.join(ROOT, "paper_1506_09067_b200", "libchaos_timing.so"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, check=True)
    return json.loads(r.stdout.strip().splitlines()[-1])


def main(out_path):
    from paper_1506_09067_b200 import perfmodel as pm
    times = measure_times()
    cyc = measure_contention()
    t148 = times[148]
    # extra cycles per iteration due to shared-weight reductions, as a fraction of the hogwild time,
    # converted to MemoryContention (seconds per image per unit): T_mem = MC * i * ep / p
    frac = max(0.0, (cyc["hogwild"] - cyc["sync"]) / cyc["hogwild"])
    mc = frac * t148["seconds"] * t148["p"] / t148["i"]
    pts = [(times[c]["p"], times[c]["seconds"], times[c]["i"]) for c in CTAS]
    # the model's i differs per point: fit on per-point rows
    rows = []
    for c in FIT:
        d = times[c]
        rows.append((d["p"], d["seconds"], d["i"]))
    # calibrate() takes one i; run it with rows normalised to i = 60000 (T scales linearly in i
    # apart from Prep, which the fit absorbs per point -- so fit on the full-i points only, and
    # check the small-p points as held-out predictions with their own i)
    fit_pts = [(p, t * 60000 / i) for p, t, i in rows]
    cal = pm.calibrate(fit_pts, 60000, 10000, 1, S, FPROP, BPROP, contention=mc)
    table = []
    for c in CTAS:
        d = times[c]
        pred = pm.predict_time(d["i"], 10000, 1, d["p"], S, cal.prep, FPROP, BPROP, cal.cpi_opf, mc,
                               parts=("prep", "train"))
        table.append({"ctas": c, "p": d["p"], "i": d["i"], "measured_s": d["seconds"], "predicted_s": pred,
                      "alpha_pct": pm.alpha(d["seconds"], pred), "held_out": c in HELD})
    held = [r["alpha_pct"] for r in table if r["held_out"]]
    whatif = pm.what_if(cal, S, FPROP, BPROP, [(592, 60000, 10000, 15), (592, 480000, 10000, 15),
                                                (1184, 60000, 10000, 15), (4736, 480000, 10000, 15)])
    rec = {"model": "PAPER.md §III-C rows (1)-(6), p = CTAs x G images in flight, s = 1.965 GHz",
           "fprop_flop": FPROP, "bprop_flop": BPROP, "cpi_x_operationfactor": cal.cpi_opf, "prep": cal.prep,
           "memory_contention_s_per_image_per_unit": mc, "contention_fraction": frac,
           "cycles_per_iteration": cyc, "fit_points_ctas": FIT, "fit_residual": cal.residual,
           "points": table, "alpha_heldout_mean_pct": sum(held) / len(held), "what_if": whatif,
           "paper_alpha_mean_pct": 15.4}
    print(json.dumps(rec, indent=1))
    if out_path:
        os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
        json.dump(rec, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
