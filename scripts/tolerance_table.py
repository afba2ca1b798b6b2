"""Evidence for the parity tolerance (R9 / R16; SURVEY C-15): plain fp32 (torch CPU
autograd, float32) against the float64 oracle on the same inputs and trajectories.

    python scripts/tolerance_table.py > profiles/r3/tolerance_table.md

Per net: (a) a 13-image gradient at the initial weights; (b) 3 sync steps (B = 64 on 150
images, lr 0.05, seed 7 -- the GPU test's trajectory) -- worst element-wise ratio to the R9
bound (1e-4 * max(|ref|, 1e-2 ||ref||_inf)) and norm ratio (1e-5 ||ref||) over the tensors, for
the weights after the steps and for the step itself, plus the smallest pool top-2 gap on the
oracle trajectory (near-ties, C-15).  Calls only oracle/ and torch (no product code)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from helpers import min_pool_gaps, parity_report, torch_grad  # noqa: E402
from oracle import Oracle  # noqa: E402


def fp32_sync(arch, p0, X, Y, lr, B):
    w = torch.tensor(p0, dtype=torch.float32).numpy()
    for s0 in range(0, len(Y), B):
        _, g, _ = torch_grad(arch, w, X[s0:s0 + B], Y[s0:s0 + B], dtype=torch.float32)
        w = (w - np.float32(lr) * g.astype(np.float32)).astype(np.float32)
    return w.astype(np.float64)


def main():
    torch.set_num_threads(os.cpu_count() or 1)
    print("| net | 13-image gradient: elem / norm (x R9) | 3 sync steps B=64, weights: elem / norm | step: elem / norm | min top-2 pool gap on the trajectory |")
    print("|---|---|---|---|---|")
    for name in ["tiny", "medium", "large", "paper_small", "paper_large"]:
        arch = sd.ARCHS[name]
        o = Oracle(arch)
        d = sd.prototype_dataset(5, 13, 0)
        p = sd.init_params(5, o.blocks()).astype(np.float64)
        ref = sum(o.sample_grad(p, d.x_train[i], d.y_train[i])[1] for i in range(13))
        _, g32, _ = torch_grad(arch, p.astype(np.float32), d.x_train, d.y_train, dtype=torch.float32)
        _, wg, wgn, _ = parity_report(g32, ref, o.blocks())
        seed, n, B, lr = 7, 150, 64, 0.05
        d = sd.prototype_dataset(seed, n, 0)
        p = sd.init_params(seed, o.blocks()).astype(np.float64)
        refp, _ = o.train_sync(p, d.x_train, d.y_train, lr, B)
        got = fp32_sync(arch, p, d.x_train, d.y_train, lr, B)
        _, ww, wwn, _ = parity_report(got, refp, o.blocks())
        _, ws, wsn, _ = parity_report(got - p, refp - p, o.blocks(), rel=1e-3, floor=1e-2, norm_rel=1e-4)
        gap = 1.0
        w = p.copy()
        for s0 in range(0, n, B):
            for i in range(s0, min(s0 + B, n)):
                gap = min(gap, min(min_pool_gaps(arch, o.forward(w, d.x_train[i])[1]), default=1.0))
            w, _ = o.train_sync(w, d.x_train[s0:s0 + B], d.y_train[s0:s0 + B], lr, B)
        print(f"| {name} | {wg:.3g} / {wgn:.3g} | {ww:.3g} / {wwn:.3g} | {ws:.3g} / {wsn:.3g} (step bound 1e-3 / 1e-4) "
              f"| {gap:.2e} |", flush=True)


if __name__ == "__main__":
    main()
