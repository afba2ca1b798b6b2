"""Hogwild convergence vs images in flight (#CTAs x G): test loss / errors per epoch.

    python scripts/hogwild_sweep.py tiny config1 EPOCHS REPS "G:CTAS,G:CTAS,..." [sync:B,...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from paper_1506_09067_b200 import OPT_GROUP, OPT_MAX_CTAS, OPT_SYNC_BATCH, SYNC, Net  # noqa: E402


def main(arch, wname, epochs, reps, settings):
    w = sd.WORKLOADS[wname]
    d = sd.make_dataset(w)
    X, Y, Xt, Yt = [torch.from_numpy(a).cuda() for a in (d.x_train, d.y_train, d.x_test, d.y_test)]
    for st in settings.split(","):
        a, b = st.split(":")
        for r in range(reps):
            net = Net(sd.ARCHS[arch], init_seed=w.seed)
            if a == "sync":
                net.set_option(OPT_SYNC_BATCH, int(b))
                mode, inflight = SYNC, int(b)
            else:
                net.set_option(OPT_GROUP, int(a))
                net.set_option(OPT_MAX_CTAS, int(b))
                mode, inflight = 0, net.launch_info()["grid"] * int(a)
            t = time.time()
            curve = []
            for e in range(epochs):
                net.train_epoch(X, Y, w.lr0 * 0.9 ** e, mode)
                ml, ne = net.evaluate(Xt, Yt)
                curve.append((round(ml, 4), ne))
            print(arch, st, "in-flight", inflight, "rep", r, curve, f"{time.time() - t:.1f}s", flush=True)
            net.close()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5])
