"""Hogwild convergence vs images in flight (#CTAs x G): test loss / errors after E epochs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthdata as sd  # noqa: E402
from paper_1506_09067_b200 import OPT_GROUP, OPT_MAX_CTAS, OPT_SYNC_BATCH, SYNC, Net  # noqa: E402


def run(arch, wname, epochs, settings):
    w = sd.WORKLOADS[wname]
    d = sd.make_dataset(w)
    X, Y, Xt, Yt = [torch.from_numpy(a).cuda() for a in (d.x_train, d.y_train, d.x_test, d.y_test)]
    for (mode, g, ctas) in settings:
        net = Net(sd.ARCHS[arch], init_seed=w.seed)
        net.set_option(OPT_GROUP, g)
        net.set_option(OPT_MAX_CTAS, ctas)
        if mode == "sync":
            net.set_option(OPT_SYNC_BATCH, ctas)
        curve = []
        t = time.time()
        for e in range(epochs):
            net.train_epoch(X, Y, w.lr0 * 0.9 ** e, SYNC if mode == "sync" else 0)
            ml, ne = net.evaluate(Xt, Yt)
            curve.append((round(ml, 5), ne))
        torch.cuda.synchronize()
        print(arch, mode, "G", g, "ctas/B", ctas, "in-flight", g * ctas if mode != "sync" else ctas,
              curve, f"{time.time() - t:.2f}s", flush=True)
        net.close()


if __name__ == "__main__":
    ep = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    run("tiny", "config1", ep, [("hog", 8, 148), ("hog", 8, 74), ("hog", 1, 148), ("hog", 8, 37), ("hog", 1, 74),
                                ("sync", 8, 1184), ("sync", 8, 592)])
    run("large", "config3", ep, [("hog", 4, 148), ("hog", 1, 148), ("hog", 4, 74), ("sync", 4, 592)])
