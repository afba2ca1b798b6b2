"""Full oracle training runs for the accuracy gates (calls only oracle/ + synthdata/).

Writes tests/golden/oracle_runs/<name>.json with per-epoch test loss / errors of
the oracle's sequential SGD (or sync-batch SGD) on BASELINE.json workloads:

  python scripts/oracle_reference_runs.py config1_seq        # tiny, 15 epochs (minutes)
  python scripts/oracle_reference_runs.py config3_seq        # large, 15 epochs (~1 h)

The lr schedule is lr0 * 0.9**e (BASELINE.json configs[1]; reading R6).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synthdata as sd  # noqa: E402
from oracle import Oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "oracle_runs")

RUNS = {
    # name: (workload, mode, batch, epochs)
    "config0_sync1": ("config0", "sync", 1, 1),
    "config1_seq": ("config1", "seq", 1, 15),
    "config1_sync64": ("config1", "sync", 64, 15),
    "config2_seq": ("config2", "seq", 1, 15),
    "config3_seq": ("config3", "seq", 1, 15),
    "config3_sync64_e1": ("config3", "sync", 64, 1),
    "config2_sync64_e1": ("config2", "sync", 64, 1),
    # the paper's Table I small net (NEXT-1) on the configs[1] data
    "paper_small_seq": ("config1", "seq", 1, 15, "paper_small"),
    # the Table I large net (NEXT-1): 69 MFLOP per image, so a bounded slice of the configs[1]
    # data (the first 3,000 training / 1,000 test images), 3 epochs (~10 min of oracle time)
    "paper_large_seq": ("config1", "seq", 1, 3, "paper_large", 3000, 1000),
}


def run(name):
    wname, mode, batch, epochs = RUNS[name][:4]
    w = sd.WORKLOADS[wname]
    arch = RUNS[name][4] if len(RUNS[name]) > 4 else w.arch
    ntr, nte = (RUNS[name][5], RUNS[name][6]) if len(RUNS[name]) > 6 else (None, None)
    d = sd.make_dataset(w, ntr, nte)
    o = Oracle(sd.ARCHS[arch])
    p = sd.init_params(w.seed, o.blocks()).astype(np.float64)
    rec = {"run": name, "workload": wname, "arch": arch, "mode": mode, "batch": batch, "epochs": epochs,
           "data_sha256": d.sha256(), "lr0": w.lr0, "n_train": len(d.y_train), "n_test": len(d.y_test),
           "per_epoch": []}
    t0 = time.time()
    ckpt = os.path.join(OUT, name + "_ckpt.npy")
    start = 0
    prev = os.path.join(OUT, name + ".json")
    if os.path.exists(ckpt) and os.path.exists(prev):
        old = json.load(open(prev))
        if old.get("data_sha256") == rec["data_sha256"] and old["per_epoch"]:
            # resume after the last completed epoch (the checkpoint holds its parameters)
            rec["per_epoch"] = old["per_epoch"]
            start = len(old["per_epoch"])
            p = np.load(ckpt)
            t0 -= old["per_epoch"][-1]["elapsed_s"]
    for e in range(start, epochs):
        lr = w.lr0 * 0.9 ** e
        if mode == "seq":
            p, sl = o.train_sgd(p, d.x_train, d.y_train, lr)
        else:
            p, sl = o.train_sync(p, d.x_train, d.y_train, lr, batch)
        tl, te = o.evaluate(p, d.x_test, d.y_test)
        rec["per_epoch"].append({"epoch": e + 1, "lr": lr, "train_mean_loss": sl / len(d.y_train),
                                 "test_mean_loss": tl, "test_errors": te, "n_test": len(d.y_test),
                                 "elapsed_s": time.time() - t0})
        print(name, rec["per_epoch"][-1], flush=True)
        os.makedirs(OUT, exist_ok=True)
        with open(os.path.join(OUT, name + ".json"), "w") as f:
            json.dump(rec, f, indent=1)
        if epochs > 1:
            np.save(ckpt, p)
    if epochs == 1 or name.startswith("config0"):
        np.save(os.path.join(OUT, name + "_params.npy"), p)


if __name__ == "__main__":
    for n in sys.argv[1:]:
        run(n)
