"""Aggregate an ncu 'cuda,sass' source-page CSV per CUDA source line.

Prints per line: stall samples, warp instructions, shared-memory wavefronts (and the
excessive ones = bank conflicts), and the top stall reasons.
  python scripts/ncu_lines.py gpurun_out/X_src.csv [top]
"""
import csv
import sys


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = None
    fname = ""
    out = []
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            # the second "Source" column shifts nothing: metric names are unique
            continue
        if hdr is None or not r or not r[0].isdigit():
            continue
        g = lambda k: num(r[hdr[k]]) if k in hdr and hdr[k] < len(r) else 0.0  # noqa: E731
        stalls = {k[6:]: g(k) for k in hdr if k.startswith("stall_") and "Not Issued" not in k}
        out.append((g("Warp Stall Sampling (All Samples)"), g("Instructions Executed"), g("L1 Wavefronts Shared"),
                    g("L1 Wavefronts Shared Excessive"), fname, int(r[0]), r[1][:70], stalls))
    ts = sum(o[0] for o in out) or 1
    ti = sum(o[1] for o in out) or 1
    tw = sum(o[2] for o in out) or 1
    tx = sum(o[3] for o in out)
    print(f"total samples {ts:.0f}, warp inst {ti:.0f}, smem wavefronts {tw:.0f} (excessive {tx:.0f})")
    for s, i, w, x, f, ln, src, st in sorted(out, key=lambda o: -o[0])[:top]:
        top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        reasons = " ".join(f"{k}:{100 * v / max(s, 1):.0f}" for k, v in top3 if v > 0)
        print(f"{100 * s / ts:5.1f}%smp {100 * i / ti:5.1f}%ins {100 * w / tw:5.1f}%wf {100 * x / tw:5.1f}%xs "
              f"{f}:{ln:<4d} {src:<70s} [{reasons}]")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
