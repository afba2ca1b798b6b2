"""Aggregate an ncu 'cuda,sass' source-page CSV per CUDA source line (stall samples, instructions)."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    fname = ""
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0]:
            continue
        try:
            k = next(i for i in range(2, len(r) - 1) if r[i] == "-" and r[i + 1] == "-")
        except StopIteration:
            continue
        vals = r[k + 2:]
        try:
            samples = int(vals[0])
            inst = int(vals[3])
        except (ValueError, IndexError):
            continue
        out.append((samples, inst, fname, int(r[0]), ",".join(r[1:k])[:90]))
    tot_s = sum(o[0] for o in out) or 1
    tot_i = sum(o[1] for o in out) or 1
    print(f"total stall samples {tot_s}, warp instructions {tot_i}")
    for s, i, f, ln, src in sorted(out, reverse=True)[:top]:
        print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% inst  {f}:{ln:<4d} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
