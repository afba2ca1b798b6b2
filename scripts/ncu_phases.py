"""Stall-sample / instruction share per kernel phase (line ranges of chaos_kernels.cuh, found by markers)."""
import csv
import re
import sys

SRC = "paper_1506_09067_b200/csrc/chaos_kernels.cuh"


def ranges():
    lines = open(SRC).read().split("\n")
    marks = []
    for i, l in enumerate(lines, 1):
        m = re.search(r"PHASE\(([^)]*)\)", l)
        if m:
            marks.append((i, m.group(1)))
    out = []
    for k, (i, name) in enumerate(marks):
        j = marks[k + 1][0] if k + 1 < len(marks) else len(lines) + 1
        out.append((i, j, name))
    return out


def main(path):
    rs = ranges()
    rows = list(csv.reader(open(path)))
    agg = {}
    fname = ""
    tot_s = tot_i = 0
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1]
        if not r or not r[0] or not r[0].isdigit():
            continue
        try:
            k = next(i for i in range(2, len(r) - 1) if r[i] == "-" and r[i + 1] == "-")
            s, ins = int(r[k + 2]), int(r[k + 5])
        except (StopIteration, ValueError, IndexError):
            continue
        tot_s += s
        tot_i += ins
        ln = int(r[0])
        name = "other"
        if fname.endswith("chaos_kernels.cuh"):
            for a, b, nm in rs:
                if a <= ln < b:
                    name = nm
        agg.setdefault(name, [0, 0])
        agg[name][0] += s
        agg[name][1] += ins
    for nm, (s, i) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{nm:28s} stall-samples {100*s/tot_s:5.1f}%   instructions {100*i/tot_i:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
