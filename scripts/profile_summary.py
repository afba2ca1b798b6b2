"""Summarise one gpu_round.sh call (gpurun_out/TAG_*) into profiles/TAG/ (tracked).

    python scripts/profile_summary.py r1a

Writes: bench.json (the bench line), launches.csv (the ncu launch list of the bench command),
launch_shares.txt (per-kernel share of the device time), ncu_metrics.txt (key counters of the
`ncu --set full` capture of the hogwild worker), lines.txt / phases.txt (per source line / per
kernel phase stall samples, instructions and shared-memory wavefronts), pytest.log, and
traffic.json (dram read+write bytes per launch of the captured kernel, used by bench.py).
"""
import csv
import io
import re
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict
from contextlib import redirect_stdout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_requests_op_red.sum", "lts__t_sectors_op_red.sum", "sm__cycles_elapsed.avg", "smsp__cycles_active.avg",
        "launch__grid_size", "launch__block_size"]


D7 = (r"^derived__(sm|smsp)__sass_thread_inst_executed_op_(ffma|fadd|fmul)_pred_on"
      r"|^smsp__sass_thread_inst_executed_op_(ffma|fadd|fmul)_pred_on\.sum$"
      r"|^l1tex__data_pipe_lsu_wavefronts_mem_shared(_op_ld|_op_st)?\.sum(\.pct_of_peak_sustained_elapsed)?$"
      r"|^l1tex__data_bank_conflicts_pipe_lsu_mem_shared(_op_ld|_op_st)?\.sum$"
      r"|^lts__t_(sectors|bytes|requests)\.sum(\.per_second|\.pct_of_peak_sustained_elapsed)?$"
      r"|^lts__t_(sectors|requests)_srcunit_tex_op_red\.sum$|^lts__t_(sectors|requests)_op_red\.sum$"
      r"|^l1tex__t_requests_pipe_lsu_mem_global_op_red\.sum$|^l1tex__t_sectors_pipe_lsu_mem_global_op_red\.sum$"
      r"|^dram__bytes\.sum\.per_second$|^sm__pipe_fma_cycles_active\.avg\.pct_of_peak_sustained_(active|elapsed)$"
      r"|^sm__pipe_fmaheavy_cycles_active|^sm__inst_executed_pipe_(fma|fmalite|fmaheavy|lsu|alu)\.avg\.pct")


def main(tag):
    src = os.path.join(ROOT, "gpurun_out", tag)
    out = os.path.join(ROOT, "profiles", tag)
    os.makedirs(out, exist_ok=True)
    for suf, name in [("_bench.json", "bench.json"), ("_launches.csv", "launches.csv"), ("_pytest.log", "pytest.log"),
                      ("_smoke.log", "smoke.log"), ("_smi.txt", "nvidia_smi.txt")]:
        if os.path.exists(src + suf):
            shutil.copy(src + suf, os.path.join(out, name))
    if os.path.exists(src + "_launches.csv"):
        rows = [r for r in csv.reader(open(src + "_launches.csv")) if len(r) > 5]
        hdr = rows[0]
        agg = defaultdict(lambda: [0, 0.0])
        for r in rows[1:]:
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                a = agg[d["Kernel Name"]]
                a[0] += 1
                a[1] += float(d["Metric Value"].replace(",", ""))
        tot = sum(v[1] for v in agg.values()) or 1
        with open(os.path.join(out, "launch_shares.txt"), "w") as f:
            f.write("launches  total_us  share  kernel (ncu --metrics gpu__time_duration.sum --clock-control none)\n")
            for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
                f.write(f"{v[0]:8d} {v[1] / 1e3:9.1f} {100 * v[1] / tot:5.1f}%  {k}\n")
    rep = src + "_full.ncu-rep"
    if os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        r = list(csv.reader(io.StringIO(raw)))
        hdr, units, vals = r[0], r[1], r[2]
        m = {h: (u, v) for h, u, v in zip(hdr, units, vals)}
        with open(os.path.join(out, "ncu_metrics.txt"), "w") as f:
            f.write(f"kernel: {m.get('Kernel Name', ('', ''))[1]}\n")
            for k in KEYS:
                if k in m:
                    f.write(f"{k:70s} {m[k][0]:>10s} {m[k][1]}\n")
            for k in sorted(m):
                if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio"):
                    f.write(f"{k:70s} {m[k][0]:>10s} {m[k][1]}\n")
            # SURVEY D-7 counters (names as this ncu build reports them): executed FP32 work per cycle
            # (derived ..._x2 = thread FFMA x 2 + FADD + FMUL per cycle), shared-memory pipe
            # utilisation, L2 throughput and the RED traffic of the hogwild publishes
            f.write("# D-7\n")
            for k in sorted(m):
                if re.search(D7, k):
                    f.write(f"{k:70s} {m[k][0]:>10s} {m[k][1]}\n")

        def val(k):
            u, v = m[k]
            v = float(v.replace(",", ""))
            return v * {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1}.get(u, 1)
        traffic = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        json.dump({"dram_bytes_per_launch": traffic, "kernel": m.get("Kernel Name", ("", ""))[1],
                   "source": f"profiles/{tag}/ncu_metrics.txt"}, open(os.path.join(out, "traffic.json"), "w"), indent=1)
        arch = "large"
        if os.path.exists(src + "_bench.json"):
            try:
                arch = json.loads(open(src + "_bench.json").read().strip().splitlines()[-1])["config"]["arch"]
            except Exception:
                pass
        lt = os.path.join(ROOT, "profiles", "latest_traffic.json")
        cur = json.load(open(lt)) if os.path.exists(lt) else {}
        cur[arch] = {"dram_bytes_per_launch": traffic, "source": f"profiles/{tag}/ncu_metrics.txt"}
        json.dump(cur, open(lt, "w"), indent=1)
        srccsv = src + "_full_src.csv"
        s = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                           capture_output=True, text=True).stdout
        open(srccsv, "w").write(s)
        import ncu_lines
        import ncu_phases
        buf = io.StringIO()
        with redirect_stdout(buf):
            ncu_lines.main(srccsv, 60)
        open(os.path.join(out, "lines.txt"), "w").write(buf.getvalue())
        buf = io.StringIO()
        with redirect_stdout(buf):
            ncu_phases.main(srccsv)
        open(os.path.join(out, "phases.txt"), "w").write(buf.getvalue())
    print("wrote", out, sorted(os.listdir(out)))


if __name__ == "__main__":
    main(sys.argv[1])
