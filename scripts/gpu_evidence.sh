#!/bin/bash
# Round-end evidence in one GPU call (run under gpurun):  bash scripts/gpu_evidence.sh TAG
# gpu_round.sh (GPU tests, smoke, bench, ncu launch list + full capture) plus the other nets' bench
# lines, the one-rank multi-GPU code paths, the reference arm, the replica emulation of the fused
# averaging and the per-phase cycles (instrumented build).  Everything lands in gpurun_out/TAG_*.
TAG=${1:-ev}
O=gpurun_out/${TAG}
bash scripts/gpu_round.sh $TAG
for a in tiny medium paper_small paper_large; do
  timeout 600 python bench.py --arch $a --no-cpu-baseline > ${O}_bench_$a.json 2> ${O}_bench_$a.err; echo "bench $a rc=$?"
done
for v in "fused strong" "async strong" "fused weak" "interval weak"; do
  set -- $v
  timeout 600 python bench.py --force-dist --avg $1 --scaling $2 --no-cpu-baseline > ${O}_dist_$1_$2.json 2> ${O}_dist_$1_$2.err; echo "dist $1 $2 rc=$?"
done
timeout 600 python bench.py --force-dist --comm chaos --scaling strong --no-cpu-baseline > ${O}_dist_fused_chaoscomm.json 2> ${O}_dist_chaoscomm.err; echo "chaoscomm rc=$?"
timeout 600 python bench.py --mode sync --no-cpu-baseline > ${O}_bench_sync.json 2> ${O}_bench_sync.err; echo "sync rc=$?"
timeout 600 python bench.py --impl reference > ${O}_bench_reference.json 2> ${O}_bench_reference.err; echo "reference rc=$?"
for R in 2 4 8; do timeout 900 python scripts/pavg_emulation_bench.py $R > ${O}_emu$R.jsonl 2>&1; echo "emu $R rc=$?"; done
python -c "from paper_1506_09067_b200 import build; build.build(timing=True)" > ${O}_build_timing.log 2>&1
timeout 600 python scripts/phase_times.py large 3 > ${O}_phase_times.txt 2>&1; echo "phases rc=$?"
