#!/bin/bash
# One GPU call (run under gpurun): GPU tests, the bench line, the ncu launch list and one
# `ncu --set full` capture of the hogwild worker kernel.  Everything lands in gpurun_out/TAG_*.
#   gpurun --timeout 2400 -- 'bash scripts/gpu_round.sh r1a'
# Steps can be skipped with SKIP_TESTS=1 / SKIP_NCU=1.
TAG=${1:-run}
ARCH=${ARCH:-large}
mkdir -p gpurun_out
O=gpurun_out/${TAG}
nvidia-smi > ${O}_smi.txt 2>&1
lscpu > ${O}_lscpu.txt 2>&1
python -c "from paper_1506_09067_b200 import build; build.build(); import oracle; oracle.build()" > ${O}_build.log 2>&1 || { echo BUILD FAILED; tail -30 ${O}_build.log; exit 1; }
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rsxf --timeout 600 > ${O}_pytest.log 2>&1
  echo "pytest rc=$?"; tail -15 ${O}_pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 ${O}_smoke.log
fi
timeout 600 python bench.py --arch $ARCH > ${O}_bench.json 2> ${O}_bench.err; echo "bench rc=$?"; cat ${O}_bench.json; tail -3 ${O}_bench.err
if [ -z "$SKIP_NCU" ]; then
  CMD="python bench.py --arch $ARCH --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
  case $ARCH in paper_large) KN="PaperLargeNetELi1ELi[0-9]+ELi0E";; large) KN="LargeNetELi4ELi[0-9]+ELi0E";; medium) KN="MediumNetELi4ELi[0-9]+ELi0E";; tiny) KN="TinyNetELi1ELi[0-9]+ELi0E";; esac
  timeout 600 $CMD > ${O}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_launches.csv $CMD > ${O}_ncu_launch.log 2>&1
  echo "launch-list rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:$KN -s 3 -c 1 \
      -o ${O}_full $CMD > ${O}_ncu_full.log 2>&1
  echo "ncu-full rc=$?"; tail -3 ${O}_ncu_full.log
fi
