#!/bin/bash
# A/B of library variants on one GPU (run under gpurun):  bash scripts/ab_run.sh TAG lib1 lib2 ...
# Each lib: samples/s of a 60,000-image hogwild epoch (quick_epoch, best of 3); *_t.so timing
# builds also print the per-phase cycle budget (phase_times).  Output: gpurun_out/TAG_ab.txt
TAG=$1; shift
ARCH=${ARCH:-large}
mkdir -p gpurun_out
O=gpurun_out/${TAG}_ab.txt
: > $O
for rep in 1 2; do
for L in "$@"; do
  P=paper_1506_09067_b200/$L
  if [[ $L == *_t.so ]]; then
    [ $rep = 1 ] && { echo "== $L phases" >> $O; CHAOS_LIB=$P timeout 300 python scripts/phase_times.py $ARCH 3 >> $O 2>&1; }
  else
    echo "== $L rep $rep" >> $O
    CHAOS_LIB=$P timeout 300 python scripts/quick_epoch.py $ARCH >> $O 2>&1
  fi
done
done
cat $O
