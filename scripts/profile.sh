#!/bin/bash
# Usage (on the GPU box): scripts/profile.sh TAG [arch]
# plain run first (must exit 0), then one ncu --set full capture of the hogwild worker kernel.
TAG=${1:-prof}; ARCH=${2:-large}
case $ARCH in large) KN="LargeNetELi4ELi[0-9]+ELi0E";; medium) KN="MediumNetELi4ELi[0-9]+ELi0E";; tiny) KN="TinyNetELi1ELi[0-9]+ELi0E";; esac
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --arch $ARCH"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:$KN -s 1 -c 1 \
    -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
