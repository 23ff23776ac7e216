#!/bin/bash
# usage: tools/prof_kernel.sh NAME KERNEL_REGEX CMD...   (run on the GPU box via gpurun)
# plain run first (must exit 0), then one ncu --set full capture of the first matching launch
name=$1; kre=$2; shift 2
"$@" > gpurun_out/${name}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$kre" -c 1 -o gpurun_out/${name} "$@" > gpurun_out/${name}_ncu.log 2>&1
