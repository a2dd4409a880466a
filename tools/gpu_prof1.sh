#!/bin/bash
# One full ncu capture (with source counters) of the kernels of one co-mining pass.
# usage: bash tools/gpu_prof1.sh TAG CONFIG KERNEL_REGEX N_KERNELS [env...]
TAG=$1; C=$2; K=$3; N=$4; shift 4
mkdir -p gpurun_out
env "$@" timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $N -c $N \
  -o gpurun_out/prof_${TAG}_${C} -f python bench.py --config $C --profile --steps 1 --warmup 1 > gpurun_out/ncu_${TAG}_${C}.log 2>&1
echo "ncu $TAG $C rc=$?"
ncu -i gpurun_out/prof_${TAG}_${C}.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${TAG}_${C}.csv 2>/dev/null
ncu -i gpurun_out/prof_${TAG}_${C}.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_src_${TAG}_${C}.csv 2>/dev/null
[ $(stat -c %s gpurun_out/prof_${TAG}_${C}.ncu-rep) -gt 25000000 ] && rm -f gpurun_out/prof_${TAG}_${C}.ncu-rep
true
