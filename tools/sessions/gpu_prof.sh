#!/bin/bash
# ncu launch list + full captures of the top kernels for one config
# usage: bash tools/gpu_prof.sh CONFIG TAG [regex] [skip] [count]
C=${1:-C2}; TAG=${2:-p}; RX=${3:-expand_kernel}; SK=${4:-0}; CN=${5:-4}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${C}_${TAG}.csv python bench.py --config $C --profile --steps 2 --warmup 3 > /dev/null 2>&1
echo "ncu launches rc=$?"
python tools/summarize_profiles.py ${TAG} $C > /dev/null 2>&1; grep "|" profiles/${TAG}_${C}.md | head -20
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -s $SK -c $CN \
    -o gpurun_out/prof_${C}_${TAG} -f python bench.py --config $C --profile --steps 1 --warmup 3 > gpurun_out/ncu_full_${C}_${TAG}.log 2>&1
echo "ncu full rc=$?"
