#!/bin/bash
# C4 bench line with the current kernels (+ the launch list of one step)
TAG=${1:-r08}
mkdir -p gpurun_out
timeout 1500 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/bench_C4_${TAG}.json 2> gpurun_out/bench_C4_${TAG}.err
echo "bench C4 rc=$?"; tail -c 300 gpurun_out/bench_C4_${TAG}.json
