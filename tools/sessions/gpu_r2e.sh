#!/bin/bash
# end-of-session evidence: bench lines C4 (default), C3, C2 + the C4 ncu captures, then C5
bash tools/gpu_r2.sh $1 skip-tests
timeout 600 python bench.py --config C3 > gpurun_out/bench_C3_$1.json 2> gpurun_out/bench_C3_$1.err; echo "bench C3 rc=$?"
timeout 2400 python tools/run_c5.py gpurun_out/c5_$1.json > gpurun_out/c5_$1.log 2>&1; echo "c5 rc=$?"; tail -c 600 gpurun_out/c5_$1.json
