#!/bin/bash
# end-of-round evidence: the whole -m gpu suite + smoke, bench lines C4 (default), C3, C2, C1, the
# C4 launch list + full ncu captures (cold / warm), C5 on one GPU and rank by rank
TAG=${1:-r2f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=pci.bus_id,name --format=csv,noheader > gpurun_out/gpu_${TAG}.txt
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ) > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest gpu rc=$?"; tail -6 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
bash tools/gpu_r2.sh $TAG skip-tests
for C in C3 C1; do
  timeout 600 python bench.py --config $C > gpurun_out/bench_${C}_${TAG}.json 2> gpurun_out/bench_${C}_${TAG}.err; echo "bench $C rc=$?"
done
timeout 2400 python tools/run_c5.py gpurun_out/c5_${TAG}.json > gpurun_out/c5_${TAG}.log 2>&1; echo "c5 rc=$?"
