#!/bin/bash
# One GPU session: parity tests, bench lines, ncu launch list + one full capture of ONE co-mining
# pass (all its kernels) per config.
# usage (from the repo root, under gpurun): bash tools/gpu_round.sh TAG "C1:4 C2:6 C3:3"
#   C:N = config and the number of co-mining kernels in one pass (flat: 2 per MG-Tree level;
#   hybrid: expand + long + lane = 3)
TAG=${1:-r04}
SPECS=${2:-"C1:4 C2:6 C3:3"}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_${TAG}.txt 2>&1
lscpu > gpurun_out/lscpu_${TAG}.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1
echo "pytest gpu rc=$?"
tail -3 gpurun_out/pytest_gpu_${TAG}.log
for S in $SPECS; do
  C=${S%%:*}
  timeout 900 python bench.py --config $C > gpurun_out/bench_${C}_${TAG}.json 2> gpurun_out/bench_${C}_${TAG}.err
  echo "bench $C rc=$?"; tail -c 400 gpurun_out/bench_${C}_${TAG}.json
done
for S in $SPECS; do
  C=${S%%:*}; N=${S##*:}
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${C}_${TAG}.csv python bench.py --config $C --profile --steps 3 --warmup 3 \
    > /dev/null 2>&1
  echo "ncu launches $C rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"flat_win|flat_entry|expand_kernel|long_kernel|comine_lane" -s 0 -c $N \
    -o gpurun_out/prof_${C}_${TAG} -f python bench.py --config $C --profile --steps 1 --warmup 3 > /dev/null 2>&1
  echo "ncu full $C rc=$?"
done
