#!/bin/bash
# Round-2 GPU session: parity suite + smoke, the default (C4) bench line, C2 bench, the C4 launch
# list and full ncu captures of one C4 co-mining pass (default cold-cache replay and
# --cache-control none), exported to raw CSV on the box (reports exceed the copy-back limit).
# usage (repo root, under gpurun): bash tools/gpu_r2.sh TAG [skip-tests]
TAG=${1:-r2a}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi_${TAG}.txt 2>&1
lscpu > gpurun_out/lscpu_${TAG}.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_${TAG}.log 2>&1
  echo "pytest gpu rc=$?"; tail -3 gpurun_out/pytest_gpu_${TAG}.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke rc=$?
fi
timeout 900 python bench.py > gpurun_out/bench_C4_${TAG}.json 2> gpurun_out/bench_C4_${TAG}.err
echo "bench C4 rc=$?"; tail -c 300 gpurun_out/bench_C4_${TAG}.json
timeout 600 python bench.py --config C2 > gpurun_out/bench_C2_${TAG}.json 2> gpurun_out/bench_C2_${TAG}.err
echo "bench C2 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_C4_${TAG}.csv python bench.py --profile --steps 3 --warmup 3 > /dev/null 2>&1
echo "ncu launches rc=$?"
for CC in all none; do
  timeout 1200 ncu --set full --clock-control none --cache-control $CC --import-source on \
    -k regex:"window_end|wdfs_kernel" -s 2 -c 2 \
    -o gpurun_out/prof_C4_${CC}_${TAG} -f python bench.py --profile --steps 1 --warmup 1 > gpurun_out/ncu_${CC}.log 2>&1
  echo "ncu full C4 cache=$CC rc=$?"
  SFX=$([ "$CC" == "none" ] && echo "_warm" || echo "")
  ncu -i gpurun_out/prof_C4_${CC}_${TAG}.ncu-rep --page raw --csv > gpurun_out/prof_C4_${TAG}${SFX}_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_C4_${CC}_${TAG}.ncu-rep --page source --csv --print-source sass -k regex:wdfs > gpurun_out/ncu_src_C4_${CC}_${TAG}.csv 2>/dev/null
  [ -f gpurun_out/prof_C4_${CC}_${TAG}.ncu-rep ] && [ $(stat -c %s gpurun_out/prof_C4_${CC}_${TAG}.ncu-rep) -gt 25000000 ] && rm -f gpurun_out/prof_C4_${CC}_${TAG}.ncu-rep
done
du -sh gpurun_out
