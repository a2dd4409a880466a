#!/bin/bash
# gpu_round.sh, then shrink gpurun_out below gpurun's 64 MiB copy-back limit: the full ncu
# captures are exported to raw CSV on the box and only reports under 20 MiB are kept.
TAG=${1:-r08}
bash tools/gpu_round.sh "$@"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo smoke rc=$?
for R in gpurun_out/prof_*_${TAG}.ncu-rep; do
  ncu -i "$R" --page raw --csv > "${R%.ncu-rep}_raw.csv" 2>/dev/null
  [ $(stat -c %s "$R") -gt 20000000 ] && rm -f "$R"
done
du -sh gpurun_out; ls -la gpurun_out
