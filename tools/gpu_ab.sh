#!/bin/bash
# Quick A/B on one config: parity subset + kernel-form timings (bench --profile lines).
# usage: bash tools/gpu_ab.sh TAG CONFIG "form1 form2 ..." [pytest-args]
TAG=${1:-ab}; C=${2:-C4}; FORMS=${3:-"hybrid"}; shift 3
mkdir -p gpurun_out
if [ -n "$1" ]; then
  timeout 1800 python -m pytest -x -q -p no:cacheprovider "$@" > gpurun_out/pytest_${TAG}.log 2>&1
  echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${TAG}.log
fi
for F in $FORMS; do
  K=${F%%+*}; X=${F#*+}; [ "$X" == "$F" ] && X=""
  N=$(echo "$F" | tr '/=+' '___')
  env MAYURA_KERNEL=$K $X timeout 900 python bench.py --config $C --profile --steps 10 --warmup 3 \
    > gpurun_out/ab_${TAG}_${C}_${N}.json 2> gpurun_out/ab_${TAG}_${C}_${N}.err
  echo "$C $F rc=$? $(python -c "import json,sys; d=json.load(open('gpurun_out/ab_${TAG}_${C}_${N}.json')); print('ms %.3f kern %.3f form %s counts %s' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['kernel_form'], sum(d['counts'].values())))" 2>&1 | tail -1)"
done
