#!/bin/bash
# quick session: parity tests + bench lines (kernel-only unless E2E=1) + optional ncu capture
# usage: [E2E=1] [CONFIGS="C1 C2"] bash tools/gpu_quick.sh [NCU_CONFIG]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_q.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu_q.log | grep -v "^$" | tail -12
EXTRA="--no-cpu-baseline --no-e2e"; [ -n "$E2E" ] && EXTRA="--no-cpu-baseline"
for C in ${CONFIGS:-C1 C2 C3}; do
timeout 400 python bench.py --config $C $EXTRA --steps 10 --warmup 3 > gpurun_out/q_${C}.json 2>gpurun_out/q_${C}.err
python -c "
import json; d=json.loads(open('gpurun_out/q_${C}.json').read().strip().splitlines()[-1]); r=d['roofline']; e=d.get('e2e') or {}
print('$C ms %.4f kern %.4f indep %.4f Balg/root %.1f frac %.4f e2e %s'%(d['ms_per_step'], r['kernel_ms'], d['independent_gpu']['ms_per_step'], r['bytes_alg_per_root'], r['frac'], e.get('s_per_step')), d['search_stats'])" || tail -5 gpurun_out/q_${C}.err
done
if [ -n "$1" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"expand|comine_lane|long" -s 3 -c 3 \
    -o gpurun_out/prof_q_$1 -f python bench.py --config $1 --profile --steps 1 --warmup 2 > /dev/null 2>&1
  echo "ncu rc=$?"
fi
