#!/bin/bash
# quick A/B session: parity tests + kernel-only bench lines for both kernels (+ optional ncu)
# usage: bash tools/gpu_quick.sh [NCU_CONFIG]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_q.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu_q.log | grep -v "^$" | tail -12
for K in ${KERNELS:-lane warp}; do for C in ${CONFIGS:-C1 C2 C3}; do
MAYURA_KERNEL=$K timeout 300 python bench.py --config $C --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/q_${K}_${C}.json 2>gpurun_out/q_${K}_${C}.err
python -c "
import json; d=json.loads(open('gpurun_out/q_${K}_${C}.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$K $C ms %.4f kern %.4f indep %.4f Balg/root %.1f frac %.4f'%(d['ms_per_step'], r['kernel_ms'], d['independent_gpu']['ms_per_step'], r['bytes_alg_per_root'], r['frac']), d['search_stats'])" || tail -5 gpurun_out/q_${K}_${C}.err
done; done
if [ -n "$1" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:comine -s 3 -c 1 \
    -o gpurun_out/prof_q_$1 -f python bench.py --config $1 --profile --steps 1 --warmup 4 > /dev/null 2>&1
  echo "ncu rc=$?"
fi
