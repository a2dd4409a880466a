#!/bin/bash
# env-var sweep of kernel-only bench lines: VAR="MAYURA_HEAVY_MIN" VALUES="0 2 4" CONFIGS="C1 C2"
for v in $VALUES; do for C in ${CONFIGS:-C1 C2 C3}; do
env $VAR=$v timeout 300 python bench.py --config $C --no-cpu-baseline --no-e2e --no-indep --steps 10 --warmup 3 > gpurun_out/sw_${v}_${C}.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/sw_${v}_${C}.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$VAR=$v $C ms %.4f kern %.4f'%(d['ms_per_step'], r['kernel_ms']), 'offl', d['search_stats']['offloads'], 'ctx', d['search_stats']['contexts'])"
done; done
