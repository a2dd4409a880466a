#!/bin/bash
# hybrid-levels sweep (kernel-only bench lines)
for L in ${LEVELS:-0 1 2}; do for C in ${CONFIGS:-C1 C2 C3}; do
MAYURA_HYBRID_LEVELS=$L timeout 300 python bench.py --config $C --no-cpu-baseline --no-e2e --no-indep --steps 10 --warmup 3 > gpurun_out/h_${L}_${C}.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/h_${L}_${C}.json').read().strip().splitlines()[-1]); r=d['roofline']
print('L=$L $C ms %.4f kern %.4f'%(d['ms_per_step'], r['kernel_ms']), 'offl', d['search_stats']['offloads'], 'ctx', d['search_stats']['contexts'])"
done; done
for C in ${CONFIGS:-C1 C2 C3}; do
MAYURA_KERNEL=bfs timeout 300 python bench.py --config $C --no-cpu-baseline --no-e2e --no-indep --steps 10 --warmup 3 > gpurun_out/hb_${C}.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/hb_${C}.json').read().strip().splitlines()[-1]); r=d['roofline']
print('bfs $C ms %.4f kern %.4f'%(d['ms_per_step'], r['kernel_ms']), 'offl', d['search_stats']['offloads'], 'ctx', d['search_stats']['contexts'])"
done
