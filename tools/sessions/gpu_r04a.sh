mkdir -p gpurun_out
for C in C1 C2 C3; do
  timeout 600 python bench.py --config $C --no-cpu-baseline > gpurun_out/b4_$C.json 2> gpurun_out/b4_$C.err
  python -c "
import json; d=json.loads(open('gpurun_out/b4_$C.json').read().strip().splitlines()[-1]); print('$C', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['s_per_step']*1e3,3), 'indep', round(d['independent_gpu']['ms_per_step'],3), 'enum', json.dumps(d['enumeration']))" || tail -5 gpurun_out/b4_$C.err
done
for C in C1 C2 C3; do timeout 600 python tools/delta_sweep.py --config $C > gpurun_out/ds_$C.log 2>&1; tail -9 gpurun_out/ds_$C.log | cut -c1-260; done
