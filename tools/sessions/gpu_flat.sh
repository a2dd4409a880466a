mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_forms.py -x -q -p no:cacheprovider 2>&1 | tail -15
for K in hybrid flat; do
 for C in C1 C2 C3; do
  MAYURA_KERNEL=$K timeout 300 python bench.py --config $C --no-cpu-baseline --no-e2e --no-indep --no-enum --steps 10 --warmup 3 > gpurun_out/fl_${K}_${C}.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/fl_${K}_${C}.json').read().strip().splitlines()[-1]); print('$K $C', round(d['ms_per_step'],4), d['counts'])" || tail -3 gpurun_out/fl_${K}_${C}.json
 done
done
MAYURA_KERNEL=flat timeout 600 ncu --set full --clock-control none --import-source on -k regex:"flat" -s 4 -c 4 \
    -o gpurun_out/prof_flat_C2 -f python bench.py --config C2 --profile --steps 1 --warmup 2 > /dev/null 2>&1
echo ncu rc=$?
MAYURA_KERNEL=flat timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_flat_C2.csv python bench.py --config C2 --profile --steps 2 --warmup 3 >/dev/null 2>&1
echo ncu2 rc=$?
