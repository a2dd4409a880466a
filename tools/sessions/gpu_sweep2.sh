# knob sweep: heavy-root threshold x breadth-first levels, C2 and C3 (kernel-only bench lines)
mkdir -p gpurun_out
for C in C2 C3; do
 for H in 0 4 8 16 32; do
  for L in 1 2; do
   MAYURA_HEAVY_MIN=$H MAYURA_HYBRID_LEVELS=$L timeout 300 python bench.py --config $C --no-cpu-baseline --no-e2e --no-indep --no-enum --steps 10 --warmup 3 > gpurun_out/sw_${C}_${H}_${L}.json 2>&1
   python -c "import json; d=json.loads(open('gpurun_out/sw_${C}_${H}_${L}.json').read().strip().splitlines()[-1]); print('$C H=$H L=$L', round(d['ms_per_step'],4))" || tail -3 gpurun_out/sw_${C}_${H}_${L}.json
  done
 done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"expand|comine_lane|long" -s 3 -c 3 \
    -o gpurun_out/prof_C2_r04 -f python bench.py --config C2 --profile --steps 1 --warmup 2 > /dev/null 2>&1
echo "ncu rc=$?"
