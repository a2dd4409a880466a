# A/B of library builds under abtest/ (MAYURA_LIB_PATH): usage bash tools/ab.sh "base pend ..." "C2 C3" [reps]
LIBS=${1:-base}; CONFS=${2:-"C2 C3"}; REPS=${3:-1}
mkdir -p gpurun_out
for r in $(seq 1 $REPS); do
for L in $LIBS; do
 export MAYURA_LIB_PATH=$PWD/abtest/lib_$L.so
 for C in $CONFS; do
  timeout 300 python bench.py --config $C --no-cpu-baseline --no-e2e --no-indep --no-enum --steps 10 --warmup 3 > gpurun_out/ab_${L}_${C}.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_${L}_${C}.json').read().strip().splitlines()[-1]); print('$L $C', round(d['ms_per_step'],4), d['search_stats']['roots'])" || tail -3 gpurun_out/ab_${L}_${C}.json
 done
done
done
