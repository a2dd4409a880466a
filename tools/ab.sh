for L in base b3 b4; do
 if [ $L = base ]; then unset MAYURA_LIB_PATH; else export MAYURA_LIB_PATH=$PWD/abtest/lib_$L.so; fi
 for C in C2 C3; do
  timeout 300 python bench.py --config $C --no-cpu-baseline --no-e2e --no-indep --steps 10 --warmup 3 > gpurun_out/ab_${L}_${C}.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_${L}_${C}.json').read().strip().splitlines()[-1]); print('$L $C', round(d['ms_per_step'],4), d['parity_vs_oracle'] if 'parity_vs_oracle' in d else '')"
 done
done
