timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do for P in 0 1; do for C in C1 C2 C3; do
  MAYURA_PDL=$P timeout 300 python bench.py --config $C --no-cpu-baseline --no-e2e --no-indep --no-enum --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$P $C', round(d['ms_per_step'],4))"
done; done; done
