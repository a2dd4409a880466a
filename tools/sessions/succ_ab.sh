MAYURA_LIB_PATH=paper_2507_14813_b200/lib/libmayura_succ2.so python -m pytest -x -q tests/test_gpu_parity.py -k "graph_build or partition" 2>&1 | tail -1
for L in "" "MAYURA_LIB_PATH=paper_2507_14813_b200/lib/libmayura_succ2.so" "" "MAYURA_LIB_PATH=paper_2507_14813_b200/lib/libmayura_succ2.so"; do
  env $L python bench.py --config C4 --no-enum --no-cpu-baseline --no-indep --steps 5 --e2e-steps 7 > gpurun_out/e2eab.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/e2eab.json').read()); print('${L:-old}'[-22:], 'e2e ms %.3f' % (d['e2e']['s_per_step']*1e3))"
done
