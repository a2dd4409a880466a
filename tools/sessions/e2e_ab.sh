for L in "" "MAYURA_LIB_PATH=paper_2507_14813_b200/lib/libmayura_oldsucc.so" "" "MAYURA_LIB_PATH=paper_2507_14813_b200/lib/libmayura_oldsucc.so"; do
  for C in C2 C4; do
    env $L python bench.py --config $C --no-enum --no-cpu-baseline --no-indep --steps 5 --e2e-steps 7 > gpurun_out/e2eab.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/e2eab.json').read()); print('$C', '${L:-new}'[-20:], 'e2e ms %.3f' % (d['e2e']['s_per_step']*1e3))"
  done
done
