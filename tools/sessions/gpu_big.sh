# C4 bench line + C5 (8-rank emulation) with the current kernels
mkdir -p gpurun_out
timeout 1500 python bench.py --config C4 --steps 5 --warmup 3 > gpurun_out/bench_C4_r05.json 2> gpurun_out/bench_C4_r05.err
echo "bench C4 rc=$?"; tail -c 300 gpurun_out/bench_C4_r05.json
timeout 2400 python tools/run_c5.py gpurun_out/c5_r05.json > gpurun_out/c5_r05.log 2>&1
echo "c5 rc=$?"; tail -5 gpurun_out/c5_r05.log
