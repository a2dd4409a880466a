#!/bin/bash
# r2 verification session: the new multi-rank / planted-bug / scale tests, and the forms suite
# against the WDFS_CHECK bounds-check build (compute-sanitizer is closed on this pool).
mkdir -p gpurun_out
python paper_2507_14813_b200/build.py --variant check -DWDFS_CHECK > /dev/null 2>&1
( time timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_multirank.py tests/test_planted_bug.py ) > gpurun_out/pytest_r2d_a.log 2>&1
echo "multirank+planted rc=$?"; tail -4 gpurun_out/pytest_r2d_a.log
( time MAYURA_LIB_PATH=paper_2507_14813_b200/lib/libmayura_check.so timeout 1500 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_forms.py tests/test_gpu_invariants.py -k "warp or hybrid" ) > gpurun_out/pytest_r2d_check.log 2>&1
echo "check build rc=$?"; tail -4 gpurun_out/pytest_r2d_check.log
( time timeout 2400 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py -k "c4_sampled or c5_sampled" ) > gpurun_out/pytest_r2d_scale.log 2>&1
echo "scale rc=$?"; tail -5 gpurun_out/pytest_r2d_scale.log
