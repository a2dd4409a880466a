for K in "warp" "hybrid" "hybrid MAYURA_HEAVY_MIN=0" "hybrid MAYURA_WDFS_SMALL=1" "warp MAYURA_WDFS_SMALL=1"; do
  set -- $K
  env MAYURA_KERNEL=$1 $2 timeout 300 python tools/dbg_c2_rev.py 2>&1 | tail -3
done
MAYURA_LIB_PATH=paper_2507_14813_b200/lib/libmayura_check.so MAYURA_KERNEL=hybrid timeout 300 python tools/dbg_c2_rev.py 2>&1 | tail -12
MAYURA_LIB_PATH=paper_2507_14813_b200/lib/libmayura_check.so MAYURA_KERNEL=warp timeout 300 python tools/dbg_c2_rev.py 2>&1 | tail -12
