#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for shape in "2048 3584 18944 1" "4096 1280 1280 1"; do
 for bn in 0 -224 -256 256; do
  for dbg in 0 1 2; do
   echo -n "shape $shape bn $bn dbg $dbg: "; RS_GEMM_SK_DEBUG=$dbg ONE_GEMM_TIME=1 python scripts/one_gemm.py $shape $bn 2>&1 | tail -1
  done
  echo -n "shape $shape bn $bn nosk: "; RS_GEMM_STREAMK_ALL=0 ONE_GEMM_TIME=1 python scripts/one_gemm.py $shape $bn 2>&1 | tail -1
 done
done
