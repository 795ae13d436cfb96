#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tcgen05_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_vit_o320 python scripts/one_gemm.py 4096 1280 1280 1 -320 > gpurun_out/ncu_vit_o.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_vit_o.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tcgen05_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_vit_o160 python scripts/one_gemm.py 4096 1280 1280 1 0 > gpurun_out/ncu_vit_o2.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_vit_o2.log
tail -1 gpurun_out/ncu_vit_o.log gpurun_out/ncu_vit_o2.log
