#!/bin/bash
# GEMM/model GPU tests, bench, and an ncu capture of the ViT down projection on 256 x 320 pair tiles.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
tail -1 gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tcgen05_kernel -c 1 \
  -o gpurun_out/ncu_vit_down320 python scripts/one_gemm.py 4096 1280 3424 1 0 > gpurun_out/ncu_vit_down.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_vit_down.log
tail -2 gpurun_out/ncu_vit_down.log
