#!/bin/bash
# 256-row long-K GEMMs on 256 x 160 pair tiles with split tails: tests + probe.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ops_gpu.py tests/test_model_gpu.py tests/test_cfg2_parity_gpu.py tests/test_decode_gpu.py tests/test_tp_gpu.py -q -p no:cacheprovider > gpurun_out/sm4_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/sm4_tests.log
tail -3 gpurun_out/sm4_tests.log
for r in 1 2; do timeout 300 python scripts/gemm_probe.py --small-m 2>&1 | grep "bn    0 split0" | grep down; done
