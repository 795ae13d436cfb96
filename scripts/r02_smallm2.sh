#!/bin/bash
# Small-M split-K threshold (32 k-blocks for <= 256-row launches): op tests, model tests, probe A/B.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ops_gpu.py tests/test_model_gpu.py tests/test_cfg2_parity_gpu.py tests/test_decode_gpu.py -q -p no:cacheprovider > gpurun_out/sm_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/sm_tests.log
tail -3 gpurun_out/sm_tests.log
for r in 1 2; do
  echo "== default"; timeout 300 python scripts/gemm_probe.py --small-m 2>&1 | grep "bn    0 split0" | grep -E "qkv|o_m"
  echo "== RS_GEMM_SMALL_MIN_KB=128"; RS_GEMM_SMALL_MIN_KB=128 timeout 300 python scripts/gemm_probe.py --small-m 2>&1 | grep "bn    0 split0" | grep -E "qkv|o_m"
done
