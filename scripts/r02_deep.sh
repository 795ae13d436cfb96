#!/bin/bash
# Residual epilogue with every chunk prefetched: GEMM op tests, then the --wide probe (compare profiles/r02_gemm_wide.txt).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ops_gpu.py -q -p no:cacheprovider -k "gemm" > gpurun_out/deep_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/deep_tests.log
tail -3 gpurun_out/deep_tests.log
timeout 600 python scripts/gemm_probe.py --wide > gpurun_out/deep_probe.log 2>&1; echo "probe exit $?" >> gpurun_out/deep_probe.log
grep -v '^\[{' gpurun_out/deep_probe.log | tail -40
