#!/bin/bash
# Wide pair tiles (256 x 320 / 448 / 512): op tests, then steady-state timing vs the current tiles.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_ops_gpu.py -q -p no:cacheprovider -k "cta_pair or streamk" > gpurun_out/wide_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/wide_tests.log
tail -3 gpurun_out/wide_tests.log
timeout 600 python scripts/gemm_probe.py --wide > gpurun_out/wide_probe.log 2>&1; echo "probe exit $?" >> gpurun_out/wide_probe.log
grep -v '^\[{' gpurun_out/wide_probe.log | tail -40
