cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ops_gpu.py -x -q -p no:cacheprovider -k "pair" > gpurun_out/pair_tests.log 2>&1; echo "exit $?" >> gpurun_out/pair_tests.log
tail -5 gpurun_out/pair_tests.log
timeout 600 python scripts/gemm_sweep.py > gpurun_out/gemm_sweep.log 2>&1; echo "exit $?" >> gpurun_out/gemm_sweep.log
grep -v '^\[' gpurun_out/gemm_sweep.log | tail -200
