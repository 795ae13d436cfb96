cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ops_gpu.py -x -q -p no:cacheprovider > gpurun_out/ops_tests.log 2>&1; echo "exit $?" >> gpurun_out/ops_tests.log
tail -n 3 gpurun_out/ops_tests.log
timeout 600 python scripts/gemm_sweep.py --quick > gpurun_out/gemm_sweep.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
tail -n 2 gpurun_out/bench.err
