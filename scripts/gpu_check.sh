cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_ops_gpu.py -x -q -p no:cacheprovider -k "attention" > gpurun_out/attn_tests.log 2>&1; echo "exit $?" >> gpurun_out/attn_tests.log
tail -n 3 gpurun_out/attn_tests.log
timeout 300 python scripts/kernel_bench.py --attn > gpurun_out/kb_attn.json 2>&1
cat gpurun_out/kb_attn.json | cut -c1-1200
