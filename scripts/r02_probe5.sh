#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/probe5; mkdir -p $O
timeout 600 compute-sanitizer --tool synccheck --print-limit 100000 python scripts/one_gemm.py 512 1280 1280 1 0 > $O/sync_gemm_res.log 2>&1; echo "exit $?" >> $O/sync_gemm_res.log
tail -3 $O/sync_gemm_res.log
timeout 600 python -m pytest tests/test_ops_gpu.py -q -p no:cacheprovider -k "gemm" > $O/ops.log 2>&1; echo "exit $?" >> $O/ops.log; tail -2 $O/ops.log
bash scripts/r02_probe4.sh
