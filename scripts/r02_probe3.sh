#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/probe3; mkdir -p $O
timeout 900 python -m pytest tests/test_pd_transfer_gpu.py tests/test_decode_gpu.py -q -p no:cacheprovider > $O/pd.log 2>&1; echo "exit $?" >> $O/pd.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 100000 python scripts/one_gemm.py 512 1280 1280 1 0 > $O/sync_gemm_res.log 2>&1; echo "exit $?" >> $O/sync_gemm_res.log
timeout 600 compute-sanitizer --tool synccheck --print-limit 100000 python scripts/one_gemm.py 512 1280 1280 0 0 > $O/sync_gemm_store.log 2>&1; echo "exit $?" >> $O/sync_gemm_store.log
for f in sync_gemm_res sync_gemm_store; do echo "== $f"; grep "error detected" $O/$f.log | sort | uniq -c; grep -A4 "error detected" $O/$f.log | grep "Device Frame" | sed 's/+0x[0-9a-f]*//' | sort | uniq -c | sort -rn | head -8; tail -2 $O/$f.log; done > $O/sync_summary.txt
tail -5 $O/pd.log; cat $O/sync_summary.txt
