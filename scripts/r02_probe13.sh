#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/probe13; mkdir -p $O
timeout 900 python -m pytest tests/test_ops_gpu.py -q -x -p no:cacheprovider -k "gemm" > $O/ops.log 2>&1; echo "exit $?" >> $O/ops.log
tail -3 $O/ops.log
timeout 900 python scripts/gemm_probe.py > $O/probe_sk.log 2>&1
RS_GEMM_STREAMK_ALL=0 timeout 900 python scripts/gemm_probe.py > $O/probe_nosk.log 2>&1
timeout 1200 python -m pytest tests/test_model_gpu.py tests/test_cfg2_parity_gpu.py -q -x -p no:cacheprovider > $O/model.log 2>&1; echo "exit $?" >> $O/model.log
tail -3 $O/model.log
for m in sk nosk; do echo "== $m"; grep "bn    0 split0" $O/probe_$m.log; done
