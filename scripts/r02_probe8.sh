#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/probe8; mkdir -p $O
timeout 900 python -m pytest tests/test_tp_group_gpu.py tests/test_tp_gpu.py -q -x -p no:cacheprovider > $O/tp.log 2>&1; echo "exit $?" >> $O/tp.log
tail -30 $O/tp.log
