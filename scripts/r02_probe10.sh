#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/probe10; mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:fa_pp -s 2 -c 1 -o $O/ncu_attn python scripts/one_attn.py 6528 > $O/n1.log 2>&1
python scripts/ncu_summary.py $O/ncu_attn.ncu-rep attn_6528 > $O/ncu_attn.json 2>&1
cat $O/ncu_attn.json | grep -E "gpu_time|tensor_pipe|xu"
