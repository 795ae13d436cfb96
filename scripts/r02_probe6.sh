#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/probe6; mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU --kernel-name-base demangled -k "regex:gemm_tcgen05_kernel<\(int\)256, \(int\)5" -s 10 -c 1 -o $O/ncu_qkv_rope python scripts/one_run.py 1 > $O/n1.log 2>&1
python scripts/ncu_summary.py $O/ncu_qkv_rope.ncu-rep qkv_rope > $O/ncu_qkv_rope.json 2>&1
timeout 900 python scripts/gemm_probe.py --small-m > $O/gemm_small.log 2>&1
cat $O/ncu_qkv_rope.json | grep -E "gpu_time|tensor_pipe_active_pct_of_active\"|dram_r"; grep -c TFLOP $O/gemm_small.log
