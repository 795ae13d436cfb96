#!/bin/bash
# Round-2 probe: GEMM / window-attention op tests, steady-state GEMM timing per
# tile choice, ncu --set full of the ViT short-K GEMMs and the window attention.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/probe
O=gpurun_out/probe
timeout 600 python -m pytest tests/test_ops_gpu.py -q -p no:cacheprovider -k "gemm or window" > $O/ops.log 2>&1; echo "exit $?" >> $O/ops.log
timeout 900 python scripts/gemm_probe.py > $O/gemm_probe.log 2>&1; echo "exit $?" >> $O/gemm_probe.log
NCU="ncu --set full --clock-control none --import-source on"
timeout 300 $NCU -k regex:gemm_tcgen05 -s 3 -c 1 -o $O/ncu_vit_o python scripts/one_gemm.py 4096 1280 1280 1 0 > $O/ncu1.log 2>&1
timeout 300 $NCU -k regex:gemm_tcgen05 -s 3 -c 1 -o $O/ncu_vit_down python scripts/one_gemm.py 4096 1280 3424 1 0 > $O/ncu2.log 2>&1
timeout 300 $NCU -k regex:gemm_tcgen05 -s 3 -c 1 -o $O/ncu_llm_down python scripts/one_gemm.py 2048 3584 18944 1 0 > $O/ncu3.log 2>&1
timeout 400 $NCU -k regex:win_attn -s 60 -c 1 -o $O/ncu_win python scripts/one_vit_window.py 1 > $O/ncu4.log 2>&1
for r in vit_o vit_down llm_down win; do python scripts/ncu_summary.py $O/ncu_$r.ncu-rep $r > $O/ncu_$r.json 2>&1; done
tail -3 $O/ops.log; grep -c TFLOP $O/gemm_probe.log; cat $O/ncu_*.json | grep -E "label|gpu_time|tensor_pipe|dram"
