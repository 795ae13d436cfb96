#!/bin/bash
# ncu --set full of the fused QKV + M-RoPE + KV-append GEMM (cfg2 2048-row chunk) and the
# weight-streaming small-M GEMMs of the first / last prefill chunks.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/probe4; mkdir -p $O
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU --kernel-name-base demangled -k "regex:gemm_tcgen05_kernel<\(int\)256, \(int\)5" -s 10 -c 1 -o $O/ncu_qkv_rope python scripts/one_run.py 1 > $O/n1.log 2>&1
timeout 300 $NCU -k regex:gemm_tcgen05 -s 3 -c 1 -o $O/ncu_down_m128 python scripts/one_gemm.py 128 3584 18944 1 0 > $O/n2.log 2>&1
timeout 300 $NCU -k regex:gemm_tcgen05 -s 3 -c 1 -o $O/ncu_gateup_m256 python scripts/one_gemm.py 256 37888 3584 2 0 > $O/n3.log 2>&1
for r in qkv_rope down_m128 gateup_m256; do python scripts/ncu_summary.py $O/ncu_$r.ncu-rep $r > $O/ncu_$r.json 2>&1; done
cat $O/ncu_*.json | grep -E "label|gpu_time|tensor_pipe_active_pct_of_active\"|dram_r"
