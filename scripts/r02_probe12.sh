#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/probe12; mkdir -p $O
RS_ATTN_EXP_BF16=1 timeout 600 python -m pytest tests/test_ops_gpu.py -q -p no:cacheprovider -k "attention" > $O/ops_bf16.log 2>&1; echo "exit $?" >> $O/ops_bf16.log
for cfg in "0 0" "1 0" "1 0x8888" "1 0x4444" "1 0x2222" "1 0xAAAA"; do set -- $cfg
  echo "== exp_bf16=$1 poly_mask=$2" >> $O/attn.log
  RS_ATTN_EXP_BF16=$1 RS_ATTN_POLY_MASK=$2 timeout 120 python scripts/attn_compare.py 8576 20 2>&1 | grep ours >> $O/attn.log
  RS_ATTN_EXP_BF16=$1 RS_ATTN_POLY_MASK=$2 timeout 120 python scripts/attn_time.py 2>&1 | tail -4 >> $O/attn.log
done
tail -3 $O/ops_bf16.log; cat $O/attn.log
