#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_ops_gpu.py -q -x -p no:cacheprovider -k "attention" 2>&1 | tail -1
ATTN_CASES="6272 2048,8192 1280,2048 2048,0 2048" bash scripts/attn_variants.sh "-DRS_PP_SUM_AFTER_P=0" "-DRS_PP_POLY_EVERY=0" "-DRS_PP_POLY_EVERY=8"
