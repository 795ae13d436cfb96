#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
touch paper_2509_24381_b200/csrc/attention_tc.cu
make -s -C paper_2509_24381_b200/csrc -j8 RS_NVFLAGS_EXTRA="-DRS_PP_POLY_DEG=2 -DRS_PP_POLY_EVERY=2" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_ops_gpu.py -q -x -p no:cacheprovider -k "attention" 2>&1 | tail -1
ATTN_CASES="6272 2048,8192 1280,2048 2048" bash scripts/attn_variants.sh "-DRS_PP_POLY_DEG=2" "-DRS_PP_POLY_DEG=2 -DRS_PP_POLY_EVERY=3" "-DRS_PP_POLY_DEG=2 -DRS_PP_POLY_EVERY=2"
