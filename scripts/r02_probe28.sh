#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
touch paper_2509_24381_b200/csrc/attention_tc.cu
make -s -C paper_2509_24381_b200/csrc -j8 RS_NVFLAGS_EXTRA="-DRS_PP_TRACE_BUILD" > /dev/null 2>&1 || echo build failed
python scripts/attn_time.py 6272 2048 3 > /dev/null
RS_PP_TRACE=1 python scripts/attn_time.py 6272 2048 1 2>&1 | grep pp-trace | tail -12
