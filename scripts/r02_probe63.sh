cd "${GRAFT_REPO_ROOT:-/root/repo}"
touch paper_2509_24381_b200/csrc/attention_tc.cu
make -s -C paper_2509_24381_b200/csrc -j8 RS_NVFLAGS_EXTRA="-DRS_PP_TRACE_BUILD" > /dev/null 2>&1
for c in "6272 2048" "2176 2048" "0 2048"; do
  for sp in "" 1 2; do echo "case $c splits=$sp"; RS_ATTN_KV_SPLITS=$sp RS_PP_TRACE=1 timeout 60 python scripts/attn_time.py $c 1 2>&1 | grep -E "pp-cta|TFLOP" | tail -2; done
done
