cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 600 python -m pytest tests/test_ops_gpu.py -q -x -k "prefill" 2>&1 | tail -1
for c in "6272 2048" "4224 2048" "2176 2048" "8192 1280" "0 2048" "8192 384"; do
  echo "case $c"
  for v in "" 0 1; do echo -n "rowsplit=[$v] "; RS_ATTN_ROW_SPLIT=$v timeout 60 python scripts/attn_time.py $c 10; done
done
