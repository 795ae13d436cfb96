cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in "6272 2048" "4224 2048" "2176 2048" "8192 1280" "0 2048"; do
  echo "case $c"
  timeout 60 python scripts/attn_time.py $c 10
  for sp in 1 2 3 4 6 8 12 16; do echo -n "splits=$sp "; RS_ATTN_KV_SPLITS=$sp timeout 60 python scripts/attn_time.py $c 10; done
done
