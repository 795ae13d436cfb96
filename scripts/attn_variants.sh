# Dev tool: rebuilds the library with each RS_NVFLAGS_EXTRA variant (on the
# GPU box) and times the prefill attention; usage: bash scripts/attn_variants.sh "-DA=1" "-DB=2" ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for v in "" "$@"; do
  touch paper_2509_24381_b200/csrc/attention_tc.cu
  make -s -C paper_2509_24381_b200/csrc -j8 RS_NVFLAGS_EXTRA="$v" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "variant [$v]"
  IFS=, read -ra CASES <<< "${ATTN_CASES:-6272 2048,8192 1280,0 2048}"
  for c in "${CASES[@]}"; do timeout 120 python scripts/attn_time.py $c 10; done
done
