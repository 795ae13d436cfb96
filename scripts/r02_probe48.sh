# softmax turn-taking variants: timing + prefill attention op tests per variant
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/probe48
for v in "" "-DRS_PP_ORDER=1" "-DRS_PP_ORDER=2"; do
  touch paper_2509_24381_b200/csrc/attention_tc.cu
  make -s -C paper_2509_24381_b200/csrc -j8 RS_NVFLAGS_EXTRA="$v" > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  echo "variant [$v]"
  for c in "6272 2048" "8192 1280" "0 2048"; do timeout 120 python scripts/attn_time.py $c 10; done
  timeout 120 python scripts/attn_compare.py 8576 10 2>&1 | head -1
  timeout 300 python -m pytest tests/test_ops_gpu.py -q -x -k "attention" 2>&1 | tail -1
done
