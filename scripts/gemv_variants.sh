# Dev tool: gemv unroll variants (rebuilds on the GPU box): bash scripts/gemv_variants.sh 2 4 8
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for u in "$@"; do
  touch paper_2509_24381_b200/csrc/gemv.cu
  make -s -C paper_2509_24381_b200/csrc -j8 RS_NVFLAGS_EXTRA="-DRS_GEMV_UNROLL=$u" > /dev/null 2>&1 || { echo "build failed $u"; continue; }
  echo "unroll $u"; timeout 300 python scripts/gemv_time.py
done
