#!/bin/bash
# Small-M (first / last prefill chunk) GEMMs: heuristic tiles with the default split-K threshold vs split-K from 32 k-blocks.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for kb in 128 32 16; do
  echo "== RS_GEMM_SMALL_MIN_KB=$kb"
  RS_GEMM_SMALL_MIN_KB=$kb timeout 300 python scripts/gemm_probe.py --small-m 2>&1 | grep -v '^\[{' | grep "bn    0 split0"
done > gpurun_out/smallm.log 2>&1
cat gpurun_out/smallm.log
