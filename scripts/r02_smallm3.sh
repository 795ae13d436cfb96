#!/bin/bash
# Small-M GEMMs: split count sweep (RS_GEMM_FORCE_SPLITS, A/B knob) vs the planner.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for sp in 0 2 3 4 5 6 8; do
  echo "== splits $sp"; RS_GEMM_FORCE_SPLITS=$sp timeout 300 python scripts/gemm_probe.py --small-m 2>&1 | grep "bn    0 split0"
done
