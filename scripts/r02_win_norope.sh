#!/bin/bash
# Upper bound on moving the window RoPE out of the attention kernel: prep skipped (dev knob, wrong results).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
# the knob only exists in a dev build (rebuilds the library in place: rebuild without the flag afterwards)
make -C paper_2509_24381_b200/csrc -j8 -B RS_NVFLAGS_EXTRA=-DRS_WIN_DEV_BUILD > /dev/null 2>&1
for i in 1 2; do
  timeout 300 python scripts/one_vit_window.py 20 2>&1 | tail -1
  RS_WIN_SKIP_ROPE=1 timeout 300 python scripts/one_vit_window.py 20 2>&1 | tail -1
done > gpurun_out/win_norope.log
cat gpurun_out/win_norope.log
