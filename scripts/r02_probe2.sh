#!/bin/bash
# Round-2 probe 2: window-attention fix, cfg4 / cfg5 on one GPU, compute-sanitizer on the smoke.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/probe2; mkdir -p $O
timeout 600 python -m pytest tests/test_ops_gpu.py -q -p no:cacheprovider -k "window" > $O/ops.log 2>&1; echo "exit $?" >> $O/ops.log
timeout 1200 python scripts/cfg45.py cfg4 cfg5 --steps 3 > $O/cfg45.json 2> $O/cfg45.err; echo "exit $?" >> $O/cfg45.err
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitizer_$tool.log 2>&1; echo "exit $?" >> $O/sanitizer_$tool.log
done
tail -2 $O/ops.log; tail -3 $O/cfg45.err; head -c 1500 $O/cfg45.json; for t in memcheck synccheck racecheck; do tail -3 $O/sanitizer_$t.log; done
