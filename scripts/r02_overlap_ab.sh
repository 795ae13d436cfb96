#!/bin/bash
# Stream overlap policy A/B on the cfg2 TTFT (interleaved, two rounds): encoder priority (default), none,
# prefill priority, encode-first ordering, fully serialised.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
run() {  # label, env...
  local label=$1; shift
  env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --cfg3-steps 0 --cfg45 0 --decode-steps 0 \
    --no-cpu-baseline --no-parity 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['ttft_ms']
print('$label', 'p50', round(t['p50'],1), 'mean', round(t['mean'],1), 'clk', d['clocks']['sm_mhz'], 'steps', t['per_step'])"
}
for r in 1 2; do
  run enc RS_STREAM_PRIO=enc
  run none RS_STREAM_PRIO=none
  run prefill RS_STREAM_PRIO=prefill
  run encfirst RS_ENCODE_FIRST=1
  run serial RS_SERIALIZE=1
done > gpurun_out/overlap_ab.log 2>&1
cat gpurun_out/overlap_ab.log
