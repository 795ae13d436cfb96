#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/probe7; mkdir -p $O
timeout 1200 python -m pytest tests/test_ops_gpu.py tests/test_model_gpu.py tests/test_tp_gpu.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "exit $?" >> $O/tests.log
RS_GEMM_SMALL_MIN_KB=32 timeout 900 python scripts/gemm_probe.py --small-m > $O/gemm_small_kb32.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --cfg3-steps 0 --decode-steps 0 --cfg45 0 --no-parity > $O/bench_default.json 2> $O/bench_default.err
RS_GEMM_SMALL_MIN_KB=32 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --cfg3-steps 0 --decode-steps 0 --cfg45 0 --no-parity > $O/bench_kb32.json 2> $O/bench_kb32.err
tail -3 $O/tests.log
for f in bench_default bench_kb32; do python -c "
import json,sys;d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]);print('$f', d['ttft_ms']['p50'], d['e2e']['p50_ms'], [ (s['M'],s['N'],s['K'],s['epi'],s['tile'],round(s['ms'],3)) for s in d['gemm_shapes'] if s['epi']==5 or s['M']<=256])"; done
