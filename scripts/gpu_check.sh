cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for ms in 200 1000 200 1000; do
timeout 900 python bench.py --no-cpu-baseline --steps 8 --decode-steps 0 --clock-sample-ms $ms > gpurun_out/bench_$ms.json 2> gpurun_out/bench.err
python -c "
import json;d=json.load(open('gpurun_out/bench_$ms.json'))
print($ms, round(d['ttft_ms']['p50'],1), [round(x) for x in d['ttft_ms']['per_step']], round(d['e2e']['p50_ms'],1), d['clocks'])"
done
