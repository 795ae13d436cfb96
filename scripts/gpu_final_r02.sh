#!/bin/bash
# Round-2 closing evidence: GPU tests, smoke, bench (N=1), reference arm, EP 1E+1P on one GPU, ncu launch list.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?" >> gpurun_out/bench_ref.err
timeout 900 python bench.py --gpus 2 --ep-same-device --steps 2 --warmup 1 > gpurun_out/bench_ep2.json 2> gpurun_out/bench_ep2.err; echo "ep2 exit $?" >> gpurun_out/bench_ep2.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --launch-list --no-cpu-baseline --decode-steps 0 > gpurun_out/bench_ncu.log 2>&1; echo "ncu exit $?" >> gpurun_out/bench_ncu.log
python scripts/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt 2>&1
tail -n 2 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.err gpurun_out/bench_ref.err gpurun_out/bench_ep2.err gpurun_out/bench_ncu.log
head -12 gpurun_out/launch_summary.txt
