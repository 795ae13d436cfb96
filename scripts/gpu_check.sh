cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_tcgen05 -s 2 -c 1 -o gpurun_out/gemm_gateup_pair_full python scripts/one_gemm.py 2048 37888 3584 2 0 > gpurun_out/ncu_full.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_full.log
tail -2 gpurun_out/ncu_full.log; tail -2 gpurun_out/bench.err
