cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fa_pp_kernel -s 2 -c 1 -o gpurun_out/attn_pp_full python scripts/one_attn.py 6144 > gpurun_out/ncu_attn.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_attn.log
tail -n 2 gpurun_out/bench.err gpurun_out/ncu_attn.log
