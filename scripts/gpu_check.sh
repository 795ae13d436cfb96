cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"rope_kv_append_vec" -s 40 -c 1 -o gpurun_out/hbm_rope python scripts/one_run.py 1 > gpurun_out/ncu_hbm.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_hbm.log
timeout 600 ncu --set full --clock-control none -k regex:"scatter_rows" -s 2 -c 1 -o gpurun_out/hbm_scatter python scripts/one_run.py 1 >> gpurun_out/ncu_hbm.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_hbm.log
tail -n 3 gpurun_out/ncu_hbm.log
