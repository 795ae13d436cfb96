cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_ops_gpu.py -x -q -p no:cacheprovider -k "attention" > gpurun_out/attn_tests.log 2>&1; echo "exit $?" >> gpurun_out/attn_tests.log
tail -n 3 gpurun_out/attn_tests.log
timeout 300 python scripts/kernel_bench.py --attn > gpurun_out/kb_attn.json 2>&1
RS_ATTN_SPLIT=0 timeout 300 python scripts/kernel_bench.py --attn > gpurun_out/kb_attn0.json 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/kb_attn.json","gpurun_out/kb_attn0.json"):
    d=json.load(open(f))
    print(f, [round(a.get("tflops", a.get("tflops_tcgen05", 0))) for a in d["attention"]])
PY
