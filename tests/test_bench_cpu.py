"""bench.py plumbing on CPU (no GPU): the multi-GPU launch, EP roles, the
reference arm's independence from the product library, and the oracle's
standalone config structs (the reference arm drives oracle/_ref with them).
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                         text=True, timeout=timeout, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    return json.loads(lines[-1])


@pytest.mark.parametrize("n,roles,placement", [
    (2, ["prefill0", "encoder0"], "EP 1E+1P"),
    (4, ["prefill0", "prefill1", "encoder0", "encoder1"], "EP 2E+2P"),
])
def test_gpus_n_spawns_ep_ranks(n, roles, placement):
    """`bench.py --gpus N` re-executes under torch.distributed.run with N
    ranks (gloo plumbing here) and by default runs the EP deployment."""
    j = _run(["--gpus", str(n), "--dry-run"])
    assert j["n_gpus"] == n
    assert [r["role"] for r in j["ranks"]] == roles
    assert len({r["pid"] for r in j["ranks"]}) == n  # one process per rank
    assert j["config"]["placement"] == placement
    assert j["config"]["transport"] == "nccl"
    assert j["config"]["workload"].startswith("cfg3")


def test_gpus_1_is_cfg2_colocated():
    j = _run(["--dry-run"])
    assert j["n_gpus"] == 1 and j["config"]["workload"].startswith("cfg2")
    assert j["config"]["placement"] == "encoder+prefill co-located, 2 streams"


def test_reference_arm_never_loads_the_product():
    """The reference arm's code path (shapes, FLOP model, scheduler timing,
    config) runs with the product package made unimportable."""
    pytest.importorskip("numpy")
    from oracle import ref
    if not os.path.exists(ref.LIB):
        pytest.skip("oracle/_ref not built")
    code = (
        "import sys; sys.modules['paper_2509_24381_b200'] = None\n"
        "import bench, argparse\n"
        "m = bench.qwen7b_shapes()\n"
        "t = bench.ref_sched_time([f'0,0,-,{bench.LAYOUT}\\n'], 1, 1, 2048, 'rserve', reps=3)\n"
        "a = argparse.Namespace(mode='ep', policy='rserve', budget=2048, ep_transport='nccl')\n"
        "print(m['llm_dim'], t[0] > 0, bench.bench_config(a, 4)['placement'])\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=120)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.split() == ["3584", "True", "EP", "2E+2P"]


def test_shapes_match_product_preset():
    import bench
    from paper_2509_24381_b200 import _native as N
    from paper_2509_24381_b200 import api
    p = api.model_preset("qwen2.5-vl-7b")
    prod = {k: getattr(p, k) for k, _ in N.rs_model_config._fields_}
    for k, v in bench.qwen7b_shapes().items():
        assert prod[k] == v, k


def test_oracle_presets_match_product_presets():
    """The oracle's model configs are the product's presets (7B and cfg5's 72B-shaped LLM)."""
    from oracle import model_oracle as mo
    from paper_2509_24381_b200 import _native as N
    from paper_2509_24381_b200 import api
    for name, oc in (("qwen2.5-vl-7b", mo.ModelConfig.qwen7b()), ("qwen2.5-vl-72b-llm", mo.ModelConfig.qwen72b_llm())):
        p = api.model_preset(name)
        prod = {k: getattr(p, k) for k, _ in N.rs_model_config._fields_}
        for k in ("vit_dim", "vit_layers", "vit_heads", "vit_ff", "vit_fullatt_every", "patch_dim", "llm_dim",
                  "llm_layers", "llm_q_heads", "llm_kv_heads", "llm_head_dim", "llm_ff", "vocab"):
            assert prod[k] == getattr(oc, k), (name, k)


def test_oracle_structs_match_product_structs():
    """oracle/ref.py's standalone SimConfig / WorkloadConfig mirrors give the
    reference the same inputs as the product's ctypes structs."""
    from oracle import ref
    if not os.path.exists(ref.LIB):
        pytest.skip("oracle/_ref not built")
    import bench
    from paper_2509_24381_b200 import api
    for seed in (1, 2, 3):
        ours = bench.cfg3_workload(seed, 4.0, 3.0)
        w, _keep = ref.workload_config(seed, 4.0, 3.0, "alternating", (4, 16), 1024, (32, 256))
        assert ref.generate_workload(w) == ours
        assert len(bench.workload_layouts(ours)) >= 3
    wl = bench.cfg3_workload(2, 32.0, 0.5)
    for stages, enc in ((1, 1), (2, 2), (4, 4)):
        sc = api.SimConfig(policy="rserve", stages=stages, token_budget=2048, embedding_batch_tokens=1024,
                           encoder_workers=enc, hidden_size=3584,
                           cost=api.CostModel(beta_enc_ms_per_token=0.01, delta_stage_ms_per_token=0.01))
        rc = ref.sim_config("rserve", stages, 2048, 1024, enc, 3584, beta_enc_ms_per_token=0.01,
                            delta_stage_ms_per_token=0.01)
        assert ref.simulate(wl, rc) == ref.simulate(wl, sc.to_c()) == api.simulate(wl, sc)[0]


def test_nearest_rank_matches_reference_definition():
    import bench
    v = list(range(1, 101))
    assert bench.nearest_rank(v, 50) == 50 and bench.nearest_rank(v, 99) == 99
    assert bench.nearest_rank([7.0], 99) == 7.0
    assert bench.nearest_rank([1, 2, 3], 50) == 2
