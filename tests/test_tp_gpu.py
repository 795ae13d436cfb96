"""Tensor parallelism inside the prefill group, loopback
shards on one B200: the LLM's heads and SwiGLU width split T ways, O / down
partials reduced per layer in shard order. The sharded model is the same
model, so first-token (and decode) logits must match the fp32 oracle within
the first-token tolerance (max|dlogit| <= 0.05 std), and the unsharded run
within the same bar."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LAYOUTS = {0: "T64|M256|M256|T32", 1: "T40|M64|T8"}
WL = "0,0,-,T64|M256|M256|T32\n1,3.5,-,T40|M64|T8\n"


def _cfg(hidden=512):
    from paper_2509_24381_b200 import api
    return api.SimConfig(policy="rserve", stages=1, token_budget=512, embedding_batch_tokens=256,
                         hidden_size=hidden, cost=api.CostModel(beta_enc_ms_per_token=0.01,
                                                                delta_stage_ms_per_token=0.01))


def _pipe(tp, model="tiny", **kw):
    from paper_2509_24381_b200 import api
    return api.Pipeline(api.model_preset(model, **kw), max_prompt_tokens=8192, slot_tokens=1 << 15,
                        kv_tokens=1 << 15, max_chunk_tokens=1024, max_encode_tokens=1024, tp_size=tp)


def test_tp2_matches_oracle_and_tp1():
    from oracle import model_oracle as mo
    cfg = mo.ModelConfig.tiny()
    w = mo.Weights(cfg)
    llm = mo.LlmOracle(cfg, w)
    runs = {}
    for tp in (1, 2):
        p = _pipe(tp)
        p.run(WL, _cfg(), clock="lockstep", payload_seed=7)
        runs[tp] = {rid: p.logits(rid)[0].copy() for rid in LAYOUTS}
        p.close()
    for rid, layout in LAYOUTS.items():
        emb = mo.request_embeddings(cfg, w, rid, layout, 7, 256)
        ref = llm.first_token_logits(llm.forward(emb, mo.mrope_positions(mo.parse_layout(layout)))[-1])
        for tp in (1, 2):
            err = np.abs(runs[tp][rid] - ref).max()
            assert err <= 0.05 * ref.std(), f"tp={tp} request {rid}: max|dlogit| {err:.4g}"
        assert np.abs(runs[2][rid] - runs[1][rid]).max() <= 0.05 * ref.std()


def test_tp2_decode_teacher_forced():
    from oracle import model_oracle as mo
    p = _pipe(2)
    p.run(WL, _cfg(), clock="lockstep", payload_seed=7, keep_kv=True)
    first = {rid: p.logits(rid)[1] for rid in LAYOUTS}
    toks, logits, _ = p.decode([0, 1], 3, want_logits=True)
    cfg = mo.ModelConfig.tiny()
    w = mo.Weights(cfg)
    llm = mo.LlmOracle(cfg, w)
    for i, (rid, layout) in enumerate(LAYOUTS.items()):
        emb = mo.request_embeddings(cfg, w, rid, layout, 7, 256)
        pos = mo.mrope_positions(mo.parse_layout(layout))
        nxt = int(pos.max()) + 1
        fed = [first[rid]] + [int(t) for t in toks[:-1, i]]
        for s in range(3):
            seq = np.concatenate([emb, w.embed_rows(np.array(fed[:s + 1]))])
            p3 = np.concatenate([pos, np.array([[nxt + k] * 3 for k in range(s + 1)])])
            ref = llm.first_token_logits(llm.forward(seq, p3)[-1])
            assert np.abs(logits[s, i] - ref).max() <= 0.05 * ref.std()
    for rid in LAYOUTS:
        p.decode_release(rid)
    p.close()


def test_tp4_qwen7b_width_shallow():
    from oracle import model_oracle as mo
    p = _pipe(4, "qwen2.5-vl-7b", vit_layers=2, vit_fullatt_every=2, llm_layers=2)
    layout = "T32|M256|T16"
    p.run(f"0,0,-,{layout}\n", _cfg(3584), clock="lockstep", payload_seed=5)
    got, _ = p.logits(0)
    cfg = mo.ModelConfig.qwen7b(vit_layers=2, vit_fullatt_every=2, llm_layers=2)
    w = mo.Weights(cfg)
    llm = mo.LlmOracle(cfg, w)
    emb = mo.request_embeddings(cfg, w, 0, layout, 5, 256)
    ref = llm.first_token_logits(llm.forward(emb, mo.mrope_positions(mo.parse_layout(layout)))[-1])
    assert np.abs(got - ref).max() <= 0.05 * ref.std()
    p.close()


def test_tp_rejects_indivisible_heads():
    from paper_2509_24381_b200 import _native as N
    with pytest.raises(N.ConfigError, match="does not divide"):
        _pipe(3)
