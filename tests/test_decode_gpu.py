"""Decode after the first token on the device, checked
step by step against the fp32 oracle with teacher forcing: step s feeds the
token the device chose at step s-1 (the first: the prefill argmax) at prompt
position T+s, M-RoPE id max(prompt ids)+1+s, and must give the oracle's
logits of the whole sequence's last row within the first-token tolerance
(max|dlogit| <= 0.05 std; argmax equal)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _tol import check_logits  # noqa: E402

LAYOUTS = {0: "T64|M256|M256|T32", 1: "T40|M64|T8"}
WL = "0,0,-,T64|M256|M256|T32\n1,3.5,-,T40|M64|T8\n"
STEPS = 5


@pytest.fixture(scope="module")
def tiny():
    from paper_2509_24381_b200 import api
    p = api.Pipeline(api.model_preset("tiny"), max_prompt_tokens=8192, slot_tokens=1 << 15,
                     kv_tokens=1 << 15, max_chunk_tokens=2048, max_encode_tokens=1024)
    yield p
    p.close()


def _cfg():
    from paper_2509_24381_b200 import api
    return api.SimConfig(policy="rserve", stages=1, token_budget=512, embedding_batch_tokens=256,
                         hidden_size=512, cost=api.CostModel(beta_enc_ms_per_token=0.01,
                                                             delta_stage_ms_per_token=0.01))


def test_decode_matches_teacher_forced_oracle(tiny):
    from oracle import model_oracle as mo
    tiny.run(WL, _cfg(), clock="lockstep", payload_seed=7, keep_kv=True)
    first = {rid: tiny.logits(rid)[1] for rid in LAYOUTS}
    toks, logits, ms = tiny.decode([0, 1], STEPS, want_logits=True)
    assert ms > 0 and toks.shape == (STEPS, 2)
    cfg = mo.ModelConfig.tiny()
    w = mo.Weights(cfg)
    llm = mo.LlmOracle(cfg, w)
    for i, (rid, layout) in enumerate(LAYOUTS.items()):
        emb = mo.request_embeddings(cfg, w, rid, layout, 7, 256)
        pos = mo.mrope_positions(mo.parse_layout(layout))
        nxt = int(pos.max()) + 1
        fed = [first[rid]] + [int(t) for t in toks[:-1, i]]
        for s in range(STEPS):
            seq = np.concatenate([emb, w.embed_rows(np.array(fed[:s + 1]))])
            p3 = np.concatenate([pos, np.array([[nxt + k] * 3 for k in range(s + 1)])])
            ref = llm.first_token_logits(llm.forward(seq, p3)[-1])
            got = logits[s, i]
            err = np.abs(got - ref).max()
            assert err <= 0.05 * ref.std(), f"request {rid} step {s}: max|dlogit| {err:.4g}"
            assert int(toks[s, i]) == int(ref.argmax())
    for rid in LAYOUTS:
        tiny.decode_release(rid)


def test_decode_is_deterministic_and_release_frees(tiny):
    from paper_2509_24381_b200 import _native as N
    runs = []
    for _ in range(2):
        tiny.run(WL, _cfg(), clock="real", payload_seed=3, keep_kv=True)
        toks, _, _ = tiny.decode([1, 0], 4)
        runs.append(toks)
        for rid in LAYOUTS:
            tiny.decode_release(rid)
    np.testing.assert_array_equal(runs[0], runs[1])
    with pytest.raises(N.RegistryError):
        tiny.decode([0], 1)


def test_decode_split_calls_equal_one_call(tiny):
    """Decoding 2 + 2 steps in two rs_decode calls equals 4 steps in one: the
    second call continues the M-RoPE ids and KV positions where the first
    stopped (the rope start was recomputed from the prompt)."""
    tiny.run(WL, _cfg(), clock="lockstep", payload_seed=3, keep_kv=True)
    one, l1, _ = tiny.decode([0, 1], 4, want_logits=True)
    for rid in LAYOUTS:
        tiny.decode_release(rid)
    tiny.run(WL, _cfg(), clock="lockstep", payload_seed=3, keep_kv=True)
    a, la, _ = tiny.decode([0, 1], 2, want_logits=True)
    b, lb, _ = tiny.decode([0, 1], 2, want_logits=True)
    for rid in LAYOUTS:
        tiny.decode_release(rid)
    np.testing.assert_array_equal(one, np.concatenate([a, b]))
    np.testing.assert_array_equal(l1, np.concatenate([la, lb]))


def test_decode_qwen7b_width_shallow():
    """Decode kernel at the 7B shapes (hd 128, GQA 7:1, vocab 152064) with 2
    layers, two requests batched, teacher-forced against the fp32 oracle."""
    from oracle import model_oracle as mo
    from paper_2509_24381_b200 import api
    m = api.model_preset("qwen2.5-vl-7b", vit_layers=2, vit_fullatt_every=2, llm_layers=2)
    p = api.Pipeline(m, max_prompt_tokens=4096, slot_tokens=8192, kv_tokens=8192,
                     max_chunk_tokens=1024, max_encode_tokens=1024)
    layouts = {0: "T32|M256|T16", 1: "T100|M64|T3"}
    wl = "0,0,-,T32|M256|T16\n1,0,-,T100|M64|T3\n"
    sc = api.SimConfig(policy="rserve", stages=1, token_budget=512, embedding_batch_tokens=256,
                       hidden_size=3584, cost=api.CostModel(beta_enc_ms_per_token=0.01,
                                                           delta_stage_ms_per_token=0.01))
    p.run(wl, sc, payload_seed=5, keep_kv=True)
    first = {rid: p.logits(rid)[1] for rid in layouts}
    steps = 3
    toks, logits, _ = p.decode([0, 1], steps, want_logits=True)
    cfg = mo.ModelConfig.qwen7b(vit_layers=2, vit_fullatt_every=2, llm_layers=2)
    w = mo.Weights(cfg)
    llm = mo.LlmOracle(cfg, w)
    for i, (rid, layout) in enumerate(layouts.items()):
        emb = mo.request_embeddings(cfg, w, rid, layout, 5, 256)
        emb16 = mo.request_embeddings(cfg, w, rid, layout, 5, 256, bf16_acts=True)
        pos = mo.mrope_positions(mo.parse_layout(layout))
        nxt = int(pos.max()) + 1
        fed = [first[rid]] + [int(t) for t in toks[:-1, i]]
        for s in range(steps):
            fed_rows = w.embed_rows(np.array(fed[:s + 1]))
            p3 = np.concatenate([pos, np.array([[nxt + k] * 3 for k in range(s + 1)])])
            ref = llm.first_token_logits(llm.forward(np.concatenate([emb, fed_rows]), p3)[-1])
            ref16 = llm.first_token_logits(llm.forward(np.concatenate([emb16, fed_rows]), p3,
                                                       bf16_acts=True)[-1])
            check_logits(logits[s, i], toks[s, i], ref, f"request {rid} step {s}", ref_bf16=ref16)
    for rid in layouts:
        p.decode_release(rid)
    p.close()
