"""EP disaggregation on the device: every rank is a context of its own
(encoder ranks hold only the ViT, prefill ranks only their LLM layers, the
last one the LM head), wired by the in-process loopback transport so the whole
protocol — ENCODE control, embeddings into P0's staging ring, residual
hand-off between stages, DONE headers, logits rows back to P0 — runs on one
B200. Bars as in test_model_gpu.py: lock-step decisions byte-identical to the
reference simulator with the same stages / encoder workers; first-token
logits within 0.1 std of the fp32 oracle; real-clock journals replay through
the reference components."""
import numpy as np
import pytest

pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CFG1 = "T64|M256|M256|T32|M256|M256"
WL = f"0,0,-,{CFG1}\n1,3.5,-,T40|M64|T8\n2,4,-,M128|T16\n"


def _cfg(stages, encoders, policy="rserve", C=256, B=384):
    from paper_2509_24381_b200 import api
    return api.SimConfig(policy=policy, stages=stages, encoder_workers=encoders, token_budget=B,
                         embedding_batch_tokens=C, hidden_size=512,
                         cost=api.CostModel(alpha_enc_ms=0.5, beta_enc_ms_per_token=0.01,
                                            eps_tx_ms=0.2, zeta_tx_ms_per_token=0.001,
                                            delta_stage_ms_per_token=0.01))


def _group(stages, encoders):
    from paper_2509_24381_b200 import api
    m = api.model_preset("tiny")
    kw = dict(max_prompt_tokens=8192, slot_tokens=1 << 15, kv_tokens=1 << 15, max_chunk_tokens=2048,
              max_encode_tokens=1024)
    ctxs = [api.ep_context(m, r, stages, encoders, **kw) for r in range(stages + encoders)]
    return api.EpGroup(stages, encoders, "loopback"), ctxs


@pytest.fixture(scope="module")
def oracle_logits():
    from oracle import model_oracle as mo
    cfg = mo.ModelConfig.tiny()
    w = mo.Weights(cfg)
    llm = mo.LlmOracle(cfg, w)
    cache = {}

    def ref(rid, layout, seed, C):
        key = (rid, layout, seed, C)
        if key not in cache:
            emb = mo.request_embeddings(cfg, w, rid, layout, seed, C)
            h = llm.forward(emb, mo.mrope_positions(mo.parse_layout(layout)))
            cache[key] = llm.first_token_logits(h[-1])
        return cache[key]
    return ref


from _tol import check_logits as _check_logits  # noqa: E402


LAYOUTS = {0: CFG1, 1: "T40|M64|T8", 2: "M128|T16"}


@pytest.mark.parametrize("stages,encoders", [(1, 1), (2, 2), (1, 2), (2, 1), (4, 4)])
def test_ep_lockstep_decisions_and_logits(stages, encoders, oracle_logits):
    from oracle import ref
    from paper_2509_24381_b200 import api
    g, ctxs = _group(stages, encoders)
    sc = _cfg(stages, encoders)
    log, journal, stats = g.run(ctxs[0], ctxs[1:], WL, sc, clock="lockstep", payload_seed=7)
    assert log == api.simulate(WL, sc)[0]
    assert log == ref.simulate(WL, sc.to_c())
    for rid, layout in LAYOUTS.items():
        _check_logits(*ctxs[0].logits(rid), oracle_logits(rid, layout, 7, 256))
    # a second run on the same group / contexts (workers restart per run)
    log2, _, _ = g.run(ctxs[0], ctxs[1:], WL, sc, clock="lockstep", payload_seed=7)
    assert log2 == log
    g.close()
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("stages,encoders", [(1, 1), (2, 2)])
def test_ep_realclock_journal_replay(stages, encoders, oracle_logits):
    from oracle import ref
    from paper_2509_24381_b200 import api
    g, ctxs = _group(stages, encoders)
    sc = _cfg(stages, encoders)
    log, journal, stats = g.run(ctxs[0], ctxs[1:], WL, sc, clock="real", payload_seed=9)
    ours = api.parse_decision_log(log)
    theirs = api.parse_decision_log(ref.replay(WL, sc.to_c(), journal))
    key = lambda recs, ks: [{k: r[k] for k in ks} for r in recs]  # noqa: E731
    assert key(ours["slice"], ["req", "chunk", "start", "end"]) == \
        key(theirs["slice"], ["req", "chunk", "start", "end"])
    assert ours.get("release") == theirs.get("release")
    assert all(float(r["ttft"]) > 0 for r in ours["req"])
    assert stats["gpu_ms"] > 0
    for rid, layout in LAYOUTS.items():
        _check_logits(*ctxs[0].logits(rid), oracle_logits(rid, layout, 9, 256))
    g.close()
    for c in ctxs:
        c.close()


def test_ep_e2e_matches_resident():
    """Host-staged pixels on the encoder ranks and logits read back on P0 give
    the same first-token logits as device-resident inputs."""
    g, ctxs = _group(2, 1)
    sc = _cfg(2, 1)
    g.run(ctxs[0], ctxs[1:], WL, sc, clock="lockstep", payload_seed=11)
    a = {rid: ctxs[0].logits(rid) for rid in LAYOUTS}
    _, _, st = g.run(ctxs[0], ctxs[1:], WL, sc, clock="lockstep", e2e=True, payload_seed=11)
    for rid in LAYOUTS:
        b, am = ctxs[0].logits(rid)
        np.testing.assert_array_equal(a[rid][0], b)
        assert am == a[rid][1]
    assert st["d2h_bytes"] == 3 * 4096 * 4
    g.close()
    for c in ctxs:
        c.close()


def test_ep_matches_colocated():
    """EP 2+2 and one co-located GPU compute the same first-token logits."""
    from paper_2509_24381_b200 import api
    m = api.model_preset("tiny")
    p = api.Pipeline(m, max_prompt_tokens=8192, slot_tokens=1 << 15, kv_tokens=1 << 15,
                     max_chunk_tokens=2048, max_encode_tokens=1024)
    sc1 = _cfg(1, 1)
    p.run(WL, sc1, clock="lockstep", payload_seed=3)
    g, ctxs = _group(2, 2)
    g.run(ctxs[0], ctxs[1:], WL, _cfg(2, 2), clock="lockstep", payload_seed=3)
    for rid in LAYOUTS:
        a, am_a = p.logits(rid)
        b, am_b = ctxs[0].logits(rid)
        np.testing.assert_allclose(a, b, atol=2e-2 * np.abs(a).max())
    g.close()
    for c in ctxs:
        c.close()
    p.close()
