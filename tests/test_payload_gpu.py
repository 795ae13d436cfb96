"""Payload files on the device engine: a payload that
restates the synthesised defaults changes nothing (bit-identical logits); a
generated payload (non-square image grids, other pixel / token seeds) gives
the first-token logits of the fp32 oracle fed the same payload, resolved by
the oracle's own reading of the file (oracle/payload.py). Tolerances as in
test_model_gpu.py."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LAYOUTS = {0: "T64|M256|M256|T32|M256|M256", 1: "T40|M64|T8"}
WL = "0,0,-,T64|M256|M256|T32|M256|M256\n1,3.5,-,T40|M64|T8\n"


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


def test_default_restating_payload_is_identity(tiny):
    tiny.run(WL, _cfg(), clock="lockstep", payload_seed=7)
    base = {rid: tiny.logits(rid) for rid in LAYOUTS}
    same = ("0,1,M,grid=16x16;seed=7\n0,2,M,grid=16x16;seed=7\n0,0,T,seed=7\n"
            "0,3,T,seed=7\n1,1,M,grid=8x8;seed=7\n1,2,T,seed=7\n")
    tiny.run(WL, _cfg(), clock="lockstep", payload_seed=7, payload=same)
    for rid in LAYOUTS:
        got, am = tiny.logits(rid)
        np.testing.assert_array_equal(got, base[rid][0])
        assert am == base[rid][1]


def test_generated_payload_matches_oracle(tiny):
    from oracle import model_oracle as mo
    from oracle import payload as op
    from paper_2509_24381_b200 import api
    text = api.generate_payload(WL, 5)
    # a non-square grid on purpose (16x16 -> 8x32 keeps 256 tokens)
    text = text.replace("0,1,M,grid=16x16", "0,1,M,grid=8x32")
    text += "1,0,T,ids=" + " ".join(str((37 * i) % 4096) for i in range(40)) + "\n"
    lines = {}
    for ln in text.splitlines():
        if ln and not ln.startswith("#"):
            lines[tuple(ln.split(",")[:2])] = ln  # the explicit ids replace the seeded line
    text = "\n".join(lines.values()) + "\n"
    tiny.run(WL, _cfg(), clock="lockstep", payload_seed=7, payload=text)
    cfg = mo.ModelConfig.tiny()
    w = mo.Weights(cfg)
    llm = mo.LlmOracle(cfg, w)
    spec = op.parse(text)
    with_payload = {rid: tiny.logits(rid)[0].copy() for rid in LAYOUTS}
    for rid, layout in LAYOUTS.items():
        res = op.resolve(layout, rid, spec.get(rid), 7, cfg.vocab)
        emb = mo.request_embeddings(cfg, w, rid, layout, 7, 256, payload=res)
        h = llm.forward(emb, mo.mrope_positions(mo.parse_layout(layout), res["item_grids"]))
        ref = llm.first_token_logits(h[-1])
        got, am = tiny.logits(rid)
        err = np.abs(got - ref).max()
        assert err <= 0.05 * ref.std(), f"request {rid}: max|dlogit| {err:.4g}"
    # and it really changed the inputs
    tiny.run(WL, _cfg(), clock="lockstep", payload_seed=7)
    for rid in LAYOUTS:
        assert np.abs(tiny.logits(rid)[0] - with_payload[rid]).max() > 1e-3


def test_payload_errors_surface_as_input_errors(tiny):
    from paper_2509_24381_b200 import _native as N
    with pytest.raises(N.InputError, match="grid 10x10 != 256 tokens"):
        tiny.run(WL, _cfg(), clock="lockstep", payload_seed=7, payload="0,1,M,grid=10x10\n")
