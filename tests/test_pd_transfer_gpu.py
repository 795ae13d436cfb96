"""PD (prefill -> decode) KV transfer (the paper serves
EPD-disaggregated, §5.1): a request prefilled on one context with
keep_kv is exported as a KV image (rs_kv_export), the image is moved to a
decode-only context (no ViT, no embedding slab) and imported (rs_kv_import);
decoding there must give exactly the tokens and logits of decoding on the
prefill context itself (same kernels over the same KV bytes: bit-equal)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WL = "0,0,-,T64|M256|M256|T32\n1,3.5,-,T40|M64|T8\n"
STEPS = 6


def _cfg(hidden):
    from paper_2509_24381_b200 import api
    return api.SimConfig(policy="rserve", stages=1, token_budget=512, embedding_batch_tokens=256,
                         hidden_size=hidden, cost=api.CostModel(beta_enc_ms_per_token=0.01,
                                                                delta_stage_ms_per_token=0.01))


def _pair(model, **kw):
    from paper_2509_24381_b200 import api
    m = api.model_preset(model)
    for k, v in kw.items():
        setattr(m, k, v)
    p = api.Pipeline(m, max_prompt_tokens=4096, slot_tokens=1 << 13, kv_tokens=1 << 13,
                     max_chunk_tokens=1024, max_encode_tokens=1024)
    d = api.Pipeline(m, max_prompt_tokens=4096, slot_tokens=64, kv_tokens=1 << 13, max_chunk_tokens=64,
                     max_encode_tokens=64, with_vit=False)
    return m, p, d


@pytest.mark.parametrize("model,kw", [("tiny", {}), ("qwen2.5-vl-7b", {"llm_layers": 2, "vit_layers": 2})])
def test_kv_transfer_decode_equals_local_decode(model, kw):
    m, pre, dec = _pair(model, **kw)
    try:
        sc = _cfg(m.llm_dim)
        pre.run(WL, sc, clock="lockstep", payload_seed=5, keep_kv=True)
        firsts = {rid: pre.logits(rid)[1] for rid in (0, 1)}
        # export both requests' KV images, then decode locally for the reference tokens
        images, metas = {}, {}
        for rid in (0, 1):
            T = 64 + 256 + 256 + 32 if rid == 0 else 40 + 64 + 8
            nbytes = pre.kv_image_bytes(T)
            buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
            metas[rid] = pre.kv_export(rid, buf.data_ptr(), nbytes)
            torch.cuda.synchronize()
            assert metas[rid].tokens == T and metas[rid].image_bytes == nbytes
            # the "link": a device-to-device copy into the decode side's receive buffer
            images[rid] = buf.clone()
            first = int(images[rid][:4].view(torch.int32).item())
            assert first == firsts[rid], "image header carries the prefill's first token"
        ref_toks, ref_logits, _ = pre.decode([0, 1], STEPS, want_logits=True)
        for rid in (0, 1):
            pre.decode_release(rid)
        for rid in (1, 0):  # import order differs from the prefill side's slots
            dec.kv_import(rid, metas[rid], images[rid].data_ptr())
        torch.cuda.synchronize()
        toks, logits, ms = dec.decode([0, 1], STEPS, want_logits=True)
        np.testing.assert_array_equal(toks, ref_toks)
        np.testing.assert_array_equal(logits, ref_logits)
        assert ms > 0
        for rid in (0, 1):
            dec.decode_release(rid)
    finally:
        pre.close()
        dec.close()


def test_kv_import_rejects_mismatched_image():
    from paper_2509_24381_b200 import _native as N
    from paper_2509_24381_b200 import api
    m, pre, dec = _pair("tiny")
    try:
        pre.run("0,0,-,T40|M64|T8\n", _cfg(m.llm_dim), clock="lockstep", payload_seed=5, keep_kv=True)
        nbytes = pre.kv_image_bytes(112)
        buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        with pytest.raises(N.ConfigError):
            pre.kv_export(0, buf.data_ptr(), nbytes - 16)  # buffer too small
        meta = pre.kv_export(0, buf.data_ptr(), nbytes)
        torch.cuda.synchronize()
        bad = N.rs_kv_meta.from_buffer_copy(meta)
        bad.kv_heads += 1
        with pytest.raises(N.ConfigError):
            dec.kv_import(0, bad, buf.data_ptr())
        dec.kv_import(0, meta, buf.data_ptr())
        with pytest.raises(N.RegistryError):
            dec.kv_import(0, meta, buf.data_ptr())  # duplicate id
        dec.decode_release(0)
        pre.decode_release(0)
        # a stage context without the head cannot export (the first token lives on the last stage)
        st = api.Pipeline(m, max_prompt_tokens=4096, slot_tokens=1 << 12, kv_tokens=1 << 12, max_chunk_tokens=512,
                          max_encode_tokens=512, with_lm_head=False)
        with pytest.raises((N.ConfigError, N.RegistryError)):
            st.kv_export(0, buf.data_ptr(), nbytes)
        st.close()
    finally:
        pre.close()
        dec.close()
