"""Tensor parallelism across ranks over peer memory: a TP
group of T contexts (rs_ctx_options.tp_group), each holding one weight shard
and an exchange buffer, connected by rs_tp_connect. Every layer's O / down
partials are reduced by tp_group_reduce_kernel: flags written into the peers'
buffers (st.release.sys) and polled (ld.acquire.sys), then the T partials read
straight from the peers' memory in rank order. On an NVSwitch box the ranks
are one process per GPU (IPC handles); here they share one B200 in one
process (device pointers) — the same kernels and the same protocol.

The group computes exactly what the loopback shards of ONE context compute
(same shard weights, same partial GEMMs, the same rank-order fp32 sum), so
the first-token logits must be bit-equal to the loopback TP context's, the
residual stream bit-equal across ranks, and within the first-token tolerance
of the unsharded model."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LAYOUT = "T16|M64|T8"
CHUNKS = [(0, 40), (40, 88)]


MODELS = {"tiny": ("tiny", {}), "7b-2l": ("qwen2.5-vl-7b", {"llm_layers": 2, "vit_layers": 2})}


def _model(name):
    from paper_2509_24381_b200 import api
    preset, kw = MODELS[name]
    return api.model_preset(preset, **kw)


def _ref_pipe(tp, name):
    from paper_2509_24381_b200 import api
    return api.Pipeline(_model(name), max_prompt_tokens=4096, slot_tokens=8192, kv_tokens=8192,
                        max_chunk_tokens=512, max_encode_tokens=512, tp_size=tp)


def _embeddings_and_ref(tp, name):
    """Encode the request on a context with the tracker, return its embedding
    rows [T, d] (bf16 bits) and that context's chunked-prefill logits."""
    p = _ref_pipe(tp, name)
    g = torch.Generator(device="cuda").manual_seed(11)
    px = torch.randn(4 * 64, 1176, device="cuda", generator=g).to(torch.bfloat16)
    p.request_create(1, LAYOUT)
    out = p.encode([(16, 80)], px.data_ptr(), on_host=False)
    p.mark_encoded(1, 16, 80, out)
    emb = p.read_slots(1, 0, 88)
    for b, e in CHUNKS:
        p.prefill_chunk([(1, b, e)])
    logits, am = p.logits(1)
    p.close()
    return emb, logits.copy(), am


@pytest.mark.parametrize("name,T", [("tiny", 2), ("7b-2l", 2), ("7b-2l", 4)])
def test_tp_group_equals_loopback_shards(name, T):
    from paper_2509_24381_b200 import api
    emb, ref_logits, ref_am = _embeddings_and_ref(T, name)
    _, full_logits, _ = _embeddings_and_ref(1, name)
    ranks = [api.Pipeline(_model(name), max_prompt_tokens=4096, slot_tokens=64, kv_tokens=8192,
                          max_chunk_tokens=512, max_encode_tokens=64, with_vit=False, tp_size=T, tp_rank=r,
                          tp_group=True)
             for r in range(T)]
    try:
        bufs = [rk.tp_buffer() for rk in ranks]
        for rk in ranks:
            rk.tp_connect([b[0] for b in bufs])
        for rk in ranks:
            rk.kv_request_create(1, LAYOUT)
        e = torch.from_numpy(emb.view(np.int16)).view(torch.bfloat16).cuda()
        xs = []
        for b, en in CHUNKS:  # every rank enqueues the same chunk sequence; nothing blocks the host
            xr = [e[b:en].clone() for _ in ranks]
            for rk, x in zip(ranks, xr):
                rk.tp_prefill([(1, b, en)], x.data_ptr())
            xs.append(xr)
        torch.cuda.synchronize()
        for xr in xs:  # the same residual stream on every rank, to the bit
            for x in xr[1:]:
                assert torch.equal(x.view(torch.int16), xr[0].view(torch.int16))
        for rk in ranks:
            logits, am = rk.tp_logits(1)
            np.testing.assert_array_equal(logits, ref_logits)
            assert am == ref_am
        err = np.abs(ref_logits - full_logits).max()
        assert err <= 0.05 * full_logits.std(), f"TP={T} vs unsharded: max|dlogit| {err:.4g}"
    finally:
        for rk in ranks:
            rk.close()


def test_tp_group_config_errors():
    from paper_2509_24381_b200 import _native as N
    from paper_2509_24381_b200 import api
    m = api.model_preset("tiny")
    with pytest.raises(N.ConfigError):
        api.Pipeline(m, max_chunk_tokens=64, with_vit=False, tp_size=2, tp_rank=2, tp_group=True)
    with pytest.raises(N.ConfigError):
        api.Pipeline(m, max_chunk_tokens=64, with_vit=True, tp_size=2, tp_rank=0, tp_group=True)
    r = api.Pipeline(m, max_prompt_tokens=512, slot_tokens=64, kv_tokens=1024, max_chunk_tokens=64,
                     max_encode_tokens=64, with_vit=False, tp_size=2, tp_rank=0, tp_group=True)
    r.kv_request_create(1, "T16")
    x = torch.zeros(16, m.llm_dim, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(N.ConfigError, match="rs_tp_connect"):
        r.tp_prefill([(1, 0, 16)], x.data_ptr())  # not connected: refused before any kernel spins
    # a peer of another shape (chunk rows) or the buffers in the wrong rank order: refused at connect
    other = api.Pipeline(m, max_prompt_tokens=512, slot_tokens=64, kv_tokens=1024, max_chunk_tokens=128,
                         max_encode_tokens=64, with_vit=False, tp_size=2, tp_rank=1, tp_group=True)
    with pytest.raises(N.ConfigError, match="exchange buffer"):
        r.tp_connect([r.tp_buffer()[0], other.tp_buffer()[0]])
    with pytest.raises(N.ConfigError, match="exchange buffer"):
        r.tp_connect([other.tp_buffer()[0], r.tp_buffer()[0]])
    other.close()
    r.close()
