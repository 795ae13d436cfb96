"""The torch fp32 mirror of the model oracle (oracle/model_oracle_torch.py)
equals the numpy oracle (oracle/model_oracle.py, itself pinned to HF
transformers in test_oracle_hf.py) on CPU, so the full-depth cfg2 check on
the GPU box (tests/test_cfg2_parity_gpu.py) uses the same checker.

Bars: the weight / pixel / token generators are bit-equal; the forwards agree
to 1e-4 relative (fp32 vs fp32, different summation order / BLAS)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import model_oracle as mo  # noqa: E402
from oracle import model_oracle_torch as mt  # noqa: E402

RTOL = 1e-4


def _rel(got, ref):
    return float(np.abs(got - ref).max() / (np.abs(ref).max() + 1e-30))


def test_generators_bit_equal():
    c = mo.ModelConfig.tiny()
    for stream, rows, cols, row0 in ((mo.wid(mo.LLM, 3, mo.QKV_W), 7, 513, 0),
                                     (mo.wid(mo.TOP, 0, mo.HEAD), 5, 96, 150000),
                                     (mo.pixel_stream(3, 9), 4, 1176, 0)):
        a = mo.uniform(c.weight_seed, stream, rows, cols, mo.WEIGHT_SCALE, row0=row0)
        b = mt.uniform(c.weight_seed, stream, rows, cols, mo.WEIGHT_SCALE, row0=row0).numpy()
        np.testing.assert_array_equal(a, b)
    ids = np.array([0, 5, 4095, 77], dtype=np.int64)
    np.testing.assert_array_equal(mo.Weights(c).embed_rows(ids),
                                  mt.Weights(c).embed_rows(torch.from_numpy(ids)).numpy())
    x = np.random.default_rng(0).standard_normal(4096).astype(np.float32)
    np.testing.assert_array_equal(mo.bf16_round(x), mt.bf16_round(torch.from_numpy(x)).numpy())


@pytest.mark.parametrize("which,vit_layers,llm_layers,layout,bf16", [
    ("tiny", None, None, "T64|M256|T1|M60|T32|M7", False),   # full tiny depth, edge windows
    ("tiny", None, None, "T16|M64|T8", True),                # bf16 activation rounding mode
    ("qwen7b", 1, 1, "T24|M64|T16|M20|T8", False),           # 7B widths, one layer each
])
def test_torch_mirror_equals_numpy(which, vit_layers, llm_layers, layout, bf16):
    kw = {}
    if vit_layers is not None:
        kw.update(vit_layers=vit_layers, llm_layers=llm_layers, vocab=4096)
    c = getattr(mo.ModelConfig, which)(**kw)
    W = mo.Weights(c)
    # numpy: Algorithm-1 batches of >= 64 tokens; torch: one pass over all items
    emb = mo.request_embeddings(c, W, 2, layout, 11, 64, bf16_acts=bf16)
    llm = mo.LlmOracle(c, W)
    h = llm.forward(emb, mo.mrope_positions(mo.parse_layout(layout)), bf16_acts=bf16)
    logits = llm.first_token_logits(h[-1])
    temb, tlogits = mt.first_token_logits(c, layout, 11, req_id=2, bf16_acts=bf16)
    tol = RTOL if not bf16 else 2e-2  # bf16 rounding flips propagate through depth
    assert _rel(temb.numpy(), emb) <= tol, _rel(temb.numpy(), emb)
    assert _rel(tlogits.numpy(), logits) <= tol, _rel(tlogits.numpy(), logits)
    assert int(tlogits.argmax()) == int(logits.argmax())
