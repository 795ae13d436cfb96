"""The fp32 numpy model oracle (oracle/model_oracle.py) on CPU.

The reference has no model math, so the oracle is pinned by (a) exactness of
its synthetic-value generator against an independent scalar restatement and
torch's bf16 rounding, (b) self-consistency properties that any correct
implementation of the path must have: chunked prefill == unchunked prefill,
and the vision encoder's output for an image does not depend on the other
images in its Algorithm-1 batch.
"""
import numpy as np
import pytest

from oracle import model_oracle as mo

M64 = (1 << 64) - 1


def _mix64_scalar(seed, stream, i):
    z = (seed * 0x9E3779B97F4A7C15 + stream * 0xD1B54A32D192ED03 + i) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def test_hash_matches_scalar_restatement():
    idx = np.array([0, 1, 2, 12345, 2**40 + 7], dtype=np.uint64)
    got = mo.mix64(20250928, mo.wid(3, 5, 1), idx)
    want = [_mix64_scalar(20250928, mo.wid(3, 5, 1), int(i)) for i in idx]
    assert [int(g) for g in got] == want


def test_bf16_rounding_matches_torch():
    torch = pytest.importorskip("torch")
    x = np.random.default_rng(0).standard_normal(100000).astype(np.float32) * 3
    x[:4] = [1.00390625, 1.01171875, -2.5e-38, 65504.0]  # ties / tiny / large
    want = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    np.testing.assert_array_equal(mo.bf16_round(x), want)


def test_uniform_weights_statistics():
    w = mo.uniform(1, mo.wid(1, 0, 1), 256, 256, mo.WEIGHT_SCALE)
    assert abs(float(w.std()) - 0.02) < 1e-3 and abs(float(w.mean())) < 1e-3
    # bf16-representable
    np.testing.assert_array_equal(mo.bf16_round(w), w)


def test_chunked_prefill_equals_unchunked():
    cfg = mo.ModelConfig.tiny()
    w = mo.Weights(cfg)
    layout = "T64|M256|T32|M128"
    emb = mo.request_embeddings(cfg, w, 0, layout, 7, 256)
    pos = mo.mrope_positions(mo.parse_layout(layout))
    llm = mo.LlmOracle(cfg, w)
    h1 = llm.forward(emb, pos)
    h2 = llm.forward(emb, pos, chunks=[100, 200, 180])
    np.testing.assert_allclose(h1, h2, atol=1e-5)


def test_vision_output_independent_of_batch():
    cfg = mo.ModelConfig.tiny()
    vis = mo.VisionOracle(cfg)
    a = (256, vis.patches(3, 1, 0, 256))
    b = (100, vis.patches(3, 1, 1, 100))
    both = vis.encode([a, b], layers=2)
    alone = vis.encode([b], layers=2)
    np.testing.assert_allclose(both[256:], alone, atol=1e-5)


def test_layout_helpers():
    assert mo.item_grid(1024) == (32, 32) and mo.item_grid(256) == (16, 16)
    assert mo.item_grid(100) == (10, 10) and mo.item_grid(7) == (1, 7)
    pos, wins, out_row = mo.item_plan(256, 4)
    assert len(pos) == 1024 and len(wins) == 16 and sorted(out_row.tolist()) == list(range(256))
    # Qwen2-VL rope index: text, then image (t, t+r, t+c), next = s + max(gh, gw)
    p = mo.mrope_positions([("T", 2), ("M", 4), ("T", 1)])
    assert p.tolist() == [[0, 0, 0], [1, 1, 1], [2, 2, 2], [2, 2, 3], [2, 3, 2], [2, 3, 3], [4, 4, 4]]
