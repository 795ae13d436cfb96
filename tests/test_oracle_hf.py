"""Pin the fp32 model oracle (oracle/model_oracle.py) to an independent
implementation: Hugging Face transformers' Qwen2.5-VL modules
(transformers/models/qwen2_5_vl/modeling_qwen2_5_vl.py, v5.5 in this image).

The reference (lmmsim) has no model arithmetic, so the
oracle restates the public Qwen2.5-VL architecture. These CPU tests load the
oracle's seeded weights into the HF modules and require the two fp32 forwards
to agree:

* the whole vision tower `Qwen2_5_VisionTransformerPretrainedModel`
  (Conv3d patch embed, 2-D rotary `rot_pos_emb`, `get_window_index` window
  permutation + `cu_window_seqlens`, window / full attention blocks, RMSNorm,
  SwiGLU MLP, `Qwen2_5_VLPatchMerger`, reverse window index) — with the HF
  pixel rows in the processor's raster (merge-group-major) order and ours in
  window-major order, so the permutation is checked explicitly;
* `Qwen2_5_VLModel.get_rope_index` (M-RoPE positions of interleaved
  text / image layouts) against `mrope_positions`;
* `Qwen2_5_VLTextModel` (decoder layers with `apply_multimodal_rotary_pos_emb`,
  GQA, final norm) + the LM head against `LlmOracle`.

Bar: relative max error <= 1e-4 (fp32 vs fp32; different summation order).
A drift of the oracle from HF fails here, on CPU, before any GPU test runs.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
hf = pytest.importorskip("transformers.models.qwen2_5_vl.modeling_qwen2_5_vl")
from transformers.models.qwen2_5_vl.configuration_qwen2_5_vl import (  # noqa: E402
    Qwen2_5_VLConfig, Qwen2_5_VLTextConfig, Qwen2_5_VLVisionConfig)

from oracle import model_oracle as mo  # noqa: E402

RTOL = 1e-4


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32))


def _rel(got, ref):
    return float(np.abs(got - ref).max() / (np.abs(ref).max() + 1e-30))


def _vision_cfg(c: mo.ModelConfig, depth: int) -> Qwen2_5_VLVisionConfig:
    e = c.vit_fullatt_every
    return Qwen2_5_VLVisionConfig(
        depth=depth, hidden_size=c.vit_dim, hidden_act="silu", intermediate_size=c.vit_ff,
        num_heads=c.vit_heads, in_channels=3, patch_size=14, spatial_merge_size=2,
        temporal_patch_size=2, window_size=112, out_hidden_size=c.llm_dim,
        fullatt_block_indexes=[i for i in range(depth) if e > 0 and i % e == e - 1])


def _text_cfg(c: mo.ModelConfig, layers: int) -> Qwen2_5_VLTextConfig:
    hd = c.llm_head_dim
    return Qwen2_5_VLTextConfig(
        vocab_size=c.vocab, hidden_size=c.llm_dim, intermediate_size=c.llm_ff,
        num_hidden_layers=layers, num_attention_heads=c.llm_q_heads,
        num_key_value_heads=c.llm_kv_heads, rms_norm_eps=c.rms_eps, hidden_act="silu",
        rope_parameters={"rope_type": "default", "rope_theta": c.rope_theta_llm,
                         "mrope_section": [hd // 8, 3 * hd // 16, 3 * hd // 16]})


def _load_vision(model, c: mo.ModelConfig, W: mo.Weights, depth: int):
    vd, ff, mi = c.vit_dim, c.vit_ff, 4 * c.vit_dim
    sd = {"patch_embed.proj.weight": _t(W.lin(mo.VIT, 0, mo.PATCH, vd, c.patch_dim)).view(vd, 3, 2, 14, 14)}
    for l in range(depth):
        p = f"blocks.{l}."
        sd[p + "norm1.weight"] = torch.ones(vd)
        sd[p + "norm2.weight"] = torch.ones(vd)
        sd[p + "attn.qkv.weight"] = _t(W.lin(mo.VIT, l, mo.QKV_W, 3 * vd, vd))
        sd[p + "attn.qkv.bias"] = _t(W.vec(mo.VIT, l, mo.QKV_B, 3 * vd))
        sd[p + "attn.proj.weight"] = _t(W.lin(mo.VIT, l, mo.O_W, vd, vd))
        sd[p + "attn.proj.bias"] = _t(W.vec(mo.VIT, l, mo.O_B, vd))
        for name, tw, tb, rows, cols in (("gate_proj", mo.GATE_W, mo.GATE_B, ff, vd),
                                         ("up_proj", mo.UP_W, mo.UP_B, ff, vd),
                                         ("down_proj", mo.DOWN_W, mo.DOWN_B, vd, ff)):
            sd[p + f"mlp.{name}.weight"] = _t(W.lin(mo.VIT, l, tw, rows, cols))
            sd[p + f"mlp.{name}.bias"] = _t(W.vec(mo.VIT, l, tb, rows))
    sd["merger.ln_q.weight"] = torch.ones(vd)
    sd["merger.mlp.0.weight"] = _t(W.lin(mo.MERGER, 0, mo.FC1_W, mi, mi))
    sd["merger.mlp.0.bias"] = _t(W.vec(mo.MERGER, 0, mo.FC1_B, mi))
    sd["merger.mlp.2.weight"] = _t(W.lin(mo.MERGER, 0, mo.FC2_W, c.llm_dim, mi))
    sd["merger.mlp.2.bias"] = _t(W.vec(mo.MERGER, 0, mo.FC2_B, c.llm_dim))
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected and all("inv_freq" in m for m in missing), (missing, unexpected)


def _load_text(model, c: mo.ModelConfig, W: mo.Weights, layers: int):
    d, hq, hkv, hd, ff = c.llm_dim, c.llm_q_heads, c.llm_kv_heads, c.llm_head_dim, c.llm_ff
    qkv_dim = (hq + 2 * hkv) * hd
    sd = {"norm.weight": torch.ones(d), "embed_tokens.weight": torch.zeros(c.vocab, d)}
    for l in range(layers):
        p = f"layers.{l}."
        wqkv = W.lin(mo.LLM, l, mo.QKV_W, qkv_dim, d)
        bqkv = W.vec(mo.LLM, l, mo.QKV_B, qkv_dim)
        cuts = [0, hq * hd, (hq + hkv) * hd, qkv_dim]
        for i, n in enumerate(("q_proj", "k_proj", "v_proj")):
            sd[p + f"self_attn.{n}.weight"] = _t(wqkv[cuts[i]:cuts[i + 1]])
            sd[p + f"self_attn.{n}.bias"] = _t(bqkv[cuts[i]:cuts[i + 1]])
        sd[p + "self_attn.o_proj.weight"] = _t(W.lin(mo.LLM, l, mo.O_W, d, hq * hd))
        sd[p + "mlp.gate_proj.weight"] = _t(W.lin(mo.LLM, l, mo.GATE_W, ff, d))
        sd[p + "mlp.up_proj.weight"] = _t(W.lin(mo.LLM, l, mo.UP_W, ff, d))
        sd[p + "mlp.down_proj.weight"] = _t(W.lin(mo.LLM, l, mo.DOWN_W, d, ff))
        sd[p + "input_layernorm.weight"] = torch.ones(d)
        sd[p + "post_attention_layernorm.weight"] = torch.ones(d)
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected and all("inv_freq" in m for m in missing), (missing, unexpected)


def _hf_pixel_order(tokens: int, patches: np.ndarray, window: int) -> np.ndarray:
    """Our window-major patch rows -> the HF processor's raster order (merge
    groups of 2x2 patches contiguous, groups row-major over the merged grid)."""
    _, _, out_row = mo.item_plan(tokens, window)
    hf_rows = np.empty_like(patches)
    for j, r in enumerate(out_row):
        hf_rows[4 * r:4 * r + 4] = patches[4 * j:4 * j + 4]
    return hf_rows


@pytest.mark.parametrize("which,depth,sizes", [
    ("tiny", 4, [64, 60, 7]),          # full tiny depth; 8x8, 6x10 (edge windows), 1x7
    ("qwen7b", 2, [64, 20]),           # 7B ViT widths (1280 / 16 x 80 / 3420, merger -> 3584)
])
def test_vision_tower_matches_hf(which, depth, sizes):
    c = getattr(mo.ModelConfig, which)(vit_layers=depth, **({"vit_fullatt_every": 2} if which == "qwen7b" else {}))
    W = mo.Weights(c)
    vis = mo.VisionOracle(c, W)
    items = [(n, vis.patches(3, 1, i, n)) for i, n in enumerate(sizes)]
    ours = vis.encode(items)
    torch.manual_seed(0)
    model = hf.Qwen2_5_VisionTransformerPretrainedModel(_vision_cfg(c, depth)).eval()
    model.config._attn_implementation = "eager"
    _load_vision(model, c, W, depth)
    pix = np.concatenate([_hf_pixel_order(n, p, c.vit_window) for n, p in items])
    grid = torch.tensor([[1, 2 * gh, 2 * gw] for gh, gw in (mo.item_grid(n) for n in sizes)])
    with torch.no_grad():
        out = model(_t(pix), grid_thw=grid).pooler_output.numpy()
    assert out.shape == ours.shape
    assert _rel(ours, out) <= RTOL, f"vision tower: rel err {_rel(ours, out):.3g}"


def _rope_index_hf(segments):
    """HF get_rope_index on a synthetic prompt: text ids 1, image tokens
    typed 1 with their (1, 2gh, 2gw) grids.

    tokens_per_second=1: v5.5's get_vision_position_ids sets an image's
    temporal id to start_position * time_interval (time_interval =
    tokens_per_second for images); Qwen2.5-VL's published rule (and v4.x
    get_rope_index: t_index * second_per_grid_t * tokens_per_second + st_idx
    with t_index = 0 for a single-frame image) gives start_position. With
    tokens_per_second = 1 both read the same, so the comparison pins the
    model's semantics rather than that multiplication."""
    vcfg = Qwen2_5_VLVisionConfig(depth=1, hidden_size=32, num_heads=2, intermediate_size=32,
                                  out_hidden_size=32, tokens_per_second=1)
    tcfg = Qwen2_5_VLTextConfig(vocab_size=16, hidden_size=32, intermediate_size=32,
                                num_hidden_layers=1, num_attention_heads=2, num_key_value_heads=1,
                                rope_parameters={"rope_type": "default", "rope_theta": 1e6,
                                                 "mrope_section": [2, 3, 3]})
    model = hf.Qwen2_5_VLModel(Qwen2_5_VLConfig(vision_config=vcfg.to_dict(), text_config=tcfg.to_dict()))
    ttype, grids = [], []
    for kind, n in segments:
        ttype += [0 if kind == "T" else 1] * n
        if kind == "M":
            gh, gw = mo.item_grid(n)
            grids.append([1, 2 * gh, 2 * gw])
    ids = torch.ones(1, len(ttype), dtype=torch.long)
    pos, _ = model.get_rope_index(ids, torch.tensor([ttype], dtype=torch.int32),
                                  image_grid_thw=torch.tensor(grids) if grids else None)
    return pos[:, 0, :].T.numpy()


# HF groups adjacent image tokens into one run (real prompts separate images
# with <|vision_start|>/<|vision_end|> text tokens), so the layouts compared
# here keep text between items.
@pytest.mark.parametrize("layout", ["T64|M256|T1|M256|T32|M256|T2|M256", "T128|M1024|T32|M1024|T32",
                                    "M60|T5|M7|T3", "T40|M64|T8", "M12|T1|M1024"])
def test_mrope_positions_match_hf_get_rope_index(layout):
    segs = mo.parse_layout(layout)
    np.testing.assert_array_equal(mo.mrope_positions(segs), _rope_index_hf(segs))


@pytest.mark.parametrize("which,layers,layout", [
    ("tiny", 4, "T64|M256|T32|M60"),       # full tiny depth, oracle request embeddings
    ("qwen7b", 1, "T24|M64|T16|M20|T8"),   # 7B LLM widths: 3584, 28 q / 4 kv x 128, ff 18944
])
def test_decoder_and_head_match_hf(which, layers, layout):
    kw = {"vocab": 2048} if which == "qwen7b" else {}
    c = getattr(mo.ModelConfig, which)(llm_layers=layers, **kw)
    W = mo.Weights(c)
    segs = mo.parse_layout(layout)
    T = sum(n for _, n in segs)
    if which == "tiny":
        emb = mo.request_embeddings(c, W, 0, layout, 7, 256)
    else:  # embeddings of the 7B-width vision tower are checked above; use N(0, 1)
        emb = np.random.default_rng(1).standard_normal((T, c.llm_dim)).astype(np.float32)
    pos3 = mo.mrope_positions(segs)
    llm = mo.LlmOracle(c, W)
    ours = llm.forward(emb, pos3)
    ours_normed = mo.rmsnorm(ours, np.ones(c.llm_dim, dtype=np.float32), c.rms_eps)
    ours_logits = llm.first_token_logits(ours[-1])
    torch.manual_seed(0)
    model = hf.Qwen2_5_VLTextModel(_text_cfg(c, layers)).eval()
    model.config._attn_implementation = "eager"
    _load_text(model, c, W, layers)
    pos_hf = torch.from_numpy(_rope_index_hf(segs).T.copy())[:, None, :]  # [3, 1, T]
    with torch.no_grad():
        h = model(inputs_embeds=_t(emb)[None], position_ids=pos_hf, use_cache=False).last_hidden_state[0]
    h = h.numpy()
    assert _rel(ours_normed, h) <= RTOL, f"decoder: rel err {_rel(ours_normed, h):.3g}"
    logits_hf = h[-1] @ W.lin(mo.TOP, 0, mo.HEAD, c.vocab, c.llm_dim).T
    assert _rel(ours_logits, logits_hf) <= RTOL
    assert int(ours_logits.argmax()) == int(logits_hf.argmax())
