"""ORACLE — test infrastructure only; never imported by the product path.

CPU fp32 restatement (numpy) of the model math behind the reference's cost
seam (encode_time_ms / stage_time_ms, proj/include/lmmsim/cost_model.hpp:
68-82): the Qwen2.5-VL-shaped vision encoder (patch embed, 2-D RoPE,
window / full attention, SwiGLU MLP, 2x2 patch merger) and the decoder LLM
(M-RoPE, GQA causal attention, SwiGLU MLP, final norm + LM head).

PARITY STATUS: the reference (lmmsim) contains no model arithmetic at all
("Numerical parity is unpinned by the reference"), so this
oracle cannot be pinned by reference golden vectors. It restates the public
Qwen2.5-VL architecture and is pinned to an independent implementation:
tests/test_oracle_hf.py loads these weights into Hugging Face transformers'
Qwen2.5-VL modules (v5.5: the whole vision tower incl. window permutation and
patch merger, get_rope_index, the text model + LM head) at tiny size (full
depth) and at 7B widths, and requires fp32 agreement to 1e-4 relative.
tests/test_model_oracle.py adds self-consistency (chunked == unchunked
prefill, encoder output independent of batch composition).

Synthetic values reproduce the device generators bit for bit:
  u = splitmix64(seed * G + stream * H + i) >> 40, scaled to [0, 1) with
  24 bits; value = bf16_rne((2u - 1) * scale)   (paper_2509_24381_b200/csrc/
  kernels.cuh mix64, elementwise.cu fill_uniform_kernel).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
G = np.uint64(0x9E3779B97F4A7C15)
H = np.uint64(0xD1B54A32D192ED03)
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)
WEIGHT_SCALE = np.float32(0.0346410162)
PIXEL_SCALE = np.float32(1.7320508076)

# tensor stream ids (paper_2509_24381_b200/csrc/model.cuh namespace wid)
VIT, MERGER, LLM, TOP = 1, 2, 3, 4
QKV_W, QKV_B, O_W, O_B, GATE_W, GATE_B, UP_W, UP_B, DOWN_W, DOWN_B = range(1, 11)
PATCH, FC1_W, FC1_B, FC2_W, FC2_B, EMBED, HEAD = range(11, 18)


def wid(comp: int, layer: int, t: int) -> int:
    return (comp << 32) | (layer << 8) | t


def mix64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed) * G + np.uint64(stream) * H + idx.astype(np.uint64)
        z = (z ^ (z >> np.uint64(30))) * C1
        z = (z ^ (z >> np.uint64(27))) * C2
        return z ^ (z >> np.uint64(31))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32)
    bias = np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))
    r = ((u + bias) & np.uint32(0xFFFF0000)).astype(np.uint32)
    return r.view(np.float32)


def uniform(seed: int, stream: int, rows: int, cols: int, scale: np.float32,
            row0: int = 0) -> np.ndarray:
    idx = (np.arange(row0, row0 + rows, dtype=np.uint64)[:, None] * np.uint64(cols)
           + np.arange(cols, dtype=np.uint64)[None, :])
    z = mix64(seed, stream, idx)
    u = (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
    return bf16_round((np.float32(2.0) * u - np.float32(1.0)) * scale)


def token_ids(seed: int, req_id: int, positions: np.ndarray, vocab: int) -> np.ndarray:
    z = mix64(seed, (6 << 32) | req_id, positions.astype(np.uint64))
    return (z % np.uint64(vocab)).astype(np.int64)


def pixel_stream(req: int, item: int) -> int:
    return (5 << 32) | (req << 12) | item


# ---------------------------------------------------------------------------
@dataclass
class ModelConfig:
    """Mirror of rs_model_config (include/rserve.h)."""
    vit_dim: int
    vit_layers: int
    vit_heads: int
    vit_ff: int
    vit_window: int
    vit_fullatt_every: int
    patch_dim: int
    llm_dim: int
    llm_layers: int
    llm_q_heads: int
    llm_kv_heads: int
    llm_head_dim: int
    llm_ff: int
    vocab: int
    rope_theta_llm: float = 1e6
    rope_theta_vit: float = 1e4
    rms_eps: float = 1e-6
    weight_seed: int = 20250928

    @staticmethod
    def tiny(**kw) -> "ModelConfig":
        base = dict(vit_dim=256, vit_layers=4, vit_heads=4, vit_ff=1024, vit_window=4,
                    vit_fullatt_every=2, patch_dim=1176, llm_dim=512, llm_layers=4,
                    llm_q_heads=8, llm_kv_heads=2, llm_head_dim=64, llm_ff=1536, vocab=4096)
        base.update(kw)
        return ModelConfig(**base)

    @staticmethod
    def qwen7b(**kw) -> "ModelConfig":
        base = dict(vit_dim=1280, vit_layers=32, vit_heads=16, vit_ff=3420, vit_window=4,
                    vit_fullatt_every=8, patch_dim=1176, llm_dim=3584, llm_layers=28,
                    llm_q_heads=28, llm_kv_heads=4, llm_head_dim=128, llm_ff=18944,
                    vocab=152064)
        base.update(kw)
        return ModelConfig(**base)

    @staticmethod
    def qwen72b_llm(**kw) -> "ModelConfig":
        """cfg5: the 7B's vision tower with a Qwen2.5-VL-72B-shaped LLM
        (product preset RS_MODEL_QWEN25VL_72B_LLM, include/rserve.h)."""
        base = dict(vit_dim=1280, vit_layers=32, vit_heads=16, vit_ff=3420, vit_window=4,
                    vit_fullatt_every=8, patch_dim=1176, llm_dim=8192, llm_layers=80,
                    llm_q_heads=64, llm_kv_heads=8, llm_head_dim=128, llm_ff=29568,
                    vocab=152064)
        base.update(kw)
        return ModelConfig(**base)

    def full_attention(self, layer: int) -> bool:
        e = self.vit_fullatt_every
        return e > 0 and layer % e == e - 1


# ---------------------------------------------------------------------------
# Layout helpers (restated from the product's batch planner; window-major
# patch order, Qwen2-VL get_rope_index positions).
def item_grid(tokens: int) -> Tuple[int, int]:
    best = 1
    h = 1
    while h * h <= tokens:
        if tokens % h == 0:
            best = h
        h += 1
    return best, tokens // best


def item_plan(tokens: int, window: int, grid: Optional[Tuple[int, int]] = None):
    """(pos_hw [P,2], windows [list of (start,end)], out_row [T]) of one item."""
    gh, gw = grid if grid is not None else item_grid(tokens)
    pos, wins, out_row = [], [], []
    p = 0
    for wy in range(0, gh, window):
        for wx in range(0, gw, window):
            y1, x1 = min(gh, wy + window), min(gw, wx + window)
            start = p
            for r in range(wy, y1):
                for c in range(wx, x1):
                    out_row.append(r * gw + c)
                    for dy in range(2):
                        for dx in range(2):
                            pos.append((2 * r + dy, 2 * c + dx))
                    p += 4
            wins.append((start, p))
    return np.array(pos, dtype=np.int64), wins, np.array(out_row, dtype=np.int64)


def mrope_positions(segments: Sequence[Tuple[str, int]],
                    grids: Optional[Sequence[Tuple[int, int]]] = None) -> np.ndarray:
    out = []
    cur = 0
    item = 0
    for kind, n in segments:
        if kind == "T":
            for _ in range(n):
                out.append((cur, cur, cur))
                cur += 1
        else:
            gh, gw = grids[item] if grids is not None else item_grid(n)
            item += 1
            for r in range(gh):
                for c in range(gw):
                    out.append((cur, cur + r, cur + c))
            cur += max(gh, gw)
    return np.array(out, dtype=np.int64)


def parse_layout(layout: str) -> List[Tuple[str, int]]:
    return [(f[0], int(f[1:])) for f in layout.split("|")]


# ---------------------------------------------------------------------------
def rmsnorm(x: np.ndarray, w: np.ndarray, eps: float) -> np.ndarray:
    var = np.mean(x.astype(np.float32) ** 2, axis=-1, keepdims=True)
    return (x / np.sqrt(var + np.float32(eps))).astype(np.float32) * w


def silu(x):
    return x / (np.float32(1.0) + np.exp(-x))


def gelu_erf(x):
    from scipy.special import erf
    return np.float32(0.5) * x * (np.float32(1.0) + erf(x / np.float32(math.sqrt(2.0)))).astype(np.float32)


def rotate(x: np.ndarray, ang: np.ndarray) -> np.ndarray:
    """x [..., hd] rotated with rotate_half pairs (i, i + hd/2); ang [..., hd/2]."""
    half = x.shape[-1] // 2
    c, s = np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)
    a, b = x[..., :half], x[..., half:]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)


def softmax(x: np.ndarray, axis=-1) -> np.ndarray:
    m = np.max(x, axis=axis, keepdims=True)
    e = np.exp(x - m)
    return e / np.sum(e, axis=axis, keepdims=True)


class Weights:
    """Lazily generated fp32 copies of the device's bf16 weights."""

    def __init__(self, cfg: ModelConfig):
        self.cfg = cfg
        self._cache: Dict[tuple, np.ndarray] = {}

    def _get(self, key, fn):
        if key not in self._cache:
            self._cache[key] = fn()
        return self._cache[key]

    def lin(self, comp, layer, t, rows, cols):
        seed = self.cfg.weight_seed
        return self._get((comp, layer, t), lambda: uniform(seed, wid(comp, layer, t), rows, cols,
                                                           WEIGHT_SCALE))

    def vec(self, comp, layer, t, n):
        return self.lin(comp, layer, t, 1, n)[0]

    def embed_rows(self, ids: np.ndarray) -> np.ndarray:
        c = self.cfg
        out = np.empty((len(ids), c.llm_dim), dtype=np.float32)
        for i, r in enumerate(ids):
            out[i] = uniform(c.weight_seed, wid(TOP, 0, EMBED), 1, c.llm_dim, WEIGHT_SCALE, row0=int(r))[0]
        return out

    def head_logits(self, h: np.ndarray, block: int = 8192) -> np.ndarray:
        c = self.cfg
        out = np.empty((h.shape[0], c.vocab), dtype=np.float32)
        for r0 in range(0, c.vocab, block):
            n = min(block, c.vocab - r0)
            w = uniform(c.weight_seed, wid(TOP, 0, HEAD), n, c.llm_dim, WEIGHT_SCALE, row0=r0)
            out[:, r0:r0 + n] = h @ w.T
        return out


# ---------------------------------------------------------------------------
class VisionOracle:
    def __init__(self, cfg: ModelConfig, weights: Optional[Weights] = None):
        self.c = cfg
        self.w = weights or Weights(cfg)

    def patches(self, payload_seed: int, req_id: int, item: int, tokens: int) -> np.ndarray:
        return uniform(payload_seed, pixel_stream(req_id, item), 4 * tokens, self.c.patch_dim,
                       PIXEL_SCALE)

    def encode(self, items: Sequence[Tuple], layers: Optional[int] = None,
               bf16_acts: bool = False) -> np.ndarray:
        """items: (tokens, patches [4*tokens, pdim][, grid (gh, gw)]) in batch
        order -> embeddings [sum tokens, d_llm] in LLM (row-major) order."""
        c, W = self.c, self.w
        rnd = bf16_round if bf16_acts else (lambda a: a)
        vd, hd, nh = c.vit_dim, c.vit_dim // c.vit_heads, c.vit_heads
        plans = [item_plan(it[0], c.vit_window, it[2] if len(it) > 2 else None) for it in items]
        items = [(it[0], it[1]) for it in items]
        x = np.concatenate([p for _, p in items]).astype(np.float32)
        pos = np.concatenate([pl[0] for pl in plans])
        P = x.shape[0]
        x = rnd(x @ W.lin(VIT, 0, PATCH, vd, c.patch_dim).T)
        quarter = hd // 4
        inv = (1.0 / (np.float32(c.rope_theta_vit) ** (np.arange(0, hd // 2, 2, dtype=np.float32)
                                                           / np.float32(hd // 2)))).astype(np.float32)
        ang = np.concatenate([pos[:, 0:1].astype(np.float32) * inv[None, :quarter],
                              pos[:, 1:2].astype(np.float32) * inv[None, :quarter]], axis=1)
        # sequences
        item_seqs, win_seqs, base = [], [], 0
        for (t, _), pl in zip(items, plans):
            item_seqs.append((base, base + 4 * t))
            win_seqs.extend([(base + a, base + b) for a, b in pl[1]])
            base += 4 * t
        ones = np.ones(vd, dtype=np.float32)
        n_layers = c.vit_layers if layers is None else layers
        for l in range(n_layers):
            xn = rnd(rmsnorm(x, ones, c.rms_eps))
            qkv = rnd(xn @ W.lin(VIT, l, QKV_W, 3 * vd, vd).T + W.vec(VIT, l, QKV_B, 3 * vd))
            q = qkv[:, :vd].reshape(P, nh, hd)
            k = qkv[:, vd:2 * vd].reshape(P, nh, hd)
            v = qkv[:, 2 * vd:].reshape(P, nh, hd)
            q = rnd(rotate(q, ang[:, None, :]))
            k = rnd(rotate(k, ang[:, None, :]))
            seqs = item_seqs if c.full_attention(l) else win_seqs
            att = np.empty((P, nh, hd), dtype=np.float32)
            for a, b in seqs:
                # batched BLAS matmuls over heads: [h, q, d] @ [h, d, k]
                qh = np.ascontiguousarray(q[a:b].transpose(1, 0, 2))
                kh = np.ascontiguousarray(k[a:b].transpose(1, 2, 0))
                vh = np.ascontiguousarray(v[a:b].transpose(1, 0, 2))
                s = np.matmul(qh, kh) / np.float32(math.sqrt(hd))
                att[a:b] = np.matmul(softmax(s), vh).transpose(1, 0, 2)
            att = rnd(att.reshape(P, vd))
            x = rnd(x + att @ W.lin(VIT, l, O_W, vd, vd).T + W.vec(VIT, l, O_B, vd))
            xn = rnd(rmsnorm(x, ones, c.rms_eps))
            g = xn @ W.lin(VIT, l, GATE_W, c.vit_ff, vd).T + W.vec(VIT, l, GATE_B, c.vit_ff)
            u = xn @ W.lin(VIT, l, UP_W, c.vit_ff, vd).T + W.vec(VIT, l, UP_B, c.vit_ff)
            h = rnd(silu(g) * u)
            x = rnd(x + h @ W.lin(VIT, l, DOWN_W, vd, c.vit_ff).T + W.vec(VIT, l, DOWN_B, vd))
        xn = rnd(rmsnorm(x, ones, c.rms_eps)).reshape(P // 4, 4 * vd)
        mi = 4 * vd
        h = rnd(gelu_erf(xn @ W.lin(MERGER, 0, FC1_W, mi, mi).T + W.vec(MERGER, 0, FC1_B, mi)))
        e = h @ W.lin(MERGER, 0, FC2_W, c.llm_dim, mi).T + W.vec(MERGER, 0, FC2_B, c.llm_dim)
        out = np.empty_like(e)
        row = 0
        for (t, _), pl in zip(items, plans):
            out[row + pl[2]] = e[row:row + t]
            row += t
        return out


class LlmOracle:
    def __init__(self, cfg: ModelConfig, weights: Optional[Weights] = None):
        self.c = cfg
        self.w = weights or Weights(cfg)

    def forward(self, emb: np.ndarray, pos3: np.ndarray, layers: Optional[int] = None,
                bf16_acts: bool = False, chunks: Optional[Sequence[int]] = None) -> np.ndarray:
        """Causal prefill of one request. emb [T, d], pos3 [T, 3] M-RoPE ids.
        chunks: optional chunk lengths (chunked prefill over a growing KV
        cache); the math must not depend on them. Returns the final hidden
        state (pre final norm) [T, d]."""
        c, W = self.c, self.w
        rnd = bf16_round if bf16_acts else (lambda a: a)
        T, d = emb.shape
        hq, hkv, hd = c.llm_q_heads, c.llm_kv_heads, c.llm_head_dim
        qkv_dim = (hq + 2 * hkv) * hd
        half = hd // 2
        inv = (1.0 / (np.float32(c.rope_theta_llm) ** (np.arange(0, hd, 2, dtype=np.float32)
                                                            / np.float32(hd)))).astype(np.float32)
        sec = np.zeros(half, dtype=np.int64)
        sec[hd // 8:hd // 8 + 3 * hd // 16] = 1
        sec[hd // 8 + 3 * hd // 16:] = 2
        ang = pos3[:, sec].astype(np.float32) * inv[None, :]  # [T, half]
        ones = np.ones(d, dtype=np.float32)
        bounds = [0]
        for n in (chunks or [T]):
            bounds.append(bounds[-1] + n)
        assert bounds[-1] == T
        x = emb.astype(np.float32).copy()
        n_layers = c.llm_layers if layers is None else layers
        for l in range(n_layers):
            wqkv = W.lin(LLM, l, QKV_W, qkv_dim, d)
            bqkv = W.vec(LLM, l, QKV_B, qkv_dim)
            wo = W.lin(LLM, l, O_W, d, hq * hd)
            wg = W.lin(LLM, l, GATE_W, c.llm_ff, d)
            wu = W.lin(LLM, l, UP_W, c.llm_ff, d)
            wd = W.lin(LLM, l, DOWN_W, d, c.llm_ff)
            kc = np.zeros((T, hkv, hd), dtype=np.float32)
            vc = np.zeros((T, hkv, hd), dtype=np.float32)
            for a, b in zip(bounds[:-1], bounds[1:]):
                xn = rnd(rmsnorm(x[a:b], ones, c.rms_eps))
                qkv = rnd(xn @ wqkv.T + bqkv)
                q = qkv[:, :hq * hd].reshape(b - a, hq, hd)
                k = qkv[:, hq * hd:(hq + hkv) * hd].reshape(b - a, hkv, hd)
                v = qkv[:, (hq + hkv) * hd:].reshape(b - a, hkv, hd)
                q = rnd(rotate(q, ang[a:b, None, :]))
                kc[a:b] = rnd(rotate(k, ang[a:b, None, :]))
                vc[a:b] = v
                g = hq // hkv
                kk = np.repeat(kc[:b], g, axis=1)
                vv = np.repeat(vc[:b], g, axis=1)
                qh = np.ascontiguousarray(q.transpose(1, 0, 2))
                s = np.matmul(qh, np.ascontiguousarray(kk.transpose(1, 2, 0))) / np.float32(math.sqrt(hd))
                mask = np.arange(b)[None, :] > np.arange(a, b)[:, None]
                s = np.where(mask[None], -np.inf, s)
                att = rnd(np.matmul(softmax(s), np.ascontiguousarray(vv.transpose(1, 0, 2)))
                          .transpose(1, 0, 2).reshape(b - a, hq * hd))
                x[a:b] = rnd(x[a:b] + att @ wo.T)
                xn = rnd(rmsnorm(x[a:b], ones, c.rms_eps))
                h = rnd(silu(xn @ wg.T) * (xn @ wu.T))
                x[a:b] = rnd(x[a:b] + h @ wd.T)
        return x

    def first_token_logits(self, hidden_last: np.ndarray) -> np.ndarray:
        c = self.c
        h = rmsnorm(hidden_last[None, :], np.ones(c.llm_dim, dtype=np.float32), c.rms_eps)
        return self.w.head_logits(h)[0]


# ---------------------------------------------------------------------------
def request_embeddings(cfg: ModelConfig, weights: Weights, req_id: int, layout: str,
                       payload_seed: int, c_tokens: int, bf16_acts: bool = False,
                       vit_layers: Optional[int] = None, payload=None) -> np.ndarray:
    """Input embeddings [T, d] of a request: text rows from the vocab table,
    multimodal rows from the vision encoder run on Algorithm-1 batches of
    >= c_tokens tokens (encoder_sched.hpp:48-74). `payload`: this request's
    resolved payload (oracle/payload.py) — item grids / pixel seeds / token ids."""
    segs = parse_layout(layout)
    vis = VisionOracle(cfg, weights)
    T = sum(n for _, n in segs)
    emb = np.zeros((T, cfg.llm_dim), dtype=np.float32)
    pos = 0
    text_pos = []
    items = []  # (item index, start, tokens)
    for kind, n in segs:
        if kind == "T":
            text_pos.extend(range(pos, pos + n))
        else:
            items.append((len(items), pos, n))
        pos += n
    if text_pos:
        tp = np.array(text_pos, dtype=np.int64)
        ids = (np.asarray(payload["text_ids"], dtype=np.int64) if payload is not None
               else token_ids(payload_seed, req_id, tp, cfg.vocab))
        emb[tp] = weights.embed_rows(ids)
    batch: List[Tuple[int, int, int]] = []
    acc = 0

    def flush():
        nonlocal batch, acc
        if not batch:
            return
        if payload is not None:
            ins = [(n, vis.patches(payload["item_seeds"][i], req_id, i, n), tuple(payload["item_grids"][i]))
                   for i, _, n in batch]
        else:
            ins = [(n, vis.patches(payload_seed, req_id, i, n)) for i, _, n in batch]
        out = vis.encode(ins, layers=vit_layers, bf16_acts=bf16_acts)
        r = 0
        for _, s, n in batch:
            emb[s:s + n] = out[r:r + n]
            r += n
        batch, acc = [], 0

    for it in items:
        batch.append(it)
        acc += it[2]
        if acc >= c_tokens:
            flush()
    flush()
    return emb
