"""ORACLE — test infrastructure only; never imported by the product path.

torch fp32 mirror of the numpy model oracle (oracle/model_oracle.py) so the
full-depth benched configuration (cfg2: Qwen2.5-VL-7B shapes, 32 ViT + 28
LLM layers, 8 images of 4096 patches, 8576 prompt tokens, ~172 TFLOP) can be
checked on the GPU box in seconds instead of CPU-hours. Same arithmetic, same
seeded weights (the splitmix64 generator restated on int64 tensors), fp32
throughout (TF32 disabled), so it is the same checker, just on another
device. tests/test_oracle_torch.py proves it equals the numpy oracle on CPU
at tiny size (full depth) and at 7B widths (1 ViT + 1 LLM layer); the numpy
oracle is in turn pinned to transformers' Qwen2.5-VL modules
(tests/test_oracle_hf.py).

Memory: weights are generated per layer and dropped after use (no 30 GB fp32
copy of the model); attention scores are formed per sequence / per KV-head
group.
"""
from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from oracle import model_oracle as mo


def _s64(u: int) -> int:
    """uint64 constant as the int64 with the same bits."""
    return u - (1 << 64) if u >= (1 << 63) else u


_G, _H = _s64(int(mo.G)), _s64(int(mo.H))
_C1, _C2 = _s64(int(mo.C1)), _s64(int(mo.C2))


def _srl(z: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def mix64(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """splitmix64 finaliser on int64 tensors (wrapping arithmetic), bit-equal
    to model_oracle.mix64 / csrc/kernels.cuh mix64."""
    base = _s64((seed * int(mo.G) + stream * int(mo.H)) & ((1 << 64) - 1))
    z = idx + base
    z = (z ^ _srl(z, 30)) * _C1
    z = (z ^ _srl(z, 27)) * _C2
    return z ^ _srl(z, 31)


def uniform(seed: int, stream: int, rows: int, cols: int, scale, row0: int = 0,
            device="cpu") -> torch.Tensor:
    idx = (torch.arange(row0, row0 + rows, dtype=torch.int64, device=device)[:, None] * cols
           + torch.arange(cols, dtype=torch.int64, device=device)[None, :])
    return _uniform_idx(seed, stream, idx, scale)


def _uniform_idx(seed, stream, idx, scale) -> torch.Tensor:
    z = mix64(seed, stream, idx)
    u = _srl(z, 40).to(torch.float32) * np.float32(1.0 / 16777216.0)
    return ((u * 2.0 - 1.0) * float(np.float32(scale))).to(torch.bfloat16).to(torch.float32)


def bf16_round(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


class Weights:
    """Per-call generation of the device's bf16 weights as fp32 tensors
    (optionally cached: the tiny model fits easily)."""

    def __init__(self, cfg: mo.ModelConfig, device="cpu", cache: bool = False):
        self.cfg = cfg
        self.device = device
        self.cache = {} if cache else None

    def lin(self, comp, layer, t, rows, cols):
        key = (comp, layer, t, rows, cols)
        if self.cache is not None and key in self.cache:
            return self.cache[key]
        w = uniform(self.cfg.weight_seed, mo.wid(comp, layer, t), rows, cols, mo.WEIGHT_SCALE,
                    device=self.device)
        if self.cache is not None:
            self.cache[key] = w
        return w

    def vec(self, comp, layer, t, n):
        return self.lin(comp, layer, t, 1, n)[0]

    def embed_rows(self, ids: torch.Tensor) -> torch.Tensor:
        c = self.cfg
        idx = ids.to(self.device, torch.int64)[:, None] * c.llm_dim + \
            torch.arange(c.llm_dim, dtype=torch.int64, device=self.device)[None, :]
        return _uniform_idx(c.weight_seed, mo.wid(mo.TOP, 0, mo.EMBED), idx, mo.WEIGHT_SCALE)

    def head_logits(self, h: torch.Tensor, block: int = 8192) -> torch.Tensor:
        c = self.cfg
        out = torch.empty(h.shape[0], c.vocab, dtype=torch.float32, device=self.device)
        for r0 in range(0, c.vocab, block):
            n = min(block, c.vocab - r0)
            w = uniform(c.weight_seed, mo.wid(mo.TOP, 0, mo.HEAD), n, c.llm_dim, mo.WEIGHT_SCALE,
                        row0=r0, device=self.device)
            out[:, r0:r0 + n] = h @ w.T
        return out


def rmsnorm(x: torch.Tensor, eps: float) -> torch.Tensor:
    var = (x * x).mean(dim=-1, keepdim=True)
    return x / torch.sqrt(var + float(np.float32(eps)))


def rotate(x: torch.Tensor, c: torch.Tensor, s: torch.Tensor) -> torch.Tensor:
    half = x.shape[-1] // 2
    a, b = x[..., :half], x[..., half:]
    return torch.cat([a * c - b * s, b * c + a * s], dim=-1)


def gelu_erf(x):
    return 0.5 * x * (1.0 + torch.erf(x / math.sqrt(2.0)))


def _attend(q, k, v, scale):
    """q [h, n, d], k/v [h, m, d] -> [h, n, d] (fp32 softmax)."""
    s = torch.matmul(q, k.transpose(-1, -2)) * scale
    return torch.matmul(torch.softmax(s, dim=-1), v)


class VisionOracle:
    """Mirror of model_oracle.VisionOracle (encode)."""

    def __init__(self, cfg: mo.ModelConfig, weights: Weights):
        self.c, self.w = cfg, weights

    def patches(self, payload_seed, req_id, item, tokens):
        return uniform(payload_seed, mo.pixel_stream(req_id, item), 4 * tokens, self.c.patch_dim,
                       mo.PIXEL_SCALE, device=self.w.device)

    def encode(self, items: Sequence[Tuple], layers: Optional[int] = None,
               bf16_acts: bool = False) -> torch.Tensor:
        c, W, dev = self.c, self.w, self.w.device
        rnd = bf16_round if bf16_acts else (lambda a: a)
        vd, hd, nh = c.vit_dim, c.vit_dim // c.vit_heads, c.vit_heads
        plans = [mo.item_plan(it[0], c.vit_window, it[2] if len(it) > 2 else None) for it in items]
        x = torch.cat([it[1].to(dev, torch.float32) for it in items])
        pos = torch.from_numpy(np.concatenate([pl[0] for pl in plans])).to(dev)
        P = x.shape[0]
        x = rnd(x @ W.lin(mo.VIT, 0, mo.PATCH, vd, c.patch_dim).T)
        quarter = hd // 4
        inv = 1.0 / (torch.tensor(float(np.float32(c.rope_theta_vit)), device=dev)
                     ** (torch.arange(0, hd // 2, 2, dtype=torch.float32, device=dev) / float(hd // 2)))
        ang = torch.cat([pos[:, 0:1].float() * inv[None, :quarter],
                         pos[:, 1:2].float() * inv[None, :quarter]], dim=1)
        cos, sin = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
        item_seqs, win_seqs, base = [], [], 0
        for it, pl in zip(items, plans):
            item_seqs.append((base, base + 4 * it[0]))
            win_seqs.extend([(base + a, base + b) for a, b in pl[1]])
            base += 4 * it[0]
        # windows grouped by length -> one batched matmul per group
        win_groups = {}
        for a, b in win_seqs:
            win_groups.setdefault(b - a, []).append(a)
        win_groups = {n: torch.tensor(starts, device=dev) for n, starts in win_groups.items()}
        scale = 1.0 / math.sqrt(hd)
        n_layers = c.vit_layers if layers is None else layers
        for l in range(n_layers):
            xn = rnd(rmsnorm(x, c.rms_eps))
            qkv = rnd(xn @ W.lin(mo.VIT, l, mo.QKV_W, 3 * vd, vd).T + W.vec(mo.VIT, l, mo.QKV_B, 3 * vd))
            q = rnd(rotate(qkv[:, :vd].reshape(P, nh, hd), cos, sin))
            k = rnd(rotate(qkv[:, vd:2 * vd].reshape(P, nh, hd), cos, sin))
            v = qkv[:, 2 * vd:].reshape(P, nh, hd)
            att = torch.empty(P, nh, hd, dtype=torch.float32, device=dev)
            if c.full_attention(l):
                for a, b in item_seqs:
                    att[a:b] = _attend(q[a:b].transpose(0, 1), k[a:b].transpose(0, 1),
                                       v[a:b].transpose(0, 1), scale).transpose(0, 1)
            else:
                for n, starts in win_groups.items():
                    rows = (starts[:, None] + torch.arange(n, device=dev)[None, :]).reshape(-1)
                    g = len(starts)
                    qg = q[rows].reshape(g, n, nh, hd).permute(0, 2, 1, 3)
                    kg = k[rows].reshape(g, n, nh, hd).permute(0, 2, 1, 3)
                    vg = v[rows].reshape(g, n, nh, hd).permute(0, 2, 1, 3)
                    att[rows] = _attend(qg, kg, vg, scale).permute(0, 2, 1, 3).reshape(g * n, nh, hd)
            att = rnd(att.reshape(P, vd))
            x = rnd(x + att @ W.lin(mo.VIT, l, mo.O_W, vd, vd).T + W.vec(mo.VIT, l, mo.O_B, vd))
            xn = rnd(rmsnorm(x, c.rms_eps))
            g_ = xn @ W.lin(mo.VIT, l, mo.GATE_W, c.vit_ff, vd).T + W.vec(mo.VIT, l, mo.GATE_B, c.vit_ff)
            u = xn @ W.lin(mo.VIT, l, mo.UP_W, c.vit_ff, vd).T + W.vec(mo.VIT, l, mo.UP_B, c.vit_ff)
            h = rnd(torch.nn.functional.silu(g_) * u)
            del g_, u
            x = rnd(x + h @ W.lin(mo.VIT, l, mo.DOWN_W, vd, c.vit_ff).T + W.vec(mo.VIT, l, mo.DOWN_B, vd))
            del h, qkv, q, k, v, att
        xn = rnd(rmsnorm(x, c.rms_eps)).reshape(P // 4, 4 * vd)
        mi = 4 * vd
        h = rnd(gelu_erf(xn @ W.lin(mo.MERGER, 0, mo.FC1_W, mi, mi).T + W.vec(mo.MERGER, 0, mo.FC1_B, mi)))
        e = h @ W.lin(mo.MERGER, 0, mo.FC2_W, c.llm_dim, mi).T + W.vec(mo.MERGER, 0, mo.FC2_B, c.llm_dim)
        out = torch.empty_like(e)
        row = 0
        for it, pl in zip(items, plans):
            out[row + torch.from_numpy(pl[2]).to(dev)] = e[row:row + it[0]]
            row += it[0]
        return out


class LlmOracle:
    """Mirror of model_oracle.LlmOracle (forward + first_token_logits)."""

    def __init__(self, cfg: mo.ModelConfig, weights: Weights):
        self.c, self.w = cfg, weights

    def forward(self, emb: torch.Tensor, pos3, layers: Optional[int] = None,
                bf16_acts: bool = False, q_block: int = 4096) -> torch.Tensor:
        c, W, dev = self.c, self.w, self.w.device
        rnd = bf16_round if bf16_acts else (lambda a: a)
        T, d = emb.shape
        hq, hkv, hd = c.llm_q_heads, c.llm_kv_heads, c.llm_head_dim
        qkv_dim = (hq + 2 * hkv) * hd
        half = hd // 2
        inv = 1.0 / (torch.tensor(float(np.float32(c.rope_theta_llm)), device=dev)
                     ** (torch.arange(0, hd, 2, dtype=torch.float32, device=dev) / float(hd)))
        sec = np.zeros(half, dtype=np.int64)
        sec[hd // 8:hd // 8 + 3 * hd // 16] = 1
        sec[hd // 8 + 3 * hd // 16:] = 2
        pos3 = torch.as_tensor(np.asarray(pos3)).to(dev)
        ang = pos3[:, torch.from_numpy(sec).to(dev)].float() * inv[None, :]
        cos, sin = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
        x = emb.to(dev, torch.float32).clone()
        scale = 1.0 / math.sqrt(hd)
        grp = hq // hkv
        n_layers = c.llm_layers if layers is None else layers
        for l in range(n_layers):
            xn = rnd(rmsnorm(x, c.rms_eps))
            qkv = rnd(xn @ W.lin(mo.LLM, l, mo.QKV_W, qkv_dim, d).T + W.vec(mo.LLM, l, mo.QKV_B, qkv_dim))
            q = rnd(rotate(qkv[:, :hq * hd].reshape(T, hq, hd), cos, sin))
            k = rnd(rotate(qkv[:, hq * hd:(hq + hkv) * hd].reshape(T, hkv, hd), cos, sin))
            v = qkv[:, (hq + hkv) * hd:].reshape(T, hkv, hd)
            att = torch.empty(T, hq, hd, dtype=torch.float32, device=dev)
            for kv in range(hkv):
                kh, vh = k[:, kv], v[:, kv]                       # [T, hd]
                for a in range(0, T, q_block):
                    b = min(T, a + q_block)
                    qh = q[a:b, kv * grp:(kv + 1) * grp].transpose(0, 1)   # [grp, n, hd]
                    s = torch.matmul(qh, kh[:b].T) * scale                # [grp, n, b]
                    mask = torch.arange(b, device=dev)[None, :] > torch.arange(a, b, device=dev)[:, None]
                    s.masked_fill_(mask[None], float("-inf"))
                    att[a:b, kv * grp:(kv + 1) * grp] = torch.matmul(torch.softmax(s, dim=-1),
                                                                     vh[:b]).transpose(0, 1)
                    del s
            att = rnd(att.reshape(T, hq * hd))
            x = rnd(x + att @ W.lin(mo.LLM, l, mo.O_W, d, hq * hd).T)
            xn = rnd(rmsnorm(x, c.rms_eps))
            g = xn @ W.lin(mo.LLM, l, mo.GATE_W, c.llm_ff, d).T
            u = xn @ W.lin(mo.LLM, l, mo.UP_W, c.llm_ff, d).T
            h = rnd(torch.nn.functional.silu(g) * u)
            del g, u
            x = rnd(x + h @ W.lin(mo.LLM, l, mo.DOWN_W, d, c.llm_ff).T)
            del h, qkv, q, k, v, att
        return x

    def first_token_logits(self, hidden_last: torch.Tensor) -> torch.Tensor:
        return self.w.head_logits(rmsnorm(hidden_last[None, :], self.c.rms_eps))[0]


def request_embeddings(cfg: mo.ModelConfig, weights: Weights, req_id: int, layout: str,
                       payload_seed: int, bf16_acts: bool = False,
                       vit_layers: Optional[int] = None) -> torch.Tensor:
    """Input embeddings [T, d] of a request (text rows from the vocab table,
    MM rows from the vision encoder). All items are encoded in one pass: the
    encoder's output does not depend on batch composition (per-image /
    per-window attention; model_oracle.request_embeddings runs the
    Algorithm-1 batches and tests/test_model_oracle.py checks the two agree)."""
    segs = mo.parse_layout(layout)
    dev = weights.device
    T = sum(n for _, n in segs)
    emb = torch.zeros(T, cfg.llm_dim, dtype=torch.float32, device=dev)
    pos, text_pos, items = 0, [], []
    for kind, n in segs:
        if kind == "T":
            text_pos.extend(range(pos, pos + n))
        else:
            items.append((len(items), pos, n))
        pos += n
    if text_pos:
        tp = np.array(text_pos, dtype=np.int64)
        ids = torch.from_numpy(mo.token_ids(payload_seed, req_id, tp, cfg.vocab))
        emb[torch.from_numpy(tp).to(dev)] = weights.embed_rows(ids)
    if items:
        vis = VisionOracle(cfg, weights)
        out = vis.encode([(n, vis.patches(payload_seed, req_id, i, n)) for i, _, n in items],
                         layers=vit_layers, bf16_acts=bf16_acts)
        r = 0
        for _, s, n in items:
            emb[s:s + n] = out[r:r + n]
            r += n
    return emb


def first_token_logits(cfg: mo.ModelConfig, layout: str, payload_seed: int, req_id: int = 0,
                       device="cpu", bf16_acts: bool = False) -> Tuple[torch.Tensor, torch.Tensor]:
    """(embeddings [T, d], first-token logits [vocab]) of one request."""
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        with torch.no_grad():
            W = Weights(cfg, device=device)
            emb = request_embeddings(cfg, W, req_id, layout, payload_seed, bf16_acts=bf16_acts)
            llm = LlmOracle(cfg, W)
            h = llm.forward(emb, mo.mrope_positions(mo.parse_layout(layout)), bf16_acts=bf16_acts)
            return emb, llm.first_token_logits(h[-1])
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
