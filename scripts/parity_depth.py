"""Where does the device's deviation from the fp32 oracle come from at full
depth? Runs the cfg2 request (or a layout given on the command line) on the
device and through the torch fp32 mirror of the oracle twice — pure fp32, and
with activations rounded to bf16 at the points the device stores them
(bf16_acts) — and prints the three pairwise max|dlogit|/std figures and the
embedding agreement. Checker code (oracle/) only outside the product path.

  python scripts/parity_depth.py [--layout L] [--llm-layers N] [--vit-layers N]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import model_oracle as mo  # noqa: E402
from oracle import model_oracle_torch as mt  # noqa: E402
from paper_2509_24381_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layout", default="T128|" + "|".join(["M1024|T32"] * 8))
ap.add_argument("--llm-layers", type=int, default=28)
ap.add_argument("--vit-layers", type=int, default=32)
ap.add_argument("--seed", type=int, default=1234)
ap.add_argument("--out", default=None)
a = ap.parse_args()

kw = dict(vit_layers=a.vit_layers, llm_layers=a.llm_layers)
if a.vit_layers < 8:
    kw["vit_fullatt_every"] = 2
pipe = api.Pipeline(api.model_preset("qwen2.5-vl-7b", **kw), max_prompt_tokens=24576,
                    slot_tokens=1 << 16, kv_tokens=1 << 16, max_chunk_tokens=2048, max_encode_tokens=1024)
sc = api.SimConfig(policy="rserve", stages=1, token_budget=2048, embedding_batch_tokens=1024,
                   hidden_size=3584, cost=api.CostModel(beta_enc_ms_per_token=0.01, delta_stage_ms_per_token=0.01))
pipe.run(f"0,0,-,{a.layout}\n", sc, clock="real", payload_seed=a.seed)
dev_logits, dev_am = pipe.logits(0)
cfg = mo.ModelConfig.qwen7b(**kw)
emb32, l32 = mt.first_token_logits(cfg, a.layout, a.seed, device="cuda")
emb16, l16 = mt.first_token_logits(cfg, a.layout, a.seed, device="cuda", bf16_acts=True)
l32, l16 = l32.cpu().numpy(), l16.cpu().numpy()


def e(x, r):
    return float(np.abs(x - r).max() / r.std())


out = {"layout": a.layout, "llm_layers": a.llm_layers, "vit_layers": a.vit_layers,
       "device_vs_fp32": e(dev_logits, l32), "device_vs_bf16acts": e(dev_logits, l16),
       "bf16acts_vs_fp32": e(l16, l32),
       "argmax": {"device": int(dev_am), "fp32": int(l32.argmax()), "bf16acts": int(l16.argmax())},
       "emb_bf16acts_vs_fp32_cos_min": float(torch.nn.functional.cosine_similarity(emb16, emb32, dim=1).min()),
       "emb_bf16acts_vs_fp32_maxrel": float((emb16 - emb32).abs().max() / emb32.abs().max())}
print(json.dumps(out))
if a.out:
    json.dump(out, open(a.out, "w"), indent=1)
pipe.close()
