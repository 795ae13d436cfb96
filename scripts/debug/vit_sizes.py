"""Encode single items of many token counts (non-square / prime merged grids)
and compare each with the fp32 oracle; reports the first failing size."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import model_oracle as mo  # noqa: E402
from paper_2509_24381_b200 import api  # noqa: E402

p = api.Pipeline(api.model_preset("tiny"), max_prompt_tokens=8192, slot_tokens=1 << 15, kv_tokens=1 << 15,
                 max_chunk_tokens=2048, max_encode_tokens=4096)
cfg = mo.ModelConfig.tiny()
w = mo.Weights(cfg)
vis = mo.VisionOracle(cfg, w)
sizes = [int(s) for s in sys.argv[1:]] or [250, 251, 257, 263, 277, 300, 307, 331, 349, 350, 1, 2, 3, 5, 7, 17]
for n in sizes:
    patches = vis.patches(3, 1, 0, n)
    pt = torch.from_numpy(patches).to(torch.bfloat16).cuda()
    out = torch.empty(n, cfg.llm_dim, dtype=torch.bfloat16, device="cuda")
    try:
        p.encode([(0, n)], pt.data_ptr(), on_host=False, out_ptr=out.data_ptr())
        torch.cuda.synchronize()
    except Exception as e:
        print(f"size {n} grid {mo.item_grid(n)}: FAILED {e}", flush=True)
        raise
    got = out.float().cpu().numpy()
    ref = vis.encode([(n, patches)])
    cos = ((got * ref).sum(1) / np.maximum(np.linalg.norm(got, axis=1) * np.linalg.norm(ref, axis=1), 1e-12)).min()
    print(f"size {n} grid {mo.item_grid(n)}: min cos {cos:.5f} maxerr {np.abs(got - ref).max():.4f}", flush=True)
