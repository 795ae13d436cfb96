"""Multi-item encode batches of odd sizes vs the fp32 oracle (CUDA_LAUNCH_BLOCKING=1)."""
import os
import random
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
rng = random.Random(5)
batches = [[250, 263], [251, 349, 300], [257, 257], [331, 1, 2, 350]] + \
          [[rng.randint(250, 350) for _ in range(rng.randint(1, 4))] for _ in range(12)]
if len(sys.argv) > 1:
    batches = [[int(x) for x in sys.argv[1].split(",")]]
for b in batches:
    items = [(n, vis.patches(3, 1, i, n)) for i, n in enumerate(b)]
    host = np.concatenate([x for _, x in items])
    pt = torch.from_numpy(host).to(torch.bfloat16).cuda()
    tot = sum(b)
    out = torch.empty(tot, cfg.llm_dim, dtype=torch.bfloat16, device="cuda")
    ranges, s = [], 0
    for n in b:
        ranges.append((s, s + n))
        s += n
    try:
        p.encode(ranges, pt.data_ptr(), on_host=False, out_ptr=out.data_ptr())
        torch.cuda.synchronize()
    except Exception as e:
        print(b, "FAILED", e, flush=True)
        raise
    got = out.float().cpu().numpy()
    ref = vis.encode(items)
    cos = ((got * ref).sum(1) / np.maximum(np.linalg.norm(got, axis=1) * np.linalg.norm(ref, axis=1), 1e-12)).min()
    print(b, f"min cos {cos:.5f}", flush=True)
