"""ViT encode of one 896x896 image (4096 patches, 32 layers: 28 window + 4
full) on the 7B-shaped encoder context, timed with CUDA events; the window
attention path is chosen by RS_VIT_WIN_TC (1 = tcgen05 kernel, 0 = mma.sync).
Used for A/B timing and ncu captures of win_attn_tc_kernel.

  python scripts/one_vit_window.py [reps]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import _native as N  # noqa: E402
from paper_2509_24381_b200 import api  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
m = api.model_preset("qwen2.5-vl-7b")
pipe = api.Pipeline(m, with_vit=True, with_lm_head=False, layer_begin=m.llm_layers, layer_end=m.llm_layers,
                    kv_tokens=0, slot_tokens=0, max_chunk_tokens=64, max_encode_tokens=1024,
                    max_prompt_tokens=4096)
px = (torch.randn(4096, 1176, device="cuda") * 0.5).to(torch.bfloat16)
out = torch.empty(1024, m.llm_dim, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    pipe.encode([(0, 1024)], px.data_ptr(), on_host=False, out_ptr=out.data_ptr())
torch.cuda.synchronize()
N.check(N.lib.rs_profile_enable(1))
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    pipe.encode([(0, 1024)], px.data_ptr(), on_host=False, out_ptr=out.data_ptr())
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
N.check(N.lib.rs_profile_enable(0))
prof = N.profile_drain()
ts.sort()
print(json.dumps({"win_tc": os.environ.get("RS_VIT_WIN_TC", "1"), "encode_ms_p50": ts[len(ts) // 2],
                  "classes": {k.split("|")[0]: round(v["ms"] / reps, 4) for k, v in prof.items()
                              if "attn" in k or "split" in k}}))
pipe.close()
