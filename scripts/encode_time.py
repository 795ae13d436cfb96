"""ViT encode of one 896x896 image (one Algorithm-1 batch, 4096 patches) on the
7B-shaped encoder, device time per encode over back-to-back reps (CUDA events
around the whole batch only), and the sum of its kernels' event times in a
separate profiled pass (gaps = the difference).

  python scripts/encode_time.py [reps]
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
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    pipe.encode([(0, 1024)], px.data_ptr(), on_host=False, out_ptr=out.data_ptr())
b.record()
torch.cuda.synchronize()
per = a.elapsed_time(b) / reps
N.check(N.lib.rs_profile_enable(1))
pipe.encode([(0, 1024)], px.data_ptr(), on_host=False, out_ptr=out.data_ptr())
torch.cuda.synchronize()
N.check(N.lib.rs_profile_enable(0))
prof = N.profile_drain()
ksum = sum(v["ms"] for v in prof.values())
print(json.dumps({"pdl": os.environ.get("RS_PDL", "1"), "encode_ms": round(per, 3), "kernel_ms_sum_profiled": round(ksum, 3),
                  "launches": sum(v["launches"] for v in prof.values())}))
pipe.close()
