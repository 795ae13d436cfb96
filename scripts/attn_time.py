"""Times the tcgen05 prefill attention on one paged slice (dev tool):
python scripts/attn_time.py POS0 ROWS [REPS]. Prints mean kernel time (CUDA
events) and the per-(query tile, key tile) cost in SM clocks."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import _native as N  # noqa: E402

hd, hq, hkv = 128, 28, 4
pos0 = int(sys.argv[1]) if len(sys.argv) > 1 else 6272
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
T = pos0 + rows
pool = (T + 63) // 64
pt = torch.arange(pool, device="cuda", dtype=torch.int32)
kc = torch.randn(pool, hkv, 64, hd, device="cuda").bfloat16()
vc = torch.randn(pool, hkv, hd, 64, device="cuda").bfloat16()
ra = ((rows + 127) // 128) * 128
qkv = torch.randn(ra, (hq + 2 * hkv) * hd, device="cuda").bfloat16()
out = torch.empty(rows, hq * hd, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream


def run():
    N.check(N.lib.rs_op_attention_prefill(qkv.data_ptr(), qkv.stride(0), ra, out.data_ptr(),
                                          out.stride(0), pos0, rows, kc.data_ptr(), vc.data_ptr(),
                                          pool, pt.data_ptr(), hq, hkv, hd, 1 / math.sqrt(hd), st))


for _ in range(3):
    run()
torch.cuda.synchronize()
N.check(N.lib.rs_profile_enable(1))
for _ in range(reps):
    run()
torch.cuda.synchronize()
N.check(N.lib.rs_profile_enable(0))
prof = N.profile_drain()
ms = sum(v["ms"] for k, v in prof.items() if k.startswith("attn_prefill"))
us = ms / reps * 1e3  # CUDA events around each launch (profiling mode)
pairs = 0  # (128-row query tile, 128-key tile) pairs
for t0 in range(0, rows, 128):
    pairs += (pos0 + min(t0 + 128, rows) + 127) // 128
pairs *= hq
flops = 4 * hd * hq * sum(pos0 + i + 1 for i in range(rows))
print(f"pos0={pos0} rows={rows}: {us:.1f} us, {flops / us / 1e6:.0f} TFLOP/s, "
      f"{us * 1.9e3 * 148 / pairs:.0f} SM-clk per tile pair (at 1.9 GHz, 148 SMs)")
