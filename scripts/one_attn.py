"""Runs the tcgen05 prefill attention once per call (for ncu captures)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import _native as N  # noqa: E402

hd, hq, hkv, pos0, rows = 128, 28, 4, int(sys.argv[1]) if len(sys.argv) > 1 else 6528, 2048
T = pos0 + rows
pool = (T + 63) // 64
pt = torch.arange(pool, device="cuda", dtype=torch.int32)
kc = torch.randn(pool, hkv, 64, hd, device="cuda").bfloat16()
vc = torch.randn(pool, hkv, hd, 64, device="cuda").bfloat16()
ra = ((rows + 127) // 128) * 128
qkv = torch.randn(ra, (hq + 2 * hkv) * hd, device="cuda").bfloat16()
out = torch.empty(rows, hq * hd, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    N.check(N.lib.rs_op_attention_prefill(qkv.data_ptr(), qkv.stride(0), ra, out.data_ptr(),
                                          out.stride(0), pos0, rows, kc.data_ptr(), vc.data_ptr(),
                                          pool, pt.data_ptr(), hq, hkv, hd, 1 / math.sqrt(hd),
                                          torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
