"""Runs the ViT full attention (tcgen05 ping-pong, varlen) on one 896x896
image (4096 patches, 16 heads, hd 80) a few times (for ncu captures)."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import _native as N  # noqa: E402

heads, hd, lens = 16, 80, [4096]
total = sum(lens)
qkv = torch.randn(total, 3 * heads * hd, device="cuda", dtype=torch.bfloat16)
cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32, device="cuda")
out = torch.empty(total, heads * hd, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    N.check(N.lib.rs_op_attention_varlen_tc(qkv.data_ptr(), qkv.stride(0), out.data_ptr(), out.stride(0),
                                            cu.data_ptr(), len(lens), total, heads, hd, 1 / math.sqrt(hd), st))
torch.cuda.synchronize()
