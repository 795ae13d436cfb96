"""Causal prefill attention at the cfg2 shape (28 q / 4 kv heads, hd 128):
our tcgen05 kernel (rs_op_attention_prefill over a paged cache) next to
torch's SDPA backends (cuDNN / flash) as library yardsticks, same FLOPs.

  python scripts/attn_compare.py [T] [reps]
"""
import math
import os
import sys

import torch
import torch.nn.functional as F

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import _native as N  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8576
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hq, hkv, hd = 28, 4, 128
flops = 2.0 * T * T * hq * hd  # causal: 4 T^2/2 per head-dim unit


def timeit(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def ours():
    pool = (T + 63) // 64
    pt = torch.arange(pool, device="cuda", dtype=torch.int32)
    kc = torch.randn(pool, hkv, 64, hd, device="cuda").bfloat16()
    vc = torch.randn(pool, hkv, hd, 64, device="cuda").bfloat16()
    ra = ((T + 255) // 256) * 256
    qkv = torch.randn(ra, (hq + 2 * hkv) * hd, device="cuda").bfloat16()
    out = torch.empty(T, hq * hd, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream

    def run():
        N.check(N.lib.rs_op_attention_prefill(qkv.data_ptr(), qkv.stride(0), ra, out.data_ptr(), out.stride(0), 0, T,
                                              kc.data_ptr(), vc.data_ptr(), pool, pt.data_ptr(), hq, hkv, hd,
                                              1 / math.sqrt(hd), st))
    return timeit(run)


def sdpa(backend):
    from torch.nn.attention import SDPBackend, sdpa_kernel
    q = torch.randn(1, hq, T, hd, device="cuda", dtype=torch.bfloat16)
    k = torch.randn(1, hkv, T, hd, device="cuda", dtype=torch.bfloat16)
    v = torch.randn(1, hkv, T, hd, device="cuda", dtype=torch.bfloat16)
    k, v = k.repeat_interleave(hq // hkv, 1), v.repeat_interleave(hq // hkv, 1)
    with sdpa_kernel([backend]):
        return timeit(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True))


res = {"ours_tcgen05": ours()}
from torch.nn.attention import SDPBackend  # noqa: E402
for name, be in (("sdpa_cudnn", SDPBackend.CUDNN_ATTENTION), ("sdpa_flash", SDPBackend.FLASH_ATTENTION)):
    try:
        res[name] = sdpa(be)
    except Exception as e:  # backend unavailable on this build
        res[name] = f"unavailable: {str(e)[:80]}"
for k, v in res.items():
    if isinstance(v, float):
        print(f"{k:14s} T={T}: {v * 1e3:8.1f} us  {flops / (v * 1e-3) / 1e12:6.0f} TFLOP/s")
    else:
        print(f"{k:14s} {v}")
