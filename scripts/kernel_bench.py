"""Isolated micro-benchmarks of the hot kernels at cfg2 shapes (B200).

Each kernel is timed alone with CUDA events on the launching stream (warm-up,
median of reps); achieved TFLOP/s or GB/s vs MEASURED_PEAKS.json. Prints one
JSON object. Usage: python scripts/kernel_bench.py [--quick]
"""
import json
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_24381_b200 import _native as N  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1590.0, "hbm_gbs": 6650.0}


def timeit(fn, reps=20, warm=3):
    s = torch.cuda.current_stream()
    for _ in range(warm):
        fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in evs:
        a.record(s)
        fn()
        b.record(s)
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in evs)
    return t[len(t) // 2]


def gemm_case(M, N_, K, epi=0, bn=0):
    A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(N_, K, device="cuda", dtype=torch.bfloat16) * 0.02
    ncols = N_ // 2 if epi == 2 else N_
    C = torch.empty(M, ncols, device="cuda", dtype=torch.float32 if epi == 4 else torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream

    def run():
        N.check(N.lib.rs_op_gemm(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), ncols, None,
                                 C.data_ptr() if epi == 1 else None, ncols if epi == 1 else 0, None,
                                 M, N_, K, epi, bn, st))
    ms = timeit(run)
    tf = 2 * M * N_ * K / ms / 1e9
    ref = timeit(lambda: torch.matmul(A, B.t()))
    return {"M": M, "N": N_, "K": K, "epi": epi, "bn": bn, "ms": ms, "tflops": tf,
            "frac": tf / PEAK["bf16_tflops"], "cublas_tflops": 2 * M * N_ * K / ref / 1e9}


def attn_case(lens, heads, hd):
    total = sum(lens)
    qkv = torch.randn(total, 3 * heads * hd, device="cuda", dtype=torch.bfloat16)
    cu = torch.tensor([0] + list(torch.tensor(lens).cumsum(0)), dtype=torch.int32, device="cuda")
    out = torch.empty(total, heads * hd, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream

    def run():
        N.check(N.lib.rs_op_attention_varlen(qkv.data_ptr(), qkv.stride(0), out.data_ptr(), out.stride(0),
                                             cu.data_ptr(), len(lens), max(lens), total, heads, hd,
                                             1 / math.sqrt(hd), st))
    ms = timeit(run)
    fl = sum(4 * n * n * hd * heads for n in lens)
    res = {"lens": f"{len(lens)}x{max(lens)}", "heads": heads, "hd": hd, "ms_mma_sync": ms,
           "tflops_mma_sync": fl / ms / 1e9}
    # tcgen05 path, measured with the profiler's per-kernel events (the op wrapper
    # allocates and synchronises around the kernels).
    N.check(N.lib.rs_profile_enable(1))
    for _ in range(5):
        N.check(N.lib.rs_op_attention_varlen_tc(qkv.data_ptr(), qkv.stride(0), out.data_ptr(),
                                                out.stride(0), cu.data_ptr(), len(lens), total,
                                                heads, hd, 1 / math.sqrt(hd), st))
    N.check(N.lib.rs_profile_enable(0))
    prof = N.profile_drain()
    a = prof["attn_vit_tcgen05"]
    res["ms_tcgen05"] = a["ms"] / a["launches"]
    res["tflops_tcgen05"] = fl / res["ms_tcgen05"] / 1e9
    return res


def prefill_case(hd, hq, hkv, pos0, rows):
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
    ms = timeit(run, reps=10)
    fl = 4 * hq * hd * sum(pos0 + i + 1 for i in range(rows))  # causal: keys <= position
    return {"prefill": f"ctx {pos0}+{rows}", "hq": hq, "hkv": hkv, "hd": hd, "ms": ms,
            "tflops": fl / ms / 1e9}


def main():
    out = {"gemm": [], "attention": []}
    for pos0 in (0, 2048, 6528):
        out["attention"].append(prefill_case(128, 28, 4, pos0, 2048))
    shapes = [
        # ViT (P = 4096 patches of one 896x896 image)
        (4096, 3840, 1280, 0), (4096, 1280, 1280, 1), (4096, 6848, 1280, 2), (4096, 1280, 3424, 1),
        (1024, 5120, 5120, 3), (1024, 3584, 5120, 0), (4096, 1280, 1176, 0),
        # LLM chunk (B = 2048 tokens)
        (2048, 4608, 3584, 0), (2048, 3584, 3584, 1), (2048, 37888, 3584, 2), (2048, 3584, 18944, 1),
        # big square sanity
        (8192, 8192, 8192, 0),
    ]
    for M, N_, K, epi in shapes if "--attn" not in sys.argv else []:
        for bn in (0, 128, 160, 192, 224, 256):
            out["gemm"].append(gemm_case(M, N_, K, epi, bn))
    out["attention"].append(attn_case([64] * 64, 16, 80))
    out["attention"].append(attn_case([4096], 16, 80))
    out["attention"].append(attn_case([2048], 28, 128))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
