"""Runs one tcgen05 GEMM shape a few times (for ncu captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import _native as N  # noqa: E402

M, Nn, K, epi, bn = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (2048, 37888, 3584, 2, 256)))
A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
B = torch.randn(Nn, K, device="cuda", dtype=torch.bfloat16) * 0.02
nc = Nn // 2 if epi == 2 else Nn
C = torch.empty(M, nc, device="cuda", dtype=torch.bfloat16)
for _ in range(4):
    N.check(N.lib.rs_op_gemm(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), nc, None,
                             C.data_ptr() if epi == 1 else None, nc if epi == 1 else 0, None,
                             M, Nn, K, epi, bn, torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
if os.environ.get("ONE_GEMM_TIME"):
    st = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        N.check(N.lib.rs_op_gemm(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), nc, None,
                                 C.data_ptr() if epi == 1 else None, nc if epi == 1 else 0, None,
                                 M, Nn, K, epi, bn, st))
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    print(f"gemm {M}x{Nn}x{K} epi{epi} bn{bn} streamk={os.environ.get('RS_GEMM_STREAMK', '1')}: "
          f"{us:.1f} us, {2 * M * Nn * K / us / 1e6:.0f} TFLOP/s")
