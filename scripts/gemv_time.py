"""Times the skinny GEMM (decode, M <= 8) at the 7B decode shapes with L2
flushed between reps (dev tool). Prints achieved weight-streaming GB/s."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import _native as N  # noqa: E402

SHAPES = [(4608, 3584, 0), (3584, 3584, 1), (37888, 3584, 2), (3584, 18944, 1)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for M in (1, 4):
    for Nn, K, epi in SHAPES:
        A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        B = torch.randn(Nn, K, device="cuda", dtype=torch.bfloat16) * 0.02
        nc = Nn // 2 if epi == 2 else Nn
        C = torch.empty(M, nc, device="cuda", dtype=torch.bfloat16)

        def run():
            N.check(N.lib.rs_op_gemm(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), nc, None,
                                     C.data_ptr() if epi == 1 else None, nc if epi == 1 else 0, None,
                                     M, Nn, K, epi, 0, st.cuda_stream))
        for _ in range(3):
            run()
        ts = []
        for _ in range(15):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            run()
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        us = ts[len(ts) // 2] * 1e3
        print(f"M={M} N={Nn} K={K} epi{epi}: {us:7.1f} us  {2 * Nn * K / us / 1e3:6.0f} GB/s", flush=True)
