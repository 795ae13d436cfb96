"""A/B in one process: the 256-row down projection with the heuristic tile vs forced variants (alternating)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import _native as N  # noqa: E402

M, Nn, K = 256, 3584, 18944
A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
B = torch.randn(Nn, K, device="cuda", dtype=torch.bfloat16) * 0.02
C = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
R = torch.randn(M, Nn, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream()


def t(bn, reps=50):
    def run():
        N.check(N.lib.rs_op_gemm(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), Nn, None, R.data_ptr(), Nn,
                                 None, M, Nn, K, 1, bn, st.cuda_stream))
    for _ in range(5):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        run()
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for r in range(3):
    print({bn: round(t(bn), 2) for bn in (0, 128, -160, -192)}, flush=True)
