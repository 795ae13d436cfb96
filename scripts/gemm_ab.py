"""Same-process A/B of GEMM tile choices (alternating rounds, so clock / cache state is shared):
python scripts/gemm_ab.py M N K EPI BN[,BN...] [ROUNDS]   (BN 0 = heuristic, < 0 = CTA pair)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import _native as N  # noqa: E402

M, Nn, K, epi = (int(x) for x in sys.argv[1:5])
bns = [int(x) for x in sys.argv[5].split(",")]
rounds = int(sys.argv[6]) if len(sys.argv) > 6 else 3
A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
B = torch.randn(Nn, K, device="cuda", dtype=torch.bfloat16) * 0.02
nc = Nn // 2 if epi == 2 else Nn
C = torch.empty(M, nc, device="cuda", dtype=torch.bfloat16)
R = torch.randn(M, nc, device="cuda", dtype=torch.bfloat16) if epi == 1 else None
st = torch.cuda.current_stream()


def t(bn, reps=50):
    def run():
        N.check(N.lib.rs_op_gemm(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), nc, None,
                                 R.data_ptr() if epi == 1 else None, nc if epi == 1 else 0,
                                 None, M, Nn, K, epi, bn, st.cuda_stream))
    for _ in range(5):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        run()
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


t(bns[0])
N.check(N.lib.rs_profile_enable(1))  # which tile the heuristic (bn 0) picks
t(0, reps=1)
torch.cuda.synchronize()
N.check(N.lib.rs_profile_enable(0))
picked = [k for k in N.profile_drain() if k.startswith("gemm_tcgen05|")]
res = {bn: [] for bn in bns}
for _ in range(rounds):
    for bn in bns:
        res[bn].append(t(bn))
print(f"{M}x{Nn}x{K} epi{epi} (heuristic {picked}): " + ", ".join(f"bn {bn}: {min(v):.2f} us (min of {rounds})" for bn, v in res.items()),
      flush=True)
