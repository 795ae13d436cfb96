"""Paged tcgen05 prefill attention over many (head_dim, heads, pos0, rows)
cases vs torch; reports the first failing case (run with CUDA_LAUNCH_BLOCKING=1)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import test_ops_gpu as t  # noqa: E402
from paper_2509_24381_b200 import _native as N  # noqa: E402

cases = [(64, 8, 2, 0, r) for r in (200, 1000, 2000, 2048, 2100, 2650, 4096)] + \
        [(64, 8, 2, p, r) for p, r in ((2000, 700), (1500, 1150), (63, 2600))] + \
        [(128, 28, 4, 0, r) for r in (2100, 4096)]
for c in cases:
    try:
        out, ref = t._paged_case(N, *c)
        err = (out.float() - ref).abs().max().item()
        print(c, "max err", err, flush=True)
    except Exception as e:
        print(c, "FAILED", e, flush=True)
        raise
