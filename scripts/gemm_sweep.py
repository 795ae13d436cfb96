"""Times the tcgen05 GEMM at the cfg2 model shapes for every tile choice
(bn > 0: single-CTA 128 x bn tiles; bn < 0: CTA-pair 256 x |bn| tiles; 0: the
heuristic) with CUDA events, inputs L2-cold (a 256 MB buffer is rewritten
between reps). Prints one line per (shape, tile) and a JSON summary."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import _native as N  # noqa: E402

SHAPES = [
    (4096, 3840, 1280, 0), (4096, 1280, 1280, 1), (4096, 6848, 1280, 2), (4096, 1280, 3424, 1),
    (1024, 5120, 5120, 3), (1024, 3584, 5120, 0), (4096, 1280, 1184, 0),
    (2048, 4608, 3584, 0), (2048, 3584, 3584, 1), (2048, 37888, 3584, 2), (2048, 3584, 18944, 1),
    (384, 4608, 3584, 0), (384, 37888, 3584, 2), (384, 3584, 18944, 1),
    (8192, 8192, 8192, 0),
]
BNS = [0, 128, 160, 192, 224, 256, -128, -160, -192, -224, -256]


def main():
    shapes = SHAPES
    if len(sys.argv) > 1 and sys.argv[1] == "--quick":
        shapes = SHAPES[:4] + SHAPES[7:11]
    if len(sys.argv) > 1 and sys.argv[1] == "--small-m":  # the first / last prefill chunks
        shapes = [(m, n, k, e) for m in (256, 128)
                  for n, k, e in ((4608, 3584, 0), (3584, 3584, 1), (37888, 3584, 2), (3584, 18944, 1))]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    res = []
    for M, Nn, K, epi in shapes:
        A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        B = torch.randn(Nn, K, device="cuda", dtype=torch.bfloat16) * 0.02
        nc = Nn // 2 if epi == 2 else Nn
        C = torch.empty(M, nc, device="cuda", dtype=torch.bfloat16)
        ref = None
        for bn in BNS:
            if epi == 2 and bn % 64 != 0:
                continue

            def run():
                N.check(N.lib.rs_op_gemm(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), nc, None,
                                         C.data_ptr() if epi == 1 else None, nc if epi == 1 else 0, None,
                                         M, Nn, K, epi, bn, st.cuda_stream))
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
            tf = 2 * M * Nn * K / us / 1e6
            if epi != 1:
                out = C.float()
                if ref is None:
                    ref = out
                ok = bool(torch.allclose(out, ref, rtol=2e-2, atol=2e-2))
            else:
                ok = None
            res.append({"M": M, "N": Nn, "K": K, "epi": epi, "bn": bn, "us": round(us, 1),
                        "tflops": round(tf), "agree": ok})
            print(f"{M:5d} {Nn:6d} {K:6d} epi{epi} bn{bn:5d}: {us:8.1f} us {tf:6.0f} TFLOP/s agree={ok}",
                  flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
