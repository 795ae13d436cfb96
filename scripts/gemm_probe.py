"""Steady-state timing of the tcgen05 GEMM at the cfg2 shapes: 50 launches back
to back on one stream (the way the model issues them: PDL overlaps each
launch's prologue with the previous one's tail), per tile choice and split
mode, with a correctness check of every variant against the first one.

  python scripts/gemm_probe.py [--quick]

bn > 0: single-CTA 128 x bn tiles; bn < 0: CTA-pair 256 x |bn| tiles; 0: the
heuristic. Modes: default env, RS_GEMM_PAIR_SPLIT=1 (split tails on pair
tiles), RS_GEMM_STREAMK=0 is process-wide and not toggled here.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import _native as N  # noqa: E402

SHAPES = [  # (M, N, K, epi, label)
    (4096, 1280, 1280, 1, "vit_o"), (4096, 1280, 3424, 1, "vit_down"), (4096, 3840, 1280, 0, "vit_qkv"),
    (4096, 6848, 1280, 2, "vit_gateup"), (4096, 1280, 1176, 0, "patch_embed"),
    (2048, 3584, 3584, 1, "llm_o"), (2048, 4608, 3584, 0, "llm_qkv"), (2048, 3584, 18944, 1, "llm_down"),
    (2048, 37888, 3584, 2, "llm_gateup"), (256, 3584, 18944, 1, "llm_down_m256"),
    (256, 37888, 3584, 2, "llm_gateup_m256"),
]
BNS = [0, 128, 160, 192, 224, 256, -128, -160, -192, -224, -256, -320]
WIDE = {"vit_o": [0, 160, -160, -320], "vit_down": [0, -160, -320], "vit_qkv": [0, -224, -320],
        "llm_o": [0, -224, -256, -448, -512], "llm_down": [0, -224, -256, -448, -512],
        "llm_gateup": [0, -256, -512]}


SMALL_M = [(m, n, k, e, f"{lab}_m{m}") for m in (128, 256)
           for n, k, e, lab in ((4608, 3584, 0, "qkv"), (3584, 3584, 1, "o"), (37888, 3584, 2, "gateup"),
                                (3584, 18944, 1, "down"))]


def main():
    shapes = [x for x in SHAPES if x[4] in WIDE] if "--wide" in sys.argv else SHAPES[:3] if "--quick" in sys.argv else SMALL_M if "--small-m" in sys.argv else SHAPES
    st = torch.cuda.current_stream()
    res = []
    for M, Nn, K, epi, label in shapes:
        A = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        B = torch.randn(Nn, K, device="cuda", dtype=torch.bfloat16) * 0.02
        nc = Nn // 2 if epi == 2 else Nn
        C = torch.empty(M, nc, device="cuda", dtype=torch.bfloat16)
        R = torch.randn(M, nc, device="cuda", dtype=torch.bfloat16) if epi == 1 else None
        ref = None
        for split in ("0", "1"):
            os.environ["RS_GEMM_PAIR_SPLIT"] = split
            for bn in (WIDE[label] if "--wide" in sys.argv else BNS):
                if epi == 2 and abs(bn) % 64 != 0:
                    continue
                if "--wide" in sys.argv and split == "1":
                    continue
                if split == "1" and bn > 0:
                    continue  # single-CTA tiles do not read the pair-split knob

                def run():
                    N.check(N.lib.rs_op_gemm(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), nc, None,
                                             R.data_ptr() if epi == 1 else None, nc if epi == 1 else 0,
                                             None, M, Nn, K, epi, bn, st.cuda_stream))
                run()
                torch.cuda.synchronize()
                out = C.float().clone()
                if ref is None:
                    ref = out
                err = ((out - ref).abs().max() / ref.abs().max().clamp_min(1e-6)).item()
                for _ in range(5):
                    run()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 50
                e0.record(st)
                for _ in range(reps):
                    run()
                e1.record(st)
                e1.synchronize()
                us = e0.elapsed_time(e1) / reps * 1e3
                tf = 2 * M * Nn * K / us / 1e6
                res.append({"shape": label, "M": M, "N": Nn, "K": K, "epi": epi, "bn": bn, "pair_split": split,
                            "us": round(us, 2), "tflops": round(tf), "maxrel_vs_first": round(err, 5)})
                print(f"{label:16s} {M:5d} {Nn:6d} {K:6d} bn{bn:5d} split{split}: {us:8.2f} us "
                      f"{tf:6.0f} TFLOP/s  dev {err:.1e}", flush=True)
    os.environ.pop("RS_GEMM_PAIR_SPLIT", None)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
