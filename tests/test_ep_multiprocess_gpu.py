"""EP across processes (one per rank) over the CUDA-IPC peer-memory
transport. On a one-GPU box every rank runs on cuda:0 — separate processes,
separate CUDA contexts, mailboxes mapped with cudaIpcOpenMemHandle — which is
the multi-GPU code path minus NVLink. Same bars as test_ep_gpu.py."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LAYOUTS = {0: "T64|M256|M256|T32|M256|M256", 1: "T40|M64|T8", 2: "M128|T16"}


@pytest.mark.parametrize("world", [2, 4])
def test_ep_ipc_processes(world, tmp_path):
    from oracle import model_oracle as mo
    out = tmp_path / "ep.json"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ep_multiprocess.py"), "--world",
                        str(world), "--same-device", "--transport", "ipc", "--json", str(out)],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    res = json.loads(out.read_text())
    assert res["exitcodes"] == [0] * world, r.stdout + r.stderr
    runs = {o["clock"]: o for rank, _, o in res["results"] if rank == 0}
    assert runs["lockstep"]["decisions_equal"]
    assert runs["real"]["gpu_ms"] > 0
    cfg = mo.ModelConfig.tiny()
    w = mo.Weights(cfg)
    llm = mo.LlmOracle(cfg, w)
    for rid, layout in LAYOUTS.items():
        emb = mo.request_embeddings(cfg, w, rid, layout, 7, 256)
        ref = llm.first_token_logits(llm.forward(emb, mo.mrope_positions(mo.parse_layout(layout)))[-1])
        for clock in ("lockstep", "real", "real_e2e"):
            got = np.asarray(runs[clock]["logits"][str(rid)], dtype=np.float32)
            assert np.abs(got - ref).max() <= 0.05 * ref.std()
