"""The asynchronous C-ABI seam driven by the reference's own event loop.

tests/native/capi_async_driver.cpp (built by the csrc Makefile) runs
lmmsim::PipelineEngine — the Simulation handler structure of the reference
(simengine.hpp:275-441) — with an ExecutionBackend that reaches the device
ONLY through include/rserve.h's non-blocking calls (rs_request_create_segments,
rs_encode_batch_async, rs_embeddings_ready, rs_prefill_chunk_async,
rs_release_async, rs_request_erase_async) and rs_poll. Its decision log must
equal the reference's run_simulation byte for byte, its first-token logits
must equal the device engine's (rs_engine_run) on the same inputs, and every
launch's completion must come back from rs_poll exactly once, in time order.
"""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "paper_2509_24381_b200", "_lib", "capi_async_driver")

WORKLOADS = {
    "cfg1": "0,0,-,T64|M256|M256|T32|M256|M256\n",
    "three": "0,0,-,T64|M256|M256|T32\n1,3.5,-,T40|M64|T8\n2,4,-,M128|T16|M60|T3\n",
}


@pytest.mark.parametrize("wl,policy,C,B", [("cfg1", 3, 256, 512), ("three", 3, 256, 384),
                                           ("three", 2, 256, 256), ("three", 1, 512, 512),
                                           ("three", 0, 256, 512)])
def test_reference_event_loop_over_async_c_abi(tmp_path, wl, policy, C, B):
    if not os.path.exists(DRIVER):
        pytest.fail("capi_async_driver not built (make -C paper_2509_24381_b200/csrc)")
    f = tmp_path / "wl.txt"
    f.write_text(WORKLOADS[wl])
    out = subprocess.run([DRIVER, str(f), str(policy), str(C), str(B), "7"], capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-3000:]
    j = json.loads(out.stdout.strip().splitlines()[-1])
    assert j["decisions_equal"], out.stderr[-4000:]
    assert j["logits_present"] and j["argmax_equal"]
    assert j["logits_max_abs_diff"] == 0.0, j
    assert j["events_ordered"] and j["events_once"] and j["events_complete"], j
    assert j["chunk_complete_events"] >= 1


def test_async_seam_errors_and_poll():
    """Reference error classes through the async calls; rs_poll reports each
    launch once, STAGE_DONE + CHUNK_COMPLETE for a chunk that ends a prompt."""
    import numpy as np
    import torch
    from paper_2509_24381_b200 import _native as N
    from paper_2509_24381_b200 import api
    p = api.Pipeline(api.model_preset("tiny"), max_prompt_tokens=4096, slot_tokens=8192, kv_tokens=8192,
                     max_chunk_tokens=1024, max_encode_tokens=512)
    with pytest.raises(N.ConfigError, match="segment token_count must be >= 1"):
        p.request_create_segments(1, [("T", 4), ("M", 0)])  # request.hpp:94-102 validate
    p.request_create_segments(1, [("T", 16), ("M", 64), ("T", 8)])
    with pytest.raises(N.RegistryError, match="duplicate request id 1"):
        p.request_create_segments(1, [("T", 4)])
    with pytest.raises(N.InputError, match="unknown encode tag"):
        p.embeddings_ready(99)
    px = torch.randn(4 * 64, 1176, device="cuda").to(torch.bfloat16)
    p.encode_batch_async(1, [(16, 80)], px.data_ptr(), on_host=False, tag=5)
    with pytest.raises(N.DependencyViolation):
        p.prefill_chunk_async([(1, 0, 40)], tag=6)  # the item is not ready yet
    ev = p.poll(wait=True)
    assert [(k, t) for k, _, t, _ in ev] == [(N.EV_ENCODE_DONE, 5)]
    p.embeddings_ready(5)
    with pytest.raises(N.InputError, match="unknown encode tag"):
        p.embeddings_ready(5)
    p.prefill_chunk_async([(1, 0, 40)], tag=7)
    p.prefill_chunk_async([(1, 40, 88)], tag=8)
    got = []
    while len(got) < 3:
        got += p.poll(wait=True)
    assert [(k, t) for k, _, t, _ in got] == [(N.EV_STAGE_DONE, 7), (N.EV_STAGE_DONE, 8),
                                             (N.EV_CHUNK_COMPLETE, 8)]
    assert got[0][3] <= got[1][3] == got[2][3]
    logits, am = p.logits(1)
    assert np.isfinite(logits).all() and 0 <= am < 4096
    with pytest.raises(N.InternalError, match="out-of-order release"):
        p.release_async(1, 40, 88, after_tag=8)
    p.release_async(1, 0, 88, after_tag=8)
    p.erase_async(1, after_tag=8)
    assert p.poll() == []
    p.close()
