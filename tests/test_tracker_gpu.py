"""Device embedding tracker (K6 scatter + bitmap, K7 ready prefix, K8 text
gather, slot release) against the host tracker mirror and the reference
semantics (tracker.hpp:44-141). Bit-exact: bitmap words, schedulable counts,
scattered bytes and gathered text-embedding bytes."""
import random

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pipe():
    from paper_2509_24381_b200 import api
    p = api.Pipeline(api.model_preset("tiny"), max_prompt_tokens=8192, slot_tokens=1 << 15,
                     kv_tokens=1 << 14, max_chunk_tokens=1024, max_encode_tokens=1024,
                     with_vit=False)
    yield p
    p.close()


def _words(total, ready):
    w = np.zeros((total + 31) // 32, dtype=np.uint32)
    for i in np.flatnonzero(ready):
        w[i // 32] |= np.uint32(1 << (i % 32))
    return w


def _layout(rng):
    segs = []
    for _ in range(rng.randint(1, 8)):
        segs.append(("M" if rng.random() < 0.5 else "T", rng.randint(1, 200)))
    return segs


def test_tracker_randomized_vs_host(pipe):
    from oracle import model_oracle as mo
    rng = random.Random(7)
    weights = mo.Weights(mo.ModelConfig.tiny())
    d = 512
    for trial in range(40):
        segs = _layout(rng)
        layout = "|".join(f"{k}{n}" for k, n in segs)
        total = sum(n for _, n in segs)
        rid = 1000 + trial
        ntext = sum(n for k, n in segs if k == "T")
        ids = np.array([rng.randrange(4096) for _ in range(ntext)], dtype=np.int32)
        pipe.request_create(rid, layout, ids)
        ready = np.zeros(total, dtype=bool)
        items, pos = [], 0
        for k, n in segs:
            if k == "T":
                ready[pos:pos + n] = True
            else:
                items.append((pos, pos + n))
            pos += n
        np.testing.assert_array_equal(pipe.read_bitmap(rid, total), _words(total, ready))
        # text embeddings gathered from the vocab table, bit-exact
        tpos = np.flatnonzero(ready)
        if len(tpos):
            got = pipe.read_slots(rid, 0, total)[tpos]
            want = weights.embed_rows(ids).view(np.uint32) >> 16
            np.testing.assert_array_equal(got, want.astype(np.uint16))
        rng.shuffle(items)
        frontier = 0
        payload = {}
        for s, e in items:
            emb = torch.randn(e - s, d, device="cuda", dtype=torch.bfloat16)
            payload[s] = emb.cpu().view(torch.int16).numpy().view(np.uint16)
            pipe.mark_encoded(rid, s, e, emb.data_ptr())
            ready[s:e] = True
            np.testing.assert_array_equal(pipe.read_bitmap(rid, total), _words(total, ready))
            host, dev = pipe.schedulable(rid)
            run_end = frontier
            while run_end < total and ready[run_end]:
                run_end += 1
            assert host == dev == run_end - frontier
            if host and rng.random() < 0.5:
                n = rng.randint(1, host)
                a, b = pipe.advance_prefill(rid, n)
                assert (a, b) == (frontier, frontier + n)
                frontier += n
        for s, e in items:
            np.testing.assert_array_equal(pipe.read_slots(rid, s, e), payload[s])
        st = pipe.tracker_stats(rid)
        assert st["all_encoded"] == 1 and st["live"] == total
        pipe.erase(rid)


def test_tracker_errors_match_reference(pipe):
    from paper_2509_24381_b200 import _native as N
    emb = torch.zeros(700, 512, device="cuda", dtype=torch.bfloat16)
    pipe.request_create(5, "T100|M500|T50|M700")
    with pytest.raises(N.AlignmentError, match=r"request 5: encode range \[100,350\) does not cover one multimodal item"):
        pipe.mark_encoded(5, 100, 350, emb.data_ptr())
    pipe.mark_encoded(5, 100, 600, emb.data_ptr())
    with pytest.raises(N.DoubleEncodeError, match=r"request 5: range \[100,600\) already encoded"):
        pipe.mark_encoded(5, 100, 600, emb.data_ptr())
    assert pipe.schedulable(5) == (650, 650)
    with pytest.raises(N.DependencyViolation, match=r"advance of 651 tokens exceeds schedulable frontier \(650 at token 0\)"):
        pipe.advance_prefill(5, 651)
    assert pipe.advance_prefill(5, 512) == (0, 512)
    assert pipe.schedulable(5) == (138, 138)
    with pytest.raises(N.InternalError, match="out-of-order release"):
        pipe.release(5, 100, 200)
    pipe.release(5, 0, 512)
    st = pipe.tracker_stats(5)
    assert st["live"] == 650 - 512 and st["peak_live"] == 650
    with pytest.raises(N.InputError):
        pipe.read_slots(5, 0, 10)  # pages of released tokens went back to the pool
    with pytest.raises(N.RegistryError, match="duplicate request id 5"):
        pipe.request_create(5, "T10")
    with pytest.raises(N.RegistryError, match="unknown request id 99"):
        pipe.mark_encoded(99, 0, 10, emb.data_ptr())
    pipe.erase(5)


def test_rejected_prefill_chunk_leaves_trackers_untouched(pipe):
    """rs_prefill_chunk validates every slice before advancing any tracker
    (ADVICE r1): an oversized or not-ready chunk raises and the frontiers stay
    where they were, so a corrected retry succeeds."""
    from paper_2509_24381_b200 import _native as N
    pipe.request_create(61, "T100|M50|T20")
    pipe.request_create(62, "T1100")
    with pytest.raises(N.ConfigError, match="exceeds max_chunk_tokens"):
        pipe.prefill_chunk([(61, 0, 100), (62, 0, 1000)])
    with pytest.raises(N.DependencyViolation, match="exceeds schedulable frontier"):
        pipe.prefill_chunk([(62, 0, 500), (61, 0, 120)])
    assert pipe.tracker_stats(61)["frontier"] == 0 and pipe.tracker_stats(62)["frontier"] == 0
    pipe.prefill_chunk([(61, 0, 100), (62, 0, 500)])
    assert pipe.tracker_stats(61)["frontier"] == 100 and pipe.tracker_stats(62)["frontier"] == 500
    pipe.erase(61)
    pipe.erase(62)
