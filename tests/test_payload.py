"""Payload files: generation keyed by the workload seed,
validation errors in the reference's InputError style, and agreement of the
product's normalised form with the oracle's independent parser. Host only."""
import pytest

WL = "0,0,-,T64|M256|M256|T32|M256|M256\n1,3.5,-,T40|M64|T8\n2,7,-,M1024|T128\n"


@pytest.fixture(scope="module")
def api():
    from paper_2509_24381_b200 import api
    return api


def test_generate_is_deterministic_and_valid(api):
    a = api.generate_payload(WL, 11)
    assert a == api.generate_payload(WL, 11)
    assert a != api.generate_payload(WL, 12)
    assert api.validate_payload(WL, a, 4096) == a  # already normalised
    from oracle import payload
    spec = payload.parse(a)
    for rid, layout in ((0, "T64|M256|M256|T32|M256|M256"), (1, "T40|M64|T8"), (2, "M1024|T128")):
        segs = layout.split("|")
        for s, seg in enumerate(segs):
            if seg[0] == "M":
                gh, gw = spec[rid]["M"][s]["grid"]
                assert gh * gw == int(seg[1:]) and max(gh, gw) <= 4 * min(gh, gw)
            else:
                assert "seed" in spec[rid]["T"][s]


def test_normalised_form_round_trips(api):
    text = "# hand written\n1,2,T,ids=1 2 3 4 5 6 7 8\n1,1,M,seed=5;grid=8x8\n\n0,1,M,grid=16x16\n"
    norm = api.validate_payload(WL, text, 4096)
    assert norm.splitlines()[0] == "# rserve payload v1"
    assert api.validate_payload(WL, norm, 4096) == norm
    from oracle import payload
    assert payload.parse(norm) == payload.parse(text)


@pytest.mark.parametrize("text,msg", [
    ("0,1,M,grid=15x17\n", "grid 15x17 != 256 tokens"),
    ("0,0,M,grid=8x8\n", "segment 0 is not multimodal"),
    ("0,1,T,seed=3\n", "segment 1 is not text"),
    ("1,2,T,ids=1 2 3\n", "3 ids for 8 tokens"),
    ("1,2,T,ids=1 2 3 4 5 6 7 4096\n", "token id 4096 outside the vocabulary"),
    ("9,0,T,seed=1\n", "request 9 is not in the workload"),
    ("0,1,M\n", "payload line 1: expected 4 comma-separated fields"),
    ("0,1,M,grid=16x16\n0,1,M,seed=2\n", "payload line 2: duplicate segment"),
    ("0,1,X,seed=2\n", "segment kind must be T or M"),
    ("0,1,M,size=3\n", "unknown multimodal key 'size'"),
])
def test_validation_errors(api, text, msg):
    from paper_2509_24381_b200 import _native as N
    with pytest.raises(N.InputError, match=msg):
        api.validate_payload(WL, text, 4096)
