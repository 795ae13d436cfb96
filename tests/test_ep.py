"""EP disaggregation host side (CPU): topology, control-message codec, and the
multi-process plumbing (per-link ncclUniqueId exchange, wire messages between
ranks, max-over-ranks timing) on a world-size-2 gloo group."""
import os
import socket

import pytest

from paper_2509_24381_b200 import api, ep_launch
from paper_2509_24381_b200 import _native as N


def test_topology_links_and_roles():
    assert api.ep_links(1, 1) == [(0, 1), (1, 0)]
    # 2+2: P0<->E0, P0<->E1, P0->P1, P1->P0
    assert api.ep_links(2, 2) == [(0, 2), (2, 0), (0, 3), (3, 0), (0, 1), (1, 0)]
    links = api.ep_links(4, 4)
    assert len(links) == 2 * 4 + 3 + 3
    assert all(0 <= a < 8 and 0 <= b < 8 and a != b for a, b in links)
    assert len(set(links)) == len(links)
    assert [api.ep_role(r, 4, 4) for r in range(8)] == \
        [("prefill", 0), ("prefill", 1), ("prefill", 2), ("prefill", 3),
         ("encoder", 0), ("encoder", 1), ("encoder", 2), ("encoder", 3)]
    assert [api.ep_stage_layers(s, 4, 28) for s in range(4)] == [(0, 7), (7, 14), (14, 21), (21, 28)]
    with pytest.raises(N.ConfigError):
        api.ep_links(1, 0)
    with pytest.raises(N.ConfigError):
        ep_launch.topology_for(3)
    assert ep_launch.topology_for(8) == (4, 4)


@pytest.mark.parametrize("text", [
    "STOP",
    "ENCODE slot=5 req=2 items=0:128-1152@0,1:1184-2208@4096",
    "ENCODE slot=0 req=18446744073709551615 items=3:0-1@12",
    "STAGE chunk=3 slices=7:0-128[T128|M1024],9:64-100[T100]",
    "STAGE chunk=0 slices=1:0-2048[T128|M1024|T32|M1024|T32|M1024|T32|M1024|T32]",
])
def test_ctrl_roundtrip(text):
    msg = api.ep_ctrl_pack(text)
    assert len(msg) == N.EP_CTRL_BYTES
    assert api.ep_ctrl_unpack(msg) == text


def test_ctrl_rejects_malformed():
    good = bytearray(api.ep_ctrl_pack("ENCODE slot=1 req=1 items=0:0-64@0"))
    with pytest.raises(N.DataError):
        api.ep_ctrl_unpack(bytes(32768))  # no magic
    bad = bytearray(good)
    bad[8] = 9  # unknown kind
    with pytest.raises(N.DataError):
        api.ep_ctrl_unpack(bytes(bad))
    bad = bytearray(good)
    bad[16] = 200  # payload length past the words written
    with pytest.raises(N.DataError):
        api.ep_ctrl_unpack(bytes(bad))
    with pytest.raises(N.DataError):
        api.ep_ctrl_unpack(bytes(good[:1024]))
    with pytest.raises(N.InputError):
        api.ep_ctrl_pack("HELLO")
    with pytest.raises(N.InputError):
        api.ep_ctrl_pack("STAGE chunk=0 slices=1:0-64[X64]")
    with pytest.raises(N.DataError):  # slice outside its request
        api.ep_ctrl_pack("STAGE chunk=0 slices=1:0-65[T64]")
    # a chunk whose slices overflow the 4096-word message is a config error
    many = ",".join(f"{i}:0-1[T1]" for i in range(900))
    with pytest.raises(N.ConfigError):
        api.ep_ctrl_pack(f"STAGE chunk=0 slices={many}")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        stages, encoders = ep_launch.topology_for(world)
        ids = ep_launch.share_link_ids(stages, encoders)
        # P0 -> E0: an ENCODE message crosses the process boundary as bytes
        if rank == 0:
            msg = api.ep_ctrl_pack("ENCODE slot=4 req=11 items=0:32-288@0")
            dist.send(torch.frombuffer(bytearray(msg), dtype=torch.uint8), dst=1)
            back = torch.zeros(N.EP_CTRL_BYTES, dtype=torch.uint8)
            dist.recv(back, src=1)
            reply = api.ep_ctrl_unpack(back.numpy().tobytes())
        else:
            buf = torch.zeros(N.EP_CTRL_BYTES, dtype=torch.uint8)
            dist.recv(buf, src=0)
            got = api.ep_ctrl_unpack(buf.numpy().tobytes())
            assert got == "ENCODE slot=4 req=11 items=0:32-288@0", got
            dist.send(torch.frombuffer(bytearray(api.ep_ctrl_pack("STOP")), dtype=torch.uint8), dst=0)
            reply = got
        t = ep_launch.max_over_ranks(10.0 + rank)
        q.put((rank, ids, reply, t, api.ep_role(rank, stages, encoders)))
    finally:
        dist.destroy_process_group()


def test_gloo_two_rank_ep_plumbing():
    """World 2 = the 1+1 EP layout: both ranks agree on the link ids, a wire
    message round-trips between processes, and timing reduces to the max."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        rank, ids, reply, t, role = q.get(timeout=180)
        out[rank] = (ids, reply, t, role)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][0] == out[1][0] and len(out[0][0]) == 2 * 128  # two links: P0->E0, E0->P0
    assert out[0][1] == "STOP"
    assert out[0][2] == out[1][2] == 11.0
    assert out[0][3] == ("prefill", 0) and out[1][3] == ("encoder", 0)
