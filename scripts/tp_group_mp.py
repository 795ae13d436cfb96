"""One rank of a cross-process TP group: launched once per rank
(torch.distributed env: RANK / WORLD_SIZE / MASTER_*), each process creates
its TP-group context on cuda:(LOCAL_RANK % device_count) — on an NVSwitch box
one GPU per rank, on a one-GPU box all ranks share it — exports its exchange
buffer's CUDA IPC handle, all-gathers the handles over gloo, opens its peers'
buffers (cudaIpcOpenMemHandle) and runs the chunked prefill of one request
whose embeddings come from a loopback-TP reference context on the same
device. Rank 0 prints one JSON line: logits bit-equal to the loopback TP
context, residual streams bit-equal across ranks.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/tp_group_mp.py
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_24381_b200 import api  # noqa: E402

LAYOUT = "T16|M64|T8"
CHUNKS = [(0, 40), (40, 88)]


def main():
    dist.init_process_group("gloo")
    rank, T = dist.get_rank(), dist.get_world_size()
    dev = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    model = api.model_preset(os.environ.get("TP_MODEL", "tiny"))
    # reference: the loopback shards of one context (every rank builds it: same bytes)
    ref = api.Pipeline(model, device=dev, max_prompt_tokens=4096, slot_tokens=8192, kv_tokens=8192,
                       max_chunk_tokens=512, max_encode_tokens=512, tp_size=T)
    g = torch.Generator(device="cuda").manual_seed(11)
    px = torch.randn(4 * 64, 1176, device="cuda", generator=g).to(torch.bfloat16)
    ref.request_create(1, LAYOUT)
    ref.mark_encoded(1, 16, 80, ref.encode([(16, 80)], px.data_ptr(), on_host=False))
    emb = ref.read_slots(1, 0, 88)
    for b, e in CHUNKS:
        ref.prefill_chunk([(1, b, e)])
    ref_logits, ref_am = ref.logits(1)
    ref.close()
    r = api.Pipeline(model, device=dev, max_prompt_tokens=4096, slot_tokens=64, kv_tokens=8192,
                     max_chunk_tokens=512, max_encode_tokens=64, with_vit=False, tp_size=T, tp_rank=rank,
                     tp_group=True)
    _, handle = r.tp_buffer()
    hs = [None] * T
    dist.all_gather_object(hs, handle)
    r.tp_connect([None] * T, hs)  # every peer through its IPC handle (own buffer: local)
    r.kv_request_create(1, LAYOUT)
    e = torch.from_numpy(emb.view(np.int16)).view(torch.bfloat16).cuda()
    xs = []
    for b, en in CHUNKS:
        x = e[b:en].clone()
        r.tp_prefill([(1, b, en)], x.data_ptr())
        xs.append(x)
    torch.cuda.synchronize()
    logits, am = r.tp_logits(1)
    digest = [x.view(torch.int16).cpu().numpy().tobytes() for x in xs]
    all_d = [None] * T
    dist.all_gather_object(all_d, digest)
    ok_logits = bool(np.array_equal(logits, ref_logits) and am == ref_am)
    oks = [None] * T
    dist.all_gather_object(oks, ok_logits)
    if rank == 0:
        print(json.dumps({"ranks": T, "devices": torch.cuda.device_count(), "logits_equal_loopback": all(oks),
                          "residual_equal_across_ranks": all(d == all_d[0] for d in all_d), "argmax": am}))
    r.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
