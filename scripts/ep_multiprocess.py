"""EP across processes, one per rank (gloo for plumbing), over the NCCL or
the CUDA-IPC transport.

    python scripts/ep_multiprocess.py [--world 2] [--same-device] [--transport ipc|nccl]

With --same-device every rank uses cuda:0 (a single-GPU box); NCCL refuses two
ranks of one communicator on one GPU, CUDA IPC does not.
"""
import argparse
import json
import os
import socket
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

WL = "0,0,-,T64|M256|M256|T32|M256|M256\n1,3.5,-,T40|M64|T8\n2,4,-,M128|T16\n"


def rank_main(rank, world, port, same, transport, q):
    import faulthandler
    faulthandler.dump_traceback_later(float(os.environ.get("RS_EP_WATCHDOG", "0")) or 1e9, exit=True)
    import torch.distributed as dist
    from paper_2509_24381_b200 import api, ep_launch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        stages, encoders = ep_launch.topology_for(world)
        dev = 0 if same else rank
        ids = ep_launch.share_link_ids(stages, encoders) if transport == "nccl" else None
        shm = ep_launch.shm_name_for_group() if transport == "ipc" else None
        m = api.model_preset("tiny")
        kw = dict(max_prompt_tokens=8192, slot_tokens=1 << 15, kv_tokens=1 << 15, max_chunk_tokens=2048,
                  max_encode_tokens=1024)
        ctx = api.ep_context(m, rank, stages, encoders, device=dev, **kw)
        print(f"rank {rank}: context ready", flush=True)
        t0 = time.time()
        g = api.EpGroup(stages, encoders, transport, rank=rank, device=dev, nccl_ids=ids,
                        slot_bytes=api.ep_slot_bytes(m, 2048, 1024), shm_name=shm)
        if transport == "ipc":
            ep_launch.connect_ipc(g)
        init_s = time.time() - t0
        print(f"rank {rank}: transport connected in {init_s:.2f}s", flush=True)
        sc = api.SimConfig(policy="rserve", stages=stages, encoder_workers=encoders, token_budget=384,
                           embedding_batch_tokens=256, hidden_size=512,
                           cost=api.CostModel(alpha_enc_ms=0.5, beta_enc_ms_per_token=0.01, eps_tx_ms=0.2,
                                              zeta_tx_ms_per_token=0.001, delta_stage_ms_per_token=0.01))
        out = None
        # the third run: real clock with host inputs and the logits read back
        # through the C-ABI (e2e) — the last stage's logits transfers are
        # waited on after their completion was polled
        for clock, e2e in (("lockstep", False), ("real", False), ("real", True)):
            print(f"rank {rank}: {clock} run (e2e={e2e})", flush=True)
            if rank == 0:
                dist.barrier()
                log, journal, stats = g.run(ctx, None, WL, sc, clock=clock, payload_seed=7, e2e=e2e)
                ok = log == api.simulate(WL, sc)[0] if clock == "lockstep" else True
                out = dict(clock=clock + ("_e2e" if e2e else ""), decisions_equal=ok, gpu_ms=stats["gpu_ms"], log=log,
                           journal=journal,
                           logits={r: ctx.logits(r)[0].tolist() for r in (0, 1, 2)},
                           argmax={r: ctx.logits(r)[1] for r in (0, 1, 2)})
                q.put((rank, init_s, out))
            else:
                g.worker_prepare(ctx, WL, payload_seed=7, e2e=e2e)
                dist.barrier()
                g.worker_run(ctx)
        dist.barrier()
        if rank != 0:
            q.put((rank, init_s, "ok"))
        g.close()
        ctx.close()
    except Exception as e:  # report, do not hang the other rank
        q.put((rank, -1, f"{type(e).__name__}: {e}"))
        raise
    finally:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--same-device", action="store_true")
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"])
    ap.add_argument("--json", default=None, help="write the per-rank results here")
    a = ap.parse_args()
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=rank_main, args=(r, a.world, port, a.same_device, a.transport, q)) for r in range(a.world)]
    for p in procs:
        p.start()
    # Drain the queue before joining: a child blocks at exit until its queued
    # results are written to the pipe.
    results = []
    expected = 3 + (a.world - 1)  # rank 0: one per run; workers: one each
    import queue
    while len(results) < expected:
        try:
            results.append(q.get(timeout=300))
        except queue.Empty:
            break
        if any(isinstance(o, str) and o != "ok" for _, _, o in results):
            break
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():  # our own child: stop it rather than hang the caller
            p.kill()
            p.join()
    for rank, init_s, out in results:
        if isinstance(out, dict):
            print(f"rank {rank} {out['clock']}: decisions_equal={out['decisions_equal']} "
                  f"gpu_ms={out['gpu_ms']:.3f} argmax={out['argmax']} init_s={init_s:.2f}")
        else:
            print(f"rank {rank}: {out}")
    print("exitcodes", [p.exitcode for p in procs])
    if a.json:
        with open(a.json, "w") as f:
            json.dump(dict(results=results, exitcodes=[p.exitcode for p in procs]), f)


if __name__ == "__main__":
    main()
