#!/usr/bin/env python
"""rserve-b200 benchmark: RServe intra-request pipeline on B200.

Metric (BASELINE.json): p50/p99 TTFT (ms) and encode+prefill tokens/s at
1/2/4/8 B200, next to the reference's CPU path.

N = 1 (BASELINE.json configs[1], "cfg2"): Qwen2.5-VL-7B-shaped model
(ViT-600M 1280x32 + 7B LLM 3584x28, random init), ONE request of 8 images
interleaved with text, T128|(M1024|T32)x8 = 8576 prompt tokens, Algorithm-1
C = 1024 (one 896x896 image = 4096 patches per encode batch), Algorithm-2
budget B = 2048, policy rserve, 1 pipeline stage, encoder and prefill
co-located on one GPU on two streams (the reference's zero-cost link).
A step = one request through the real-clock engine (encode -> tracker ->
chunked prefill -> first-token logits); value = prompt tokens / device time
(CUDA events, origin -> last completion) over K steps. The line also carries
a "cfg3" block: the same Poisson request stream the N > 1 runs measure, here
co-located, so every N reports that workload; "cfg4" (the C sweep
128-2048 over that stream) and "cfg5" (64 x M256 + T128 on the 72B-shaped LLM,
145 GB of weights) run co-located after it — their 4E+4P placement needs 8 GPUs.

N > 1 (configs[2]/[3], "cfg3"): the paper's EP deployment, one process per
GPU — 1E+1P (N=2), 2E+2P with a 2-stage CPP pipeline (N=4), 4E+4P with 4
stages (N=8); rank 0 = P0 runs the engine and the device tracker; embeddings
move E_w -> P0 and residuals P_s -> P_s+1 over NCCL send/recv on per-link
side streams (--ep-transport ipc: CUDA-IPC peer memory). Workload: the
reference generator (workload.hpp:139-172) with template "alternating",
U[4,16] images of 1024 tokens, text segments U[32,256], seeds {1,2,3}.
value = throughput plateau (Poisson at a saturating 32 req/s, ~16 requests per
step; tokens/s = sum prompt tokens / makespan, metrics.hpp:78-81); ttft_ms =
nearest-rank p50/p99 over all requests of the 4 req/s latency runs
(workload.hpp:184-192); a "cfg2" block gives the single-request TTFT on the
same placement. `python bench.py --gpus N` re-executes itself under
torch.distributed.run when not already launched by it.

e2e = the same metric through the public C-ABI with pixel patches copied H2D
from pinned host memory and the first-token logits read back D2H inside the
timed region. Inputs (16 GB of weights, 77+ MB of pixels per request) exceed
the 126 MB L2, so no explicit flush between steps.

Parity evidence, outside every timed region: each timed run's event journal
is replayed through the reference's own components (oracle/_ref, compiled
from /root/reference) and must reproduce the run's slices and release order
(decisions_replay_ok); the cfg2 first-token logits are compared with the fp32
oracle (oracle/model_oracle_torch.py, same GPU, TF32 off): logit_err_over_std.

--impl reference: the reference's path on the host CPU, on the same config —
the reference scheduler itself (oracle/_ref run_simulation + journal replay,
timed) plus the fp32 numpy restatement of the model math (the reference
performs none) timed on a bounded sample (one ViT layer on one 896x896 image
+ one LLM layer on one B-token chunk) and extrapolated by FLOPs, labelled as
such; cfg1 (tiny model) runs in full on the oracle. Never loads the product.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LAYOUT = "T128|" + "|".join(["M1024|T32"] * 8)
PROMPT_TOKENS = 128 + 8 * 1056
C_TOKENS = 1024
CFG1_LAYOUT = "T64|M256|M256|T32|M256|M256"
# cfg3 request stream: template alternating, U[4,16] items of
# 1024 tokens (896x896 images), text U[32,256]; seeds {1,2,3}
CFG3 = {"pattern": "alternating", "mm_items": (4, 16), "mm_tokens": 1024, "text_tokens": (32, 256),
        "seeds": (1, 2, 3), "tput_rate": 32.0, "tput_duration_s": 0.5, "lat_rate": 4.0,
        "lat_duration_s": 3.0}
MAX_PROMPT = 16 * 1024 + 17 * 256  # largest cfg3 request
EP_LAYOUTS = {2: (1, 1), 4: (2, 2), 8: (4, 4)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return j["bf16_tflops"], j.get("bf16_tflops_sustained", j["bf16_tflops"]), j["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


def nearest_rank(sorted_vals, pct):
    """workload.hpp:184-192 nearest-rank percentile."""
    if not sorted_vals:
        return None
    return sorted_vals[max(0, -(-pct * len(sorted_vals) // 100) - 1)]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, device, interval_ms=200):
        self.device = device
        self.interval_ms = interval_ms
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            try:
                p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                                     stdout=subprocess.PIPE, text=True)
            except OSError:
                return
            while not self._stop.is_set():
                line = p.stdout.readline()
                if not line:
                    break
                self.samples.append([x.strip() for x in line.split(",")])
            p.terminate()
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        # nvidia-smi's NVML start-up takes driver locks that can stall CUDA
        # calls for ~100 ms: let it reach its first sample before timing
        t0 = time.time()
        while not self.samples and time.time() - t0 < 5.0:
            time.sleep(0.05)
        time.sleep(0.2)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=3)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        loaded = [v for v in sm if v > 0.5 * max(mx or [1])] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.samples)}


# ---- model work --------------------------------------------------------------
def qwen7b_shapes():
    """Model shapes from the oracle's config (the reference arm must not load
    the product library); equal to rs_model_preset(qwen2.5-vl-7b)."""
    from oracle import model_oracle as mo
    c = mo.ModelConfig.qwen7b()
    return {k: getattr(c, k) for k in ("vit_dim", "vit_layers", "vit_heads", "vit_ff", "vit_window",
                                       "vit_fullatt_every", "patch_dim", "llm_dim", "llm_layers",
                                       "llm_q_heads", "llm_kv_heads", "llm_head_dim", "llm_ff", "vocab")}


def image_flops(m, img_tokens=1024):
    """ViT + merger FLOPs of one image of `img_tokens` LLM tokens."""
    vd, ff, P = m["vit_dim"], m["vit_ff"], 4 * img_tokens
    vit = 2 * P * vd * 1176 + m["vit_layers"] * 2 * P * (4 * vd * vd + 3 * vd * ff)
    nfull = m["vit_layers"] // m["vit_fullatt_every"]
    vit += (m["vit_layers"] - nfull) * (P // 64) * 4 * 64 * 64 * vd + nfull * 4 * P * P * vd
    mi = 4 * vd
    return vit + 2 * img_tokens * (mi * mi + mi * m["llm_dim"])


def prefill_flops(m, T):
    d, hd = m["llm_dim"], m["llm_head_dim"]
    qkv = (m["llm_q_heads"] + 2 * m["llm_kv_heads"]) * hd
    dense = T * m["llm_layers"] * 2 * (d * qkv + m["llm_q_heads"] * hd * d + 3 * d * m["llm_ff"])
    attn = m["llm_layers"] * 2 * T * T * m["llm_q_heads"] * hd  # causal: 4*T^2/2
    return dense + attn + 2 * d * m["vocab"]


def layout_flops(m, layout):
    segs = [(f[0], int(f[1:])) for f in layout.split("|")]
    T = sum(n for _, n in segs)
    return sum(image_flops(m, n) for k, n in segs if k == "M"), prefill_flops(m, T), T


def model_flops(m):
    """Algorithmic FLOPs of one cfg2 request (encode, prefill)."""
    e, p, _ = layout_flops(m, LAYOUT)
    return e, p


def workload_layouts(wl):
    return [line.split(",", 3)[3] for line in wl.strip().splitlines() if line.strip()]


# ---- launch ------------------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_under_torchrun(n):
    """`bench.py --gpus N` outside torchrun: one rank per GPU, same arguments."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def ep_mode(args, ws):
    return ws > 1 and args.mode == "ep"


def bench_config(args, ws):
    """The workload every arm reports at this N (identical dict in both arms)."""
    if ep_mode(args, ws):
        stages, encoders = EP_LAYOUTS[ws]
        return {"workload": "cfg3: Qwen2.5-VL-7B-shaped (random init), Poisson stream of "
                            "alternating text/image requests, U[4,16] images of 896x896 (1024 "
                            "tokens), text U[32,256], seeds {1,2,3}; throughput plateau at "
                            f"{CFG3['tput_rate']:g} req/s, TTFT at {CFG3['lat_rate']:g} req/s",
                "model": "qwen2.5-vl-7b-shaped", "policy": args.policy, "C": C_TOKENS,
                "B": args.budget, "stages": stages, "encoders": encoders,
                "placement": f"EP {encoders}E+{stages}P", "parallelism": f"ep{encoders}+pp{stages}",
                "transport": args.ep_transport, "l2": "inputs (16 GB weights) >> 126 MB L2; no flush"}
    return {"workload": "cfg2: Qwen2.5-VL-7B-shaped (random init), 1 request "
                        "T128|(M1024|T32)x8 = 8576 tokens, 8 images of 896x896",
            "model": "qwen2.5-vl-7b-shaped", "global_batch": 1, "seq_len": PROMPT_TOKENS,
            "policy": args.policy, "C": C_TOKENS, "B": args.budget, "stages": 1,
            "placement": "encoder+prefill co-located, 2 streams" if ws == 1 else
                         f"{ws} independent co-located replicas",
            "parallelism": "replicas" if ws > 1 else "single",
            "l2": "inputs (16 GB weights) >> 126 MB L2; no flush"}


# ---- helpers over the product API ------------------------------------------------------------
def cfg3_workload(seed, rate, duration_s):
    from paper_2509_24381_b200 import api
    t = api.RequestTemplate(CFG3["pattern"], api.IntDistribution(*CFG3["mm_items"]),
                            api.IntDistribution(CFG3["mm_tokens"]),
                            api.IntDistribution(*CFG3["text_tokens"]))
    return api.generate_workload(api.WorkloadConfig(arrival_rate=rate, duration_s=duration_s,
                                                    seed=seed, templates=[t]))


def stream_stats(log):
    """Per-run request TTFTs and the reference throughput definition:
    sum prompt tokens / (last completion - first arrival) (metrics.hpp:78-81)."""
    from paper_2509_24381_b200 import api
    p = api.parse_decision_log(log)
    res = p["result"][0]
    reqs = p["req"]
    tokens = sum(int(r["prompt"]) for r in reqs)
    makespan = float(res["last_completion"]) - float(res["first_arrival"])
    return {"ttfts": [float(r["ttft"]) for r in reqs], "tokens": tokens, "makespan_ms": makespan,
            "requests": len(reqs), "completed": all(r["completed"] == "1" for r in reqs)}


class Replayer:
    """Journal replay of timed runs through the reference's own components
    (oracle/_ref, the checker): slices and release order must be equal."""

    def __init__(self):
        self.ok, self.runs, self.err = True, 0, None
        try:
            from oracle import ref
            ref.lib()
            self.ref = ref
        except Exception as e:  # pragma: no cover - _ref not built
            self.ref, self.ok, self.err = None, False, f"oracle/_ref unavailable: {e}"

    def check(self, wl, sc, log, journal):
        if self.ref is None:
            return
        from paper_2509_24381_b200 import api
        try:
            theirs = api.parse_decision_log(self.ref.replay(wl, sc.to_c(), journal))
        except Exception as e:
            self.ok, self.err = False, str(e)[:300]
            return
        ours = api.parse_decision_log(log)
        key = lambda recs: [(r["req"], r["chunk"], r["start"], r["end"]) for r in recs]  # noqa: E731
        same = key(ours.get("slice", [])) == key(theirs.get("slice", [])) and \
            ours.get("release") == theirs.get("release")
        self.runs += 1
        if not same:
            self.ok = False
            self.err = self.err or f"run {self.runs}: slices/releases differ from the reference replay"

    def summary(self):
        return {"decisions_replay_ok": bool(self.ok and self.runs > 0), "replayed_runs": self.runs,
                "replay_error": self.err,
                "method": "every timed run's event journal replayed through the reference's "
                          "tracker / Algorithm-1 / Algorithm-2 / release code (oracle/_ref)"}


def cfg2_logit_parity(logits, argmax, device):
    """cfg2 first-token logits vs the fp32 oracle at full depth (checker)."""
    import numpy as np
    from oracle import model_oracle as mo
    from oracle import model_oracle_torch as mt
    t0 = time.perf_counter()
    _, ref = mt.first_token_logits(mo.ModelConfig.qwen7b(), LAYOUT, 1234, req_id=0, device=device)
    _, ref16 = mt.first_token_logits(mo.ModelConfig.qwen7b(), LAYOUT, 1234, req_id=0, device=device,
                                     bf16_acts=True)
    ref, ref16 = ref.cpu().numpy(), ref16.cpu().numpy()
    err = float(np.abs(np.asarray(logits) - ref).max() / ref.std())
    err16 = float(np.abs(ref16 - ref).max() / ref.std())
    return {"logit_err_over_std": err, "bf16_storage_oracle_err_over_std": err16,
            "within_tolerance": err <= min(0.15, err16) and int(argmax) == int(ref.argmax()),
            "argmax": int(argmax), "oracle_argmax": int(ref.argmax()),
            "argmax_equal": int(argmax) == int(ref.argmax()),
            "tolerance": "argmax equal and max|dlogit| <= min(0.15 std, the fp32 oracle's own "
                         "deviation when rounded to bf16 at the device's storage points)",
            "oracle": "fp32 torch mirror of oracle/model_oracle.py, full depth, TF32 off",
            "oracle_s": round(time.perf_counter() - t0, 1)}


def group_profile(raw):
    """Kernel classes from the profiler's labels: GEMM launches are labelled
    per shape ("gemm_tcgen05|M|N|K|epi|BN|CG") and grouped on the prefix; the
    per-shape rows are returned separately (sorted by time)."""
    out, shapes, attn = {}, [], []
    for k, v in raw.items():
        base = k.split("|")[0]
        a = out.setdefault(base, {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0})
        for f in a:
            a[f] += v[f]
        if base == "attn_prefill_tcgen05" and "|" in k:
            items, keys, splits = (int(x) for x in k.split("|")[1:])
            attn.append({"items": items, "max_keys": keys, "kv_splits": splits,
                         "launches": v["launches"], "ms": round(v["ms"], 3)})
        elif "|" in k:
            M, Nn, K, epi, bn, cg = (int(x) for x in k.split("|")[1:])
            shapes.append({"M": M, "N": Nn, "K": K, "epi": epi, "tile": f"{128 * cg}x{bn}",
                           "launches": v["launches"], "ms": round(v["ms"], 3),
                           "tflops": round(v["flops"] / (v["ms"] / 1e3) / 1e12, 1) if v["ms"] else None})
    shapes.sort(key=lambda r: -r["ms"])
    attn.sort(key=lambda r: -r["ms"])
    return out, shapes, attn


# Bound of each kernel class: tensor-bound classes against the
# burst bf16 peak, HBM-bound ones against the copy peak.
KERNEL_BOUNDS = {"gemm_tcgen05": "tensor", "attn_prefill_tcgen05": "tensor", "attn_vit_tcgen05": "tensor",
                 "attn_vit_window_tc": "hbm", "tracker_scatter_k6": "hbm", "rmsnorm": "hbm",
                 "rmsnorm_gather": "hbm", "vit_qkv_split": "hbm", "gemv_small_m": "hbm"}


def kernel_rooflines(prof, pk_tflops, hbm_gbs):
    """Per kernel class of the profiling step: algorithmic FLOPs (tensor) or
    bytes (HBM) each launch declares / its CUDA-event time, as a fraction of
    the bound's measured peak. Event-bracketed launches (no PDL overlap), so
    microsecond kernels read low."""
    out = {}
    for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"]):
        bound = KERNEL_BOUNDS.get(k)
        if bound is None or v["ms"] <= 0:
            continue
        if bound == "tensor" and v["flops"] > 0:
            a = v["flops"] / (v["ms"] / 1e3) / 1e12
            out[k] = {"bound": "tensor", "achieved": round(a, 1), "peak": pk_tflops, "unit": "TFLOP/s",
                      "frac": round(a / pk_tflops, 3), "ms_per_step": round(v["ms"], 3)}
        elif bound == "hbm" and v["bytes"] > 0:
            a = v["bytes"] / (v["ms"] / 1e3) / 1e9
            out[k] = {"bound": "hbm", "achieved": round(a, 1), "peak": hbm_gbs, "unit": "GB/s",
                      "frac": round(a / hbm_gbs, 3), "ms_per_step": round(v["ms"], 3)}
    return out


def sim_cfg(args, m, stages=1, encoders=1, c_tokens=C_TOKENS, beta_enc=0.01):
    from paper_2509_24381_b200 import api
    return api.SimConfig(policy=args.policy, stages=stages, token_budget=args.budget,
                         embedding_batch_tokens=c_tokens, encoder_workers=encoders,
                         hidden_size=m["llm_dim"],
                         cost=api.CostModel(beta_enc_ms_per_token=beta_enc, delta_stage_ms_per_token=0.01))


def summarize_stream(runs, tokens_key="gpu"):
    """runs: [(stream_stats, run_stats)] -> throughput + TTFT percentiles."""
    tokens = sum(s["tokens"] for s, _ in runs)
    makespan = sum(s["makespan_ms"] for s, _ in runs)
    ttfts = sorted(t for s, _ in runs for t in s["ttfts"])
    return {"tokens_per_s": tokens / (makespan / 1e3) if makespan > 0 else None,
            "requests": sum(s["requests"] for s, _ in runs), "tokens": tokens,
            "makespan_ms": [round(s["makespan_ms"], 2) for s, _ in runs],
            "ttft_ms": {"p50": nearest_rank(ttfts, 50), "p99": nearest_rank(ttfts, 99),
                        "mean": sum(ttfts) / len(ttfts) if ttfts else None},
            "all_completed": all(s["completed"] for s, _ in runs)}


# ---- our arm, one GPU (co-located) or replicas -----------------------------------------------
def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    from paper_2509_24381_b200 import _native as N
    from paper_2509_24381_b200 import api
    mcfg = api.model_preset("qwen2.5-vl-7b")
    m = {k: getattr(mcfg, k) for k, _ in N.rs_model_config._fields_}
    pipe = api.Pipeline(mcfg, device=local, max_prompt_tokens=MAX_PROMPT, slot_tokens=1 << 19,
                        kv_tokens=1 << 19, max_chunk_tokens=args.budget, max_encode_tokens=C_TOKENS)
    wl = f"0,0,-,{LAYOUT}\n"
    sc = sim_cfg(args, m)
    replay = Replayer()
    chunk_sizes = {}
    # Profiling step: kernels serialised on one stream (per-kernel event times
    # without cross-stream queueing), event order from a cost model in which
    # encoding outruns prefill, as it does on the device (PDL + encoder
    # stream priority) -> the same prefill chunk plan as the timed steps.
    sc_prof = sim_cfg(args, m, beta_enc=0.0001)
    last = {}

    def step(e2e=False, serialize=False, check=False):
        s = sc_prof if serialize else sc
        log, journal, st = pipe.run(wl, s, clock="lockstep" if serialize else "real", e2e=e2e,
                                    payload_seed=1234, serialize=serialize)
        if check:
            replay.check(wl, s, log, journal)
        parsed = api.parse_decision_log(log)
        rec = parsed["req"][0]
        sizes = {}
        for sl in parsed.get("slice", []):
            sizes[sl["chunk"]] = sizes.get(sl["chunk"], 0) + int(sl["end"]) - int(sl["start"])
        chunk_sizes["serialized" if serialize else "e2e" if e2e else "timed"] = list(sizes.values())
        last["log"], last["journal"] = log, journal
        return float(rec["ttft"]), st

    for _ in range(args.warmup):
        step()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ttfts, dev_ms, launches, host_gaps, journals = [], [], 0, [], []
    with ClockSampler(local, args.clock_sample_ms) as clk:
        for _ in range(args.steps):
            t, st = step()
            journals.append((last["log"], last["journal"]))
            ttfts.append(t)
            dev_ms.append(st["gpu_ms"])
            host_gaps.append([round(st["host_max_gap_ms"], 2), round(st["host_max_call_ms"], 2),
                              int(st["host_max_call_kind"]), round(st["host_max_launch_ms"], 2)])
            launches += st["kernel_launches"]
    torch.cuda.synchronize()
    if args.launch_list:
        # ncu launch-list pass: only the plain warm-up + timed steps above
        pipe.close()
        if rank == 0:
            print(json.dumps({"launch_list": True, "steps": args.steps, "warmup": args.warmup,
                              "ttft_ms": ttfts, "note": "timed under a profiler: not a bench value"}))
        return
    for log, journal in journals:  # parity evidence, outside the timed region
        replay.check(wl, sc, log, journal)
    logits_cfg2, am_cfg2 = pipe.logits(0)
    # Per-kernel-class timing for the roofline: one extra step with CUDA events
    # around every launch, encoders on the prefill stream (serialised) so each
    # event pair measures the kernel alone, not cross-stream queueing.
    N.check(N.lib.rs_profile_enable(1))
    prof_ttft, prof_st = step(serialize=True, check=True)
    torch.cuda.synchronize()
    N.check(N.lib.rs_profile_enable(0))
    prof_raw = N.profile_drain()
    prof, gemm_shapes, attn_shapes = group_profile(prof_raw)
    # e2e through the public API: H2D pixels from pinned host + D2H logits in the timed region
    e2e_wall, e2e_gpu, h2d, d2h, e2e_gaps = [], [], 0, 0, []
    for _ in range(max(1, args.warmup // 2)):
        step(e2e=True)
    for _ in range(args.steps):
        t, st = step(e2e=True)
        e2e_wall.append(st["wall_ms"])
        e2e_gpu.append(st["gpu_ms"])
        e2e_gaps.append([round(st["host_max_gap_ms"], 2), round(st["host_last_seen_ms"], 2),
                         round(st["host_finish_sync_ms"], 2)])
        h2d, d2h = st["h2d_bytes"], st["d2h_bytes"]
    # cfg3: the Poisson request stream the N > 1 runs measure, co-located here
    cfg3 = None
    if args.cfg3_steps > 0 and ws == 1:
        try:
            cfg3 = run_cfg3_colocated(args, pipe, m, replay)
        except Exception as e:  # recorded; the headline line must still print
            cfg3 = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
    # Decode after the first token (the reference stops at TTFT):
    # the request's KV stays on the device, then greedy decode steps.
    decode = None
    if args.decode_steps > 0:
        try:
            decode = run_decode(args, pipe, wl, sc, m)
        except Exception as e:  # recorded; the headline line must still print
            decode = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
    total_ms = sum(dev_ms)
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms, sum(e2e_wall)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_total = t.tolist()
    else:
        e2e_total = sum(e2e_wall)
    value = ws * args.steps * PROMPT_TOKENS / (total_ms / 1e3)
    e2e_value = ws * args.steps * PROMPT_TOKENS / (e2e_total / 1e3)
    ttft_steps = list(ttfts)
    ttfts.sort()
    p50, p99 = nearest_rank(ttfts, 50), nearest_rank(ttfts, 99)
    pk, pk_sus, hbm, pk_kind = peaks()
    g = prof.get("gemm_tcgen05", {"ms": 0.0, "flops": 0.0, "launches": 0, "bytes": 0.0})
    achieved = g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else 0.0
    prof_total_ms = sum(v["ms"] for v in prof.values())
    vit_f, llm_f = model_flops(m)
    bound_ms = (vit_f + llm_f) / (pk * 1e12) * 1e3
    bound_sus_ms = (vit_f + llm_f) / (pk_sus * 1e12) * 1e3
    ncu_full = None
    ncu_path = os.path.join(ROOT, "profiles", "r01_ncu_gemm_pair_full.json")
    if os.path.exists(ncu_path):
        ncu_full = json.load(open(ncu_path))
    parity = replay.summary()
    if rank == 0 and not args.no_parity:
        try:
            parity.update(cfg2_logit_parity(logits_cfg2, am_cfg2, f"cuda:{local}"))
        except Exception as e:
            parity["logit_check_error"] = f"{type(e).__name__}: {str(e)[:300]}"
    line = {
        "metric": "encode+prefill tokens/s (p50/p99 TTFT ms alongside)",
        "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "ttft_ms": {"p50": p50, "p99": p99, "mean": sum(ttfts) / len(ttfts),
                    "percentiles": "nearest-rank over the K timed steps of the one cfg2 request "
                                   "(the request-level distribution is in cfg3)",
                    "per_step": [round(x, 2) for x in ttft_steps], "host_max_gap_ms": host_gaps,
                    "roofline_bound_ms": bound_ms, "roofline_frac": bound_ms / p50,
                    "roofline_bound_ms_sustained_peak": bound_sus_ms,
                    "roofline_note": "bound = model FLOPs / measured burst bf16 peak; the sustained "
                                     "(power-capped) bound beside"},
        "config": bench_config(args, ws),
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "p50_ms": statistics.median(e2e_wall),
                "wall_ms_per_step": [round(x, 2) for x in e2e_wall],
                "gpu_ms_per_step": [round(x, 2) for x in e2e_gpu],
                "host_max_gap_and_last_seen_ms": e2e_gaps,
                "timing": "host wall clock of each run (H2D pixels from pinned memory + D2H logits inside)"},
        "gpu_launches": launches,
        "roofline": {"bound": "tensor", "kernel": "gemm_tcgen05 (all GEMMs of the step)",
                     "achieved": achieved, "peak": pk, "unit": "TFLOP/s",
                     "frac": achieved / pk if pk else None,
                     "peak_kind": pk_kind + " burst bf16 (MEASURED_PEAKS.json bf16_tflops)",
                     "peak_sustained": pk_sus, "frac_of_sustained": achieved / pk_sus if pk_sus else None,
                     "method": "CUDA events around every GEMM launch of one serialised profiling "
                               "step (encode on the prefill stream); achieved = sum(2MNK) / "
                               "sum(event time)",
                     "traffic": ncu_full["traffic_bytes"] if ncu_full else None,
                     "traffic_note": (f"dram read+write bytes per launch of the dominant GEMM "
                                      f"({ncu_full['shape']['M']}x{ncu_full['shape']['N']}x"
                                      f"{ncu_full['shape']['K']} {ncu_full['shape']['epilogue']}, "
                                      f"{ncu_full['shape']['tile']}) from one ncu --set full capture "
                                      f"(profiles/r01_ncu_gemm_pair_full.json); algorithmic "
                                      f"{ncu_full['algorithmic_bytes']:.0f} B; tensor pipe "
                                      f"{ncu_full['tensor_pipe_active_pct_of_elapsed']:.1f}% active")
                     if ncu_full else None,
                     "share_of_kernel_time": g["ms"] / prof_total_ms if prof_total_ms else None},
        "parity": parity,
        "profiling_step": {"note": "one extra step, kernels serialised on one stream with CUDA "
                                   "events around each launch; lock-step event order giving the "
                                   "timed steps' chunk plan", "gpu_ms": prof_st["gpu_ms"],
                           "kernel_ms_sum": prof_total_ms},
        "kernel_classes": {k: {"launches": v["launches"], "ms_per_step": v["ms"],
                               "share": v["ms"] / prof_total_ms if prof_total_ms else None,
                               # achieved rates from the algorithmic work each launch declares
                               "tflops": v["flops"] / (v["ms"] / 1e3) / 1e12 if v["ms"] and v["flops"] else None,
                               "gbs": v["bytes"] / (v["ms"] / 1e3) / 1e9 if v["ms"] and v["bytes"] else None}
                           for k, v in prof.items()},
        "rooflines": kernel_rooflines(prof, pk, hbm),
        "gemm_shapes": gemm_shapes[:16],
        "attn_prefill_shapes": attn_shapes,
        "cfg3": cfg3,
        "decode": decode,
        "prefill_chunk_tokens": chunk_sizes,
        "model_tflop_per_request": {"encode": vit_f / 1e12, "prefill": llm_f / 1e12},
        "clocks": clk.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args, reps=1)
        except Exception as e:
            line["cpu_baseline"] = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
    pipe.close()
    if ws == 1 and args.cfg45:
        # configs 4 / 5 (their 4E+4P placement needs 8 GPUs): co-located here,
        # after the cfg2 context is gone (cfg5's 72B weights take 145 GB); a
        # failure is recorded, never allowed to cost the headline line
        for key, fn, steps in (("cfg4", run_cfg4, 1), ("cfg5", run_cfg5, 2)):
            try:
                line[key] = fn(steps)
            except Exception as e:  # e.g. a box with less free HBM than cfg5's 150 GB
                line[key] = {"error": f"{type(e).__name__}: {str(e)[:300]}"}
    if rank == 0:
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


def run_decode(args, pipe, wl, sc, m):
    """Greedy decode of the cfg2 request after its first token:
    the request's KV stays on the device (keep_kv), then batched decode steps."""
    pipe.run(wl, sc, clock="real", payload_seed=1234, keep_kv=True)
    pipe.decode([0], 2)
    pipe.decode_release(0)
    pipe.run(wl, sc, clock="real", payload_seed=1234, keep_kv=True)
    # PD (prefill -> decode) transfer of the request's KV image, imported as
    # request 1 on the same context (the cross-GPU move is the caller's copy)
    import torch
    nbytes = pipe.kv_image_bytes(PROMPT_TOKENS)
    img = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    meta = pipe.kv_export(0, img.data_ptr(), nbytes, stream=st.cuda_stream)
    pipe.kv_import(1, meta, img.data_ptr(), stream=st.cuda_stream)
    e1.record(st)
    e1.synchronize()
    pd_ms = e0.elapsed_time(e1)
    toks, _, dms = pipe.decode([0], args.decode_steps)
    toks_pd, _, _ = pipe.decode([1], args.decode_steps)
    pipe.decode_release(0)
    pipe.decode_release(1)
    del img
    hbm_gbs = peaks()[2]
    llm_bytes = 2.0 * (m["llm_layers"] * (m["llm_dim"] * (m["llm_q_heads"] + 2 * m["llm_kv_heads"]) *
                                           m["llm_head_dim"] + m["llm_q_heads"] * m["llm_head_dim"] *
                                           m["llm_dim"] + 3 * m["llm_dim"] * m["llm_ff"]) +
                       m["vocab"] * m["llm_dim"])
    decode = {"steps": args.decode_steps, "batch": 1, "ms_per_step": dms / args.decode_steps,
              "tokens_per_s": args.decode_steps / (dms / 1e3),
              "context_tokens": PROMPT_TOKENS,
              "roofline": {"bound": "hbm", "bytes_per_step": llm_bytes,
                           "bound_ms": llm_bytes / (hbm_gbs * 1e9) * 1e3,
                           "frac": (llm_bytes / (hbm_gbs * 1e9) * 1e3) / (dms / args.decode_steps)},
              "note": "greedy decode of the cfg2 request after its first token (device time, "
                      "CUDA events); per step every LLM weight is read once (batch 1)",
              "pd_transfer": {"image_bytes": nbytes, "export_import_ms": pd_ms,
                              "gbs": 2.0 * 2 * nbytes / (pd_ms / 1e3) / 1e9,
                              "decoded_tokens_equal": bool((toks == toks_pd).all()),
                              "note": "rs_kv_export + rs_kv_import of the 8576-token KV (pack + unpack, "
                                      "each reads and writes the image: 4 x bytes); decoding the imported "
                                      "request gives the local request's tokens"}}
    return decode


def run_cfg3_colocated(args, pipe, m, replay):
    """cfg3 on one GPU: throughput plateau (saturating Poisson stream) and the
    TTFT distribution at the latency rate, seeds {1,2,3}."""
    sc = sim_cfg(args, m)
    out = {}
    for mode, rate, dur in (("throughput", CFG3["tput_rate"], CFG3["tput_duration_s"]),
                            ("latency", CFG3["lat_rate"], CFG3["lat_duration_s"])):
        seeds = CFG3["seeds"][:args.cfg3_steps]
        pipe.run(cfg3_workload(seeds[0], rate, dur), sc, clock="real", payload_seed=1234)  # warm
        runs = []
        for s in seeds:
            wl = cfg3_workload(s, rate, dur)
            log, journal, st = pipe.run(wl, sc, clock="real", payload_seed=1234)
            replay.check(wl, sc, log, journal)
            runs.append((stream_stats(log), st))
        out[mode] = dict(summarize_stream(runs), rate_req_s=rate, duration_s=dur, seeds=list(seeds))
    return dict(out, placement="co-located", note="same workload as the N>1 EP lines")


# ---- north_star configs 4 and 5 on one GPU (appended to the N = 1 line) ------------------------
CFG5_LAYOUT = "|".join(["M256"] * 64) + "|T128"


def run_cfg4(steps):
    import torch
    from paper_2509_24381_b200 import _native as N
    from paper_2509_24381_b200 import api
    mcfg = api.model_preset("qwen2.5-vl-7b")
    m = {k: getattr(mcfg, k) for k, _ in N.rs_model_config._fields_}
    pipe = api.Pipeline(mcfg, max_prompt_tokens=MAX_PROMPT, slot_tokens=1 << 19, kv_tokens=1 << 19,
                        max_chunk_tokens=2048, max_encode_tokens=2048 + 1024)
    replay = Replayer()
    wl = cfg3_workload(1, CFG3["lat_rate"], CFG3["lat_duration_s"])
    rows = []
    for C in (128, 256, 512, 1024, 2048):
        ns = argparse.Namespace(policy="rserve", budget=2048)
        sc = sim_cfg(ns, m, c_tokens=C)
        pipe.run(wl, sc, clock="real", payload_seed=1234)  # warm (plans, workspaces)
        runs = []
        for _ in range(steps):
            log, journal, st = pipe.run(wl, sc, clock="real", payload_seed=1234)
            replay.check(wl, sc, log, journal)
            runs.append((stream_stats(log), st))
        s = summarize_stream(runs)
        rows.append({"C": C, "ttft_p50_ms": s["ttft_ms"]["p50"], "ttft_p99_ms": s["ttft_ms"]["p99"],
                     "tokens_per_s": s["tokens_per_s"], "requests": s["requests"] // steps,
                     "all_completed": s["all_completed"]})
        print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    pipe.close()
    return {"workload": "cfg4: cfg3 stream (alternating, U[4,16] x M1024, text U[32,256], Poisson "
                        f"{CFG3['lat_rate']} req/s for {CFG3['lat_duration_s']} s, seed 1), "
                        "7B-shaped, B=2048, co-located on 1 GPU (the paper's 4E+4P needs 8)",
            "sweep": rows, **replay.summary()}


def run_cfg5(steps):
    import torch
    from paper_2509_24381_b200 import _native as N
    from paper_2509_24381_b200 import api
    mcfg = api.model_preset("qwen2.5-vl-72b-llm")
    m = {k: getattr(mcfg, k) for k, _ in N.rs_model_config._fields_}
    T = 64 * 256 + 128
    pipe = api.Pipeline(mcfg, max_prompt_tokens=T, slot_tokens=T + 4096, kv_tokens=T + 4096,
                        max_chunk_tokens=2048, max_encode_tokens=1024)
    wl = f"0,0,-,{CFG5_LAYOUT}\n"
    ns = argparse.Namespace(policy="rserve", budget=2048)
    sc = sim_cfg(ns, m, c_tokens=1024)
    replay = Replayer()
    enc_f, pre_f, T2 = layout_flops(m, CFG5_LAYOUT)
    assert T2 == T
    for _ in range(2):
        pipe.run(wl, sc, clock="real", payload_seed=99)
    ttfts, dev = [], []
    for _ in range(steps):
        log, journal, st = pipe.run(wl, sc, clock="real", payload_seed=99)
        replay.check(wl, sc, log, journal)
        rec = api.parse_decision_log(log)["req"][0]
        ttfts.append(float(rec["ttft"]))
        dev.append(st["gpu_ms"])
    logits, am = pipe.logits(0)
    pipe.close()
    ttfts.sort()
    peak = peaks()[0]
    bound_ms = (enc_f + pre_f) / (peak * 1e12) * 1e3
    p50 = nearest_rank(ttfts, 50)
    return {"workload": "cfg5: ConsecutiveMm 64 x M256 + T128 = 16512 tokens, 72B-shaped LLM + 1280-wide ViT "
                        "(random init), C=1024, B=2048, rserve, co-located on 1 GPU (the paper's 4E+4P needs 8)",
            "ttft_ms": {"p50": p50, "p99": nearest_rank(ttfts, 99), "per_step": [round(t, 2) for t in ttfts]},
            "tokens_per_s": T / (p50 / 1e3),
            "tflop_per_request": {"encode": enc_f / 1e12, "prefill": pre_f / 1e12},
            "roofline": {"bound_ms_burst_peak": bound_ms, "frac": bound_ms / p50, "peak_tflops": peak},
            "logits_finite": bool(torch.isfinite(torch.as_tensor(logits)).all()), "argmax": am,
            **replay.summary()}


# ---- our arm, N > 1: EP deployment -----------------------------------------------------------
def run_ep(args):
    """The paper's EP deployment on N = 2/4/8 GPUs (E+P = 1+1, 2+2, 4+4):
    encoder ranks run the ViT, prefill ranks the LLM stages, rank 0 the engine
    and the device tracker. value = cfg3 throughput plateau timed on P0's
    device clock (origin event -> last logits arrival; the max over ranks: no
    rank's work ends later than its data reaches P0)."""
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    from paper_2509_24381_b200 import _native as N
    from paper_2509_24381_b200 import api, ep_launch
    stages, encoders = ep_launch.topology_for(ws)
    dev = 0 if args.ep_same_device else local
    torch.cuda.set_device(dev)
    # NCCL process group over all N ranks (plumbing: ids, barriers, max over
    # ranks) — its init lines prove the N-rank job; gloo when all ranks share
    # one GPU (protocol check on a one-GPU box)
    backend = "gloo" if args.ep_same_device else "nccl"
    dist.init_process_group(backend, device_id=None if backend == "gloo" else torch.device(f"cuda:{dev}"))
    pdev = None if backend == "gloo" else torch.device(f"cuda:{dev}")
    mcfg = api.model_preset("qwen2.5-vl-7b")
    m = {k: getattr(mcfg, k) for k, _ in N.rs_model_config._fields_}
    ctx = api.ep_context(mcfg, rank, stages, encoders, device=dev, max_prompt_tokens=MAX_PROMPT,
                         slot_tokens=1 << 19, kv_tokens=1 << 19, max_chunk_tokens=args.budget,
                         max_encode_tokens=C_TOKENS)
    transport = args.ep_transport
    role = api.ep_role(rank, stages, encoders)
    links = api.ep_links(stages, encoders)
    manifest = {"rank": rank, "role": f"{role[0]}{role[1]}", "device": dev, "transport": transport,
                "links_out": [f"{a}->{b}" for a, b in links if a == rank],
                "links_in": [f"{a}->{b}" for a, b in links if b == rank]}
    print("[ep-manifest] " + json.dumps(manifest), file=sys.stderr, flush=True)

    def make_group(tr):
        ids = ep_launch.share_link_ids(stages, encoders, device=pdev) if tr == "nccl" else None
        shm = ep_launch.shm_name_for_group() if tr == "ipc" else None
        g = api.EpGroup(stages, encoders, tr, rank=rank, device=dev, nccl_ids=ids,
                        slot_bytes=api.ep_slot_bytes(mcfg, args.budget, C_TOKENS), shm_name=shm)
        if tr == "ipc":
            ep_launch.connect_ipc(g)
        dist.barrier()
        return g

    watchdog = threading.Timer(args.ep_watchdog_s, lambda: (
        print(json.dumps({"error": f"EP rank {rank}: no progress within {args.ep_watchdog_s} s "
                                   f"(transport {transport})"}), flush=True), os._exit(3)))
    watchdog.daemon = True
    watchdog.start()
    fallback = None
    try:
        g = make_group(transport)
        ok = 1
    except Exception as e:  # e.g. NCCL refuses the link comms: keep the run on CUDA IPC
        fallback = f"{transport} link setup failed on rank {rank}: {str(e)[:200]}"
        print("[ep] " + fallback, file=sys.stderr, flush=True)
        ok = 0
    flag = torch.tensor([ok], device=pdev) if pdev is not None else torch.tensor([ok])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) == 0:
        if ok:
            g.close()
        transport = "nccl" if transport == "ipc" else "ipc"
        manifest["transport"] = transport
        fallback = fallback or f"a peer's link setup failed: switched to {transport}"
        g = make_group(transport)
    replay = Replayer() if rank == 0 else None

    def runs(workloads, e2e=False, sc=None, check=True):
        """One engine run per workload; rank 0 returns [(log, journal, stats)]."""
        sc = sc or sim_cfg(args, m, stages, encoders)
        out = []
        for wl in workloads:
            if rank != 0:
                g.worker_prepare(ctx, wl, payload_seed=1234, e2e=e2e)
            dist.barrier()
            if rank == 0:
                log, journal, st = g.run(ctx, None, wl, sc, clock="real", e2e=e2e, payload_seed=1234)
                if check:
                    replay.check(wl, sc, log, journal)
                out.append((log, journal, st))
            else:
                g.worker_run(ctx)
        return out

    seeds = CFG3["seeds"]
    tput_wls = [cfg3_workload(seeds[i % len(seeds)], CFG3["tput_rate"], CFG3["tput_duration_s"])
                for i in range(args.steps)]
    lat_wls = [cfg3_workload(s, CFG3["lat_rate"], CFG3["lat_duration_s"]) for s in seeds]
    cfg2_wl = f"0,0,-,{LAYOUT}\n"
    # warm-up: the single request, then the stream
    runs([cfg2_wl] * max(1, args.warmup - 1), check=False)
    runs(tput_wls[:1], check=False)
    watchdog.cancel()
    with ClockSampler(dev, args.clock_sample_ms) as clk:
        timed = runs(tput_wls)
    lat = runs(lat_wls)
    single = runs([cfg2_wl] * 3)
    single_logits = ctx.logits(0) if rank == 0 else None
    timed_e2e = runs(tput_wls[:max(1, args.steps // 2)], e2e=True)
    total_ms = ep_launch.max_over_ranks(sum(st["gpu_ms"] for _, _, st in timed), device=pdev)
    e2e_total = ep_launch.max_over_ranks(sum(st["wall_ms"] for _, _, st in timed_e2e), device=pdev)
    alt = None
    if args.ep_compare and not args.ep_same_device:
        other = "ipc" if transport == "nccl" else "nccl"
        try:
            g2 = make_group(other)
            g_saved, g = g, g2
            alt_runs = runs(tput_wls[:2])
            g = g_saved
            g2.close()
            if rank == 0:
                ss = summarize_stream([(stream_stats(lg), st) for lg, _, st in alt_runs])
                alt = {"transport": other, "tokens_per_s": ss["tokens_per_s"], "steps": len(alt_runs)}
        except Exception as e:  # keep the primary measurement
            alt = {"transport": other, "error": str(e)[:300]}
    if rank == 0:
        tp = summarize_stream([(stream_stats(lg), st) for lg, _, st in timed])
        lt = summarize_stream([(stream_stats(lg), st) for lg, _, st in lat])
        e2 = summarize_stream([(stream_stats(lg), st) for lg, _, st in timed_e2e])
        tokens = sum(stream_stats(lg)["tokens"] for lg, _, _ in timed)
        e2e_tokens = sum(stream_stats(lg)["tokens"] for lg, _, _ in timed_e2e)
        single_ttft = sorted(float(api.parse_decision_log(lg)["req"][0]["ttft"]) for lg, _, _ in single)
        parity = replay.summary()
        if not args.no_parity:
            parity.update(cfg2_logit_parity(*single_logits, f"cuda:{dev}"))
        st_e = timed_e2e[-1][2]
        # pixels are uploaded on the encoder ranks: 4 patches x 1176 bf16 per image token
        px_bytes = sum(4 * n * m["patch_dim"] * 2 for wl in tput_wls[:len(timed_e2e)]
                       for lay in workload_layouts(wl) for n in
                       (int(f[1:]) for f in lay.split("|") if f[0] == "M")) / len(timed_e2e)
        line = {
            "metric": "encode+prefill tokens/s (p50/p99 TTFT ms alongside)",
            "value": tokens / (total_ms / 1e3), "unit": "tokens/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "ttft_ms": {"p50": lt["ttft_ms"]["p50"], "p99": lt["ttft_ms"]["p99"],
                        "mean": lt["ttft_ms"]["mean"], "requests": lt["requests"],
                        "rate_req_s": CFG3["lat_rate"],
                        "percentiles": "nearest-rank over every request of the 3 latency runs"},
            "config": bench_config(args, ws),
            "throughput_plateau": dict(tp, rate_req_s=CFG3["tput_rate"],
                                       value_basis="sum prompt tokens / max-over-ranks device time "
                                                   "(origin -> last logits)"),
            "latency_runs": lt,
            "cfg2": {"ttft_ms": {"p50": nearest_rank(single_ttft, 50), "p99": nearest_rank(single_ttft, 99)},
                     "runs": len(single_ttft), "tokens": PROMPT_TOKENS},
            "e2e": {"value": e2e_tokens / (e2e_total / 1e3), "unit": "tokens/s",
                    "h2d_bytes_per_step": st_e["h2d_bytes"] + px_bytes, "d2h_bytes_per_step": st_e["d2h_bytes"],
                    "h2d_note": "P0's uploads (control, token ids) + the encoder ranks' pixel uploads",
                    "ttft_ms": e2["ttft_ms"],
                    "timing": "host wall clock of each run (H2D pixels from pinned memory on the "
                              "encoder ranks + D2H logits inside)"},
            "gpu_launches": sum(st["kernel_launches"] for _, _, st in timed),
            "gpu_launches_scope": "rank 0 (P0) kernels; worker ranks launch their own",
            "roofline": ep_roofline(m, tput_wls, total_ms, ws),
            "parity": parity,
            "transport_alt": alt,
            "transport": transport, "transport_fallback": fallback,
            "ep_manifest": {"ranks": ws, "process_group": backend, "links": [f"{a}->{b}" for a, b in links],
                            "p2p_communicators": len(links) if transport == "nccl" else 0,
                            "rank0": manifest},
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    dist.barrier()
    g.close()
    ctx.close()
    dist.destroy_process_group()


def ep_roofline(m, workloads, total_ms, ws):
    """Whole-job algorithmic FLOPs of the timed stream (ViT +
    merger per image, dense + causal attention + LM head per request) over the
    max-over-ranks device time, against N x the burst bf16 peak."""
    pk = peaks()[0]
    flops = sum(sum(layout_flops(m, lay)[:2]) for wl in workloads for lay in workload_layouts(wl))
    achieved = flops / (total_ms / 1e3) / 1e12
    return {"bound": "tensor", "unit": "TFLOP/s", "achieved": achieved, "peak": pk * ws,
            "frac": achieved / (pk * ws), "traffic": None,
            "note": "whole job (all N GPUs): model FLOPs of the timed cfg3 stream / device time; "
                    "per-kernel rooflines are in the N=1 line"}


# ---- CPU baseline / reference arm (never loads the product library) -------------------------
def cpu_info():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


_CPU_SAMPLE = {}


def cpu_sample(budget):
    """Times the numpy oracle on one ViT layer (one 896x896 image) and one
    LLM layer (one B-token chunk). Returns (s, FLOPs) per sample."""
    import numpy as np
    from oracle import model_oracle as mo
    if "w" not in _CPU_SAMPLE:  # weight generation once, outside every timed sample
        cfg = mo.ModelConfig.qwen7b(vit_layers=1, vit_fullatt_every=8, llm_layers=1)
        _CPU_SAMPLE.update(cfg=cfg, w=mo.Weights(cfg))
    cfg, w = _CPU_SAMPLE["cfg"], _CPU_SAMPLE["w"]
    vis = mo.VisionOracle(cfg, w)
    patches = vis.patches(1, 0, 0, 1024)
    vis.encode([(1024, patches)], layers=1)
    t0 = time.perf_counter()
    vis.encode([(1024, patches)], layers=1)
    t_vit = time.perf_counter() - t0
    llm = mo.LlmOracle(cfg, w)
    T = min(budget, PROMPT_TOKENS)
    emb = np.random.default_rng(0).standard_normal((T, cfg.llm_dim)).astype(np.float32) * 0.02
    pos = np.repeat(np.arange(T)[:, None], 3, axis=1)
    llm.forward(emb[:16], pos[:16], layers=1)
    t0 = time.perf_counter()
    llm.forward(emb, pos, layers=1)
    t_llm = time.perf_counter() - t0
    vd, ff, P = cfg.vit_dim, cfg.vit_ff, 4096
    f_vit = 2 * P * vd * 1176 + 2 * P * (4 * vd * vd + 3 * vd * ff) + (P // 64) * 4 * 64 * 64 * vd \
        + 2 * 1024 * (4 * vd * 4 * vd + 4 * vd * cfg.llm_dim)
    d, hd = cfg.llm_dim, cfg.llm_head_dim
    qkv = (cfg.llm_q_heads + 2 * cfg.llm_kv_heads) * hd
    f_llm = T * 2 * (d * qkv + cfg.llm_q_heads * hd * d + 3 * d * cfg.llm_ff) + 2 * T * T * cfg.llm_q_heads * hd
    return t_vit, f_vit, t_llm, f_llm


def ref_sched_time(workloads, stages, encoders, budget, policy, reps=200):
    """The reference scheduler itself (oracle/_ref = /root/reference headers,
    -O2): run_simulation on each workload, seconds per workload."""
    from oracle import ref
    sc = ref.sim_config(policy, stages, budget, C_TOKENS, encoders, 3584,
                        beta_enc_ms_per_token=0.01, delta_stage_ms_per_token=0.01)
    return [ref.time_simulate(wl, sc, reps) / 1e9 for wl in workloads]


def cfg1_full_cpu():
    """cfg1 (tiny model, T64|M256|M256|T32|M256|M256, C=256) in full on the
    fp32 oracle: encode + prefill + first-token logits, measured (not
    extrapolated)."""
    from oracle import model_oracle as mo
    cfg = mo.ModelConfig.tiny()
    w = mo.Weights(cfg)
    mo.request_embeddings(cfg, w, 0, CFG1_LAYOUT, 7, 256, vit_layers=1)  # weights warm
    t0 = time.perf_counter()
    emb = mo.request_embeddings(cfg, w, 0, CFG1_LAYOUT, 7, 256)
    llm = mo.LlmOracle(cfg, w)
    h = llm.forward(emb, mo.mrope_positions(mo.parse_layout(CFG1_LAYOUT)))
    llm.first_token_logits(h[-1])
    s = time.perf_counter() - t0
    return {"ttft_ms": s * 1e3, "tokens": 1120, "tokens_per_s": 1120 / s,
            "note": "cfg1 in full on the CPU fp32 oracle (measured)"}


def cpu_request_seconds(m, layouts, rates):
    """Extrapolated CPU seconds for a list of request layouts."""
    t_vit, f_vs, t_llm, f_ls = rates
    tot = 0.0
    for lay in layouts:
        e, p, _ = layout_flops(m, lay)
        tot += t_vit * e / f_vs + t_llm * p / f_ls
    return tot


def cpu_baseline(args, reps=1):
    m = qwen7b_shapes()
    rates = cpu_sample(args.budget)
    req_s = cpu_request_seconds(m, [LAYOUT], rates)
    sched = None
    try:
        sched = ref_sched_time([f"0,0,-,{LAYOUT}\n"], 1, 1, args.budget, args.policy)[0]
    except Exception:  # oracle/_ref not built on this box
        pass
    return dict({"value": PROMPT_TOKENS / req_s, "unit": "tokens/s", "cores": os.cpu_count(),
                 "kind": "port", "ttft_ms": req_s * 1e3,
                 "sample": f"numpy fp32 oracle: 1 ViT layer on one 896x896 image ({rates[0]:.2f} s) + "
                           f"1 LLM layer on a {min(args.budget, PROMPT_TOKENS)}-token chunk "
                           f"({rates[2]:.2f} s), extrapolated by FLOPs to the full cfg2 request "
                           "(extrapolated)",
                 "reference_scheduler_us": None if sched is None else sched * 1e6}, **cpu_info())


def run_reference(args):
    """The reference's CPU path on the same config as our arm at this N. The
    reference (lmmsim) performs no model arithmetic; the model math is the
    fp32 numpy restatement, timed on a bounded sample per step and
    extrapolated; the scheduler is the reference's own code (oracle/_ref)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    # every host thread for the BLAS the numpy oracle runs on: torch.distributed.run
    # exports OMP_NUM_THREADS=1 to its children and BLAS size their pools at
    # import, so rank 0 re-runs this arm in a child with the full count
    nproc = str(os.cpu_count())
    if ws > 1 and os.environ.get("OMP_NUM_THREADS") != nproc and not os.environ.get("RS_REF_CHILD"):
        env = dict(os.environ, OMP_NUM_THREADS=nproc, OPENBLAS_NUM_THREADS=nproc, MKL_NUM_THREADS=nproc,
                   RS_REF_CHILD="1")
        subprocess.run([sys.executable] + sys.argv, env=env, check=True)
        return
    from oracle import ref
    m = qwen7b_shapes()
    ep = ep_mode(args, ws)
    if ep:
        stages, encoders = EP_LAYOUTS[ws]
        seeds = CFG3["seeds"]
        wls = [ref.generate_workload(ref.workload_config(seeds[i % len(seeds)], CFG3["tput_rate"],
                                                         CFG3["tput_duration_s"], CFG3["pattern"],
                                                         CFG3["mm_items"], CFG3["mm_tokens"],
                                                         CFG3["text_tokens"])[0])
               for i in range(args.steps)]
    else:
        stages, encoders = 1, 1
        wls = [f"0,0,-,{LAYOUT}\n"] * args.steps
    for _ in range(args.warmup):
        cpu_sample(args.budget)
    per_step, tokens, ttfts, sched_s = [], 0, [], []
    t_all = time.perf_counter()
    for wl in wls:
        rates = cpu_sample(args.budget)
        lays = workload_layouts(wl)
        sched = ref_sched_time([wl], stages, encoders, args.budget, args.policy, reps=20)[0]
        # one host: requests are served one after another
        acc = 0.0
        for lay in lays:
            acc += cpu_request_seconds(m, [lay], rates)
            ttfts.append(acc * 1e3)
        per_step.append(acc + sched)
        sched_s.append(sched)
        tokens += sum(layout_flops(m, lay)[2] for lay in lays)
    wall = time.perf_counter() - t_all
    value = tokens / sum(per_step)
    ttfts.sort()
    cfg1 = cfg1_full_cpu()
    line = {
        "impl": "reference",
        "metric": "encode+prefill tokens/s (p50/p99 TTFT ms alongside)",
        "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True,
        "scaling": "strong" if ep else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "ttft_ms": {"p50": nearest_rank(ttfts, 50), "p99": nearest_rank(ttfts, 99),
                    "note": "requests served back to back on the host (arrival times ignored)"},
        "config": bench_config(args, ws),
        "cpu_baseline": dict({"value": value, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                              "sample": "per step: numpy fp32 oracle (all host threads via BLAS), 1 ViT "
                                        "layer (4096 patches) + 1 LLM layer (B-token chunk), "
                                        "extrapolated by FLOPs to every request of the step's "
                                        "workload; plus the reference scheduler itself "
                                        "(oracle/_ref run_simulation, measured). The reference "
                                        "(lmmsim) performs no model arithmetic."},
                             **cpu_info()),
        "reference_scheduler_us_per_step": [round(x * 1e6, 2) for x in sched_s],
        "cfg1_full": cfg1,
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--budget", type=int, default=2048, help="Algorithm-2 token budget B")
    ap.add_argument("--policy", default="rserve")
    ap.add_argument("--mode", default="ep", choices=["ep", "replicas"],
                    help="N>1: the EP deployment (default) or N independent co-located replicas")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the fp32-oracle logits check")
    ap.add_argument("--cfg3-steps", type=int, default=3, help="N=1: cfg3 seeds to run (0: skip)")
    ap.add_argument("--clock-sample-ms", type=int, default=200,
                    help="nvidia-smi sampling interval during the timed steps")
    ap.add_argument("--decode-steps", type=int, default=32,
                    help="greedy decode steps after the first token (0: skip)")
    ap.add_argument("--cfg45", type=int, default=1, help="N=1: also run cfg4 (C sweep) and cfg5 (72B) (0: skip)")
    ap.add_argument("--launch-list", action="store_true",
                    help="run only the warm-up + timed steps (for the ncu launch list); no JSON bench line")
    ap.add_argument("--ep", action="store_true", help="(compat) same as --mode ep")
    ap.add_argument("--ep-transport", default="nccl", choices=["ipc", "nccl"])
    ap.add_argument("--ep-compare", action="store_true",
                    help="also time the other EP transport for two steps")
    ap.add_argument("--ep-same-device", action="store_true",
                    help="all EP ranks on cuda:0 (protocol check on a one-GPU box; timing not meaningful)")
    ap.add_argument("--ep-watchdog-s", type=float, default=900.0)
    ap.add_argument("--dry-run", action="store_true",
                    help="launch + roles + manifest only (CPU plumbing check; no GPU work)")
    args = ap.parse_args()
    ws, rank, _ = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args.gpus))
    if "WORLD_SIZE" in os.environ and ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    if args.ep_same_device:
        args.ep_transport = "ipc"  # NCCL refuses two ranks of a communicator on one GPU
    if args.dry_run:
        dry_run(args)
    elif args.impl == "reference":
        run_reference(args)
    elif ep_mode(args, ws):
        run_ep(args)
    else:
        run_ours(args)


def dry_run(args):
    """Plumbing only (CPU, gloo): every rank reports its EP role and links;
    rank 0 prints the manifest line the real run would carry."""
    ws, rank, _ = dist_env()
    import torch.distributed as dist
    if ws > 1:
        dist.init_process_group("gloo")
    if ep_mode(args, ws):
        stages, encoders = EP_LAYOUTS[ws]
        role = ("prefill", rank) if rank < stages else ("encoder", rank - stages)
    else:
        stages, encoders, role = 1, 1, ("colocated", 0)
    mine = {"rank": rank, "role": f"{role[0]}{role[1]}", "pid": os.getpid()}
    allr = [None] * ws
    if ws > 1:
        dist.all_gather_object(allr, mine)
    else:
        allr = [mine]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": ws, "config": bench_config(args, ws),
                          "ranks": allr}))
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
