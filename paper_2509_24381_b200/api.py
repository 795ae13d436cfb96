"""Python mirror of the reference's host API, over the rserve-b200 C-ABI.

Names and meanings follow proj/include/lmmsim/ (simengine.hpp SimConfig,
cost_model.hpp CostModel, workload.hpp WorkloadConfig / RequestTemplate,
token_sched.hpp Policy). Errors are raised as the same exception classes
(errors.hpp:23-80). Everything here is a thin ctypes layer: the scheduling
core is C++ (include/lmmsim/) and the compute is sm_100a CUDA.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from . import _native as N

POLICIES = {"vanilla_pp": 0, "epd_baseline": 1, "intra_only": 2, "rserve": 3}
PATTERNS = {"alternating": 0, "consecutive_mm": 1, "text_first": 2}
WHOLE_REQUEST = 0xFFFFFFFFFFFFFFFF


@dataclass
class CostModel:  # cost_model.hpp:37-45
    alpha_enc_ms: float = 0.0
    beta_enc_ms_per_token: float = 0.0
    eps_tx_ms: float = 0.0
    zeta_tx_ms_per_token: float = 0.0
    gamma_stage_ms: float = 0.0
    delta_stage_ms_per_token: float = 0.0
    kappa_attn_ms: float = 0.0
    tp_speedup: float = 1.0


@dataclass
class SimConfig:  # simengine.hpp:48-75
    policy: str = "rserve"
    pipeline_mode: Optional[str] = None  # "cpp" | "vanilla" | None (policy default)
    stages: int = 4
    token_budget: int = 512
    embedding_batch_tokens: int = 1024  # or WHOLE_REQUEST
    encoder_workers: int = 1
    release_at: str = "last_stage"
    hidden_size: int = 4096
    cost: CostModel = field(default_factory=CostModel)

    def to_c(self) -> N.rs_sim_config:
        c = N.rs_sim_config()
        if self.policy not in POLICIES:
            raise N.ConfigError(f"policy: unknown name '{self.policy}' (expected vanilla_pp, "
                                "epd_baseline, intra_only or rserve)")
        c.policy = POLICIES[self.policy]
        c.pipeline_mode = {None: -1, "cpp": 0, "vanilla": 1}[self.pipeline_mode]
        c.stages = self.stages
        c.encoder_workers = self.encoder_workers
        c.token_budget = self.token_budget
        c.embedding_batch_tokens = self.embedding_batch_tokens
        c.release_at = 0 if self.release_at == "first_stage" else 1
        c.hidden_size = self.hidden_size
        for k in ("alpha_enc_ms", "beta_enc_ms_per_token", "eps_tx_ms", "zeta_tx_ms_per_token",
                  "gamma_stage_ms", "delta_stage_ms_per_token", "kappa_attn_ms", "tp_speedup"):
            setattr(c.cost, k, getattr(self.cost, k))
        return c


@dataclass
class IntDistribution:
    lo: int = 1
    hi: Optional[int] = None  # None = constant(lo)

    def to_c(self) -> N.rs_int_dist:
        d = N.rs_int_dist()
        d.uniform = 0 if self.hi is None else 1
        d.lo = self.lo
        d.hi = self.lo if self.hi is None else self.hi
        return d


@dataclass
class RequestTemplate:  # workload.hpp:71-107
    pattern: str = "alternating"
    num_mm_items: IntDistribution = field(default_factory=lambda: IntDistribution(1))
    mm_item_tokens: IntDistribution = field(default_factory=lambda: IntDistribution(512))
    text_segment_tokens: IntDistribution = field(default_factory=lambda: IntDistribution(128))
    probability: float = 1.0


@dataclass
class WorkloadConfig:  # workload.hpp:109-136
    arrival_rate: float = 1.0
    duration_s: float = 10.0
    seed: int = 0
    templates: List[RequestTemplate] = field(default_factory=lambda: [RequestTemplate()])
    slo_ttft_ms: Optional[float] = None

    def to_c(self):
        arr = (N.rs_template * len(self.templates))()
        for i, t in enumerate(self.templates):
            arr[i].pattern = PATTERNS[t.pattern]
            arr[i].num_mm_items = t.num_mm_items.to_c()
            arr[i].mm_item_tokens = t.mm_item_tokens.to_c()
            arr[i].text_segment_tokens = t.text_segment_tokens.to_c()
            arr[i].probability = t.probability
        w = N.rs_workload_config()
        w.arrival_rate = self.arrival_rate
        w.duration_s = self.duration_s
        w.seed = self.seed
        w.templates = C.cast(arr, C.POINTER(N.rs_template))
        w.n_templates = len(self.templates)
        w.has_slo = 0 if self.slo_ttft_ms is None else 1
        w.slo_ttft_ms = self.slo_ttft_ms or 0.0
        return w, arr  # keep `arr` alive


def _dist_from_json(j) -> IntDistribution:
    if "constant" in j:
        return IntDistribution(int(j["constant"]))
    lo, hi = j["uniform"]
    return IntDistribution(int(lo), int(hi))


def experiment_from_json(j: dict):
    """(WorkloadConfig template, SimConfig, policies, rates, seeds, slo) from an
    experiment JSON (config.hpp:171-300 key names)."""
    w = j["workload"]
    if "file" in w:  # fixed workload file (config.hpp:184-188): no generator
        templates = []
        w = dict(w, duration_s=0.0, templates=[])
    templates = [RequestTemplate(t["pattern"], _dist_from_json(t["num_mm_items"]),
                                 _dist_from_json(t["mm_item_tokens"]),
                                 _dist_from_json(t["text_segment_tokens"]), float(t["probability"]))
                 for t in w["templates"]]
    cm = j["cost_model"]
    cost = CostModel(**{k: float(v) for k, v in cm.items()})
    c = j["embedding_batch_size_C"]
    sim = SimConfig(stages=int(j["stages"]), token_budget=int(j["token_budget_B"]),
                    embedding_batch_tokens=WHOLE_REQUEST if c == "whole_request" else int(c),
                    encoder_workers=int(j.get("encoder_workers", 1)),
                    release_at=j.get("release_at", "last_stage"),
                    pipeline_mode=j.get("pipeline_mode"), hidden_size=int(j.get("hidden_size", 4096)),
                    cost=cost)
    slo = j.get("slo_ttft_ms")
    wl = WorkloadConfig(duration_s=float(w["duration_s"]), templates=templates,
                        slo_ttft_ms=None if slo is None else float(slo))
    return wl, sim, list(j["policies"]), [float(r) for r in j["rates"]], \
        [int(s) for s in j["seeds"]], slo


def _out():
    return C.c_char_p()


def generate_workload(cfg: WorkloadConfig) -> str:
    w, keep = cfg.to_c()
    out = _out()
    N.check(N.lib.rs_generate_workload(C.byref(w), C.byref(out)))
    return N.take_string(out)


def generate_payload(workload: str, seed: int) -> str:
    """Payload file (rserve.h "payload files") for a workload:
    per image a grid drawn among its token count's factorisations (aspect <= 4)
    and a pixel seed, per text segment a token-id seed, all keyed by `seed`."""
    out = _out()
    N.check(N.lib.rs_payload_generate(workload.encode(), seed, C.byref(out)))
    return N.take_string(out)


def validate_payload(workload: str, payload: str, vocab: int) -> str:
    """Checks a payload file against a workload; returns its normalised text.
    Raises InputError ("payload line N: ..." / "payload: request ...")."""
    out = _out()
    N.check(N.lib.rs_payload_validate(workload.encode(), payload.encode(), vocab, C.byref(out)))
    return N.take_string(out)


def simulate(workload: str, cfg: SimConfig) -> Tuple[str, str]:
    """run_simulation on the analytic cost model -> (decision log, journal)."""
    res, jr = _out(), _out()
    c = cfg.to_c()
    N.check(N.lib.rs_simulate(workload.encode(), C.byref(c), C.byref(res), C.byref(jr)))
    return N.take_string(res), N.take_string(jr)


def experiment_cell(wcfg: WorkloadConfig, cfg: SimConfig, slo_ttft_ms: Optional[float]) -> str:
    w, keep = wcfg.to_c()
    c = cfg.to_c()
    out = _out()
    N.check(N.lib.rs_experiment_cell(C.byref(w), C.byref(c),
                                     -1.0 if slo_ttft_ms is None else float(slo_ttft_ms),
                                     C.byref(out)))
    return N.take_string(out)


def plan_batches(layout: str, request_id: int, c_tokens: int) -> str:
    out = _out()
    N.check(N.lib.rs_plan_batches(layout.encode(), request_id, c_tokens, C.byref(out)))
    return N.take_string(out)


def parse_decision_log(text: str) -> Dict[str, list]:
    """Decision log text -> {'result': dict, 'req': [...], 'slice': [...], ...}."""
    out: Dict[str, list] = {}
    for line in text.splitlines():
        kind, *fields = line.split(" ")
        rec = {}
        for f in fields:
            k, _, v = f.partition("=")
            rec[k] = v
        out.setdefault(kind, []).append(rec)
    return out


# ---------------------------------------------------------------------------
MODEL_PRESETS = {"tiny": 0, "qwen2.5-vl-7b": 1, "qwen2.5-vl-72b-llm": 2}


def model_preset(name: str, **overrides) -> N.rs_model_config:
    m = N.rs_model_config()
    N.check(N.lib.rs_model_preset(MODEL_PRESETS[name], C.byref(m)))
    for k, v in overrides.items():
        setattr(m, k, v)
    return m


class Pipeline:
    """One device context (rs_ctx): weights, embedding slots, KV pools."""

    def __init__(self, model: N.rs_model_config, device: int = 0, max_prompt_tokens: int = 32768,
                 slot_tokens: int = 65536, kv_tokens: int = 65536, max_chunk_tokens: int = 2048,
                 max_encode_tokens: int = 2048, layer_begin: int = 0, layer_end: int = 0,
                 with_vit: bool = True, with_lm_head: bool = True, tp_size: int = 1,
                 tp_rank: int = 0, tp_group: bool = False):
        self.model = model
        o = N.rs_ctx_options()
        o.device = device
        o.max_prompt_tokens = max_prompt_tokens
        o.slot_tokens = slot_tokens
        o.kv_tokens = kv_tokens
        o.max_chunk_tokens = max_chunk_tokens
        o.max_encode_tokens = max_encode_tokens
        o.layer_begin = layer_begin
        o.layer_end = layer_end
        o.with_vit = int(with_vit)
        o.with_lm_head = int(with_lm_head)
        o.tp_size = tp_size
        o.tp_rank = tp_rank
        o.tp_group = int(tp_group)
        self.opts = o
        h = C.c_void_p()
        N.check(N.lib.rs_ctx_create(C.byref(model), C.byref(o), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            N.check(N.lib.rs_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # tracker data plane -------------------------------------------------------
    def request_create(self, req_id: int, layout: str, text_ids=None):
        ptr = None
        if text_ids is not None:
            import numpy as np
            arr = np.ascontiguousarray(text_ids, dtype=np.int32)
            self._keep = arr
            ptr = arr.ctypes.data
        N.check(N.lib.rs_request_create(self.h, req_id, layout.encode(), ptr))

    def mark_encoded(self, req_id: int, start: int, end: int, emb_dev_ptr: int):
        N.check(N.lib.rs_mark_encoded(self.h, req_id, start, end, emb_dev_ptr))

    def schedulable(self, req_id: int) -> Tuple[int, int]:
        a, b = C.c_uint64(), C.c_uint64()
        N.check(N.lib.rs_schedulable(self.h, req_id, C.byref(a), C.byref(b)))
        return a.value, b.value

    def advance_prefill(self, req_id: int, n: int) -> Tuple[int, int]:
        a, b = C.c_uint64(), C.c_uint64()
        N.check(N.lib.rs_advance_prefill(self.h, req_id, n, C.byref(a), C.byref(b)))
        return a.value, b.value

    def release(self, req_id: int, start: int, end: int):
        N.check(N.lib.rs_release(self.h, req_id, start, end))

    def erase(self, req_id: int):
        N.check(N.lib.rs_request_erase(self.h, req_id))

    def read_bitmap(self, req_id: int, total_tokens: int):
        import numpy as np
        out = np.zeros((total_tokens + 31) // 32, dtype=np.uint32)
        N.check(N.lib.rs_read_bitmap(self.h, req_id, out.ctypes.data, out.size))
        return out

    def read_slots(self, req_id: int, start: int, end: int):
        import numpy as np
        d = self.model.llm_dim
        out = np.zeros((end - start, d), dtype=np.uint16)
        N.check(N.lib.rs_read_slots(self.h, req_id, start, end, out.ctypes.data))
        return out

    def tracker_stats(self, req_id: int) -> Dict[str, int]:
        a = (C.c_uint64 * 6)()
        N.check(N.lib.rs_tracker_stats(self.h, req_id, a))
        keys = ("live", "peak_live", "released", "frontier", "schedulable", "all_encoded")
        return dict(zip(keys, list(a)))

    # compute --------------------------------------------------------------------
    def encode(self, items: Sequence[Tuple[int, int]], patches_ptr: int, on_host: bool,
               out_ptr: Optional[int] = None) -> int:
        """ViT forward of one Algorithm-1 batch; returns the output device pointer."""
        arr = (C.c_uint64 * (2 * len(items)))(*[v for it in items for v in it])
        out = C.c_void_p(out_ptr)
        N.check(N.lib.rs_encode(self.h, arr, len(items), patches_ptr, int(on_host), C.byref(out)))
        return out.value

    # asynchronous seam (include/rserve.h "caller-owned event loop") -----------
    def request_create_segments(self, req_id: int, segments: Sequence[Tuple[str, int]], text_ids=None):
        arr = (N.rs_segment * len(segments))(*[N.rs_segment(0 if k == "T" else 1, n) for k, n in segments])
        ptr = None
        if text_ids is not None:
            import numpy as np
            self._keep = np.ascontiguousarray(text_ids, dtype=np.int32)
            ptr = self._keep.ctypes.data
        N.check(N.lib.rs_request_create_segments(self.h, req_id, arr, len(segments), ptr))

    def encode_batch_async(self, req_id: int, items: Sequence[Tuple[int, int]], patches_ptr: int,
                           on_host: bool, tag: int, stream: Optional[int] = None):
        arr = (C.c_uint64 * (2 * len(items)))(*[v for it in items for v in it])
        N.check(N.lib.rs_encode_batch_async(self.h, req_id, arr, len(items), patches_ptr, int(on_host),
                                            stream, tag))

    def embeddings_ready(self, tag: int):
        N.check(N.lib.rs_embeddings_ready(self.h, tag))

    def prefill_chunk_async(self, slices: Sequence[Tuple[int, int, int]], tag: int, stream: Optional[int] = None):
        arr = (C.c_uint64 * (3 * len(slices)))(*[v for s in slices for v in s])
        N.check(N.lib.rs_prefill_chunk_async(self.h, arr, len(slices), stream, tag))

    def release_async(self, req_id: int, start: int, end: int, after_tag: int):
        N.check(N.lib.rs_release_async(self.h, req_id, start, end, after_tag))

    def erase_async(self, req_id: int, after_tag: int):
        N.check(N.lib.rs_request_erase_async(self.h, req_id, after_tag))

    def poll(self, wait: bool = False, cap: int = 64) -> List[Tuple[int, int, int, float]]:
        """Completed launches: [(kind, stage, tag, time_ms)] in completion order."""
        ev = (N.rs_event * cap)()
        n = C.c_int32()
        N.check(N.lib.rs_poll(self.h, ev, cap, int(wait), C.byref(n)))
        return [(ev[i].kind, ev[i].stage, ev[i].tag, ev[i].time_ms) for i in range(n.value)]

    def prefill_chunk(self, slices: Sequence[Tuple[int, int, int]]):
        arr = (C.c_uint64 * (3 * len(slices)))(*[v for s in slices for v in s])
        N.check(N.lib.rs_prefill_chunk(self.h, arr, len(slices)))

    def logits(self, req_id: int):
        import numpy as np
        out = np.zeros(self.model.vocab, dtype=np.float32)
        am = C.c_int32()
        N.check(N.lib.rs_logits(self.h, req_id, out.ctypes.data, C.byref(am)))
        return out, am.value

    def synchronize(self):
        N.check(N.lib.rs_synchronize(self.h))

    def decode(self, request_ids: Sequence[int], steps: int, want_logits: bool = False):
        """Greedy decode after the first token (rserve.h rs_decode) for requests
        kept by run(keep_kv=True) -> (tokens [steps, n] int32, logits
        [steps, n, vocab] float32 or None, device ms)."""
        import numpy as np
        n = len(request_ids)
        ids = (C.c_uint64 * n)(*request_ids)
        toks = np.zeros((steps, n), dtype=np.int32)
        logits = np.zeros((steps, n, self.model.vocab), dtype=np.float32) if want_logits else None
        ms = C.c_double()
        N.check(N.lib.rs_decode(self.h, ids, n, steps, toks.ctypes.data_as(C.POINTER(C.c_int32)),
                                logits.ctypes.data_as(C.POINTER(C.c_float)) if logits is not None else None,
                                C.byref(ms)))
        return toks, logits, ms.value

    def decode_release(self, request_id: int):
        N.check(N.lib.rs_decode_release(self.h, request_id))

    # tensor parallelism across GPUs (rserve.h rs_tp_*)
    def tp_buffer(self):
        """(device pointer, 64-byte CUDA IPC handle) of this rank's exchange buffer."""
        ptr = C.c_void_p()
        handle = (C.c_uint8 * 64)()
        N.check(N.lib.rs_tp_buffer(self.h, C.byref(ptr), handle))
        return ptr.value, bytes(handle)

    def tp_connect(self, ptrs, handles=None):
        """ptrs[r]: rank r's buffer when it lives in this process (else None);
        handles[r]: its IPC handle (64 bytes) otherwise."""
        T = len(ptrs)
        arr = (C.c_void_p * T)(*[p or None for p in ptrs])
        hb = None
        if handles is not None:
            hb = (C.c_uint8 * (64 * T)).from_buffer_copy(b"".join(h or bytes(64) for h in handles))
        N.check(N.lib.rs_tp_connect(self.h, arr, hb))

    def kv_request_create(self, req_id: int, layout: str):
        N.check(N.lib.rs_kv_request_create(self.h, req_id, layout.encode()))

    def tp_prefill(self, slices, x_ptr: int, stream: int = 0):
        """Enqueue one chunk on this TP rank: slices [(id, start, end)], x_ptr the
        chunk's input rows [M, d] bf16 (device; updated in place)."""
        flat = (C.c_uint64 * (3 * len(slices)))(*[v for s in slices for v in s])
        N.check(N.lib.rs_tp_prefill(self.h, flat, len(slices), x_ptr, stream or None))

    def tp_logits(self, req_id: int):
        import numpy as np
        out = np.empty(self.model.vocab, dtype=np.float32)
        am = C.c_int32()
        N.check(N.lib.rs_tp_logits(self.h, req_id, out.ctypes.data_as(C.POINTER(C.c_float)), C.byref(am)))
        return out, am.value

    # PD (prefill -> decode) KV transfer (rserve.h rs_kv_export / rs_kv_import)
    def kv_image_bytes(self, tokens: int) -> int:
        out = C.c_uint64()
        N.check(N.lib.rs_kv_image_bytes(self.h, tokens, C.byref(out)))
        return out.value

    def kv_export(self, request_id: int, dst_ptr: int, cap_bytes: int, stream: int = 0) -> "N.rs_kv_meta":
        """Packs a kept request's KV (+ first token) into the device buffer
        dst_ptr; enqueued on `stream` (0: the context's aux stream)."""
        meta = N.rs_kv_meta()
        N.check(N.lib.rs_kv_export(self.h, request_id, dst_ptr, cap_bytes, C.byref(meta), stream or None))
        return meta

    def kv_import(self, request_id: int, meta: "N.rs_kv_meta", src_ptr: int, stream: int = 0):
        """Creates kept request `request_id` from a KV image (device pointer)."""
        N.check(N.lib.rs_kv_import(self.h, request_id, C.byref(meta), src_ptr, stream or None))

    def run(self, workload: str, cfg: SimConfig, clock: str = "lockstep", e2e: bool = False,
            payload_seed: int = 7, serialize: bool = False, payload: Optional[str] = None,
            keep_kv: bool = False):
        """Engine run on this device -> (decision log, journal, stats dict).
        `payload`: optional payload file text (grids, pixel seeds, token ids).
        `keep_kv`: completed requests stay on the device for decode()."""
        o = N.rs_run_options()
        o.clock = 1 if clock == "real" else 0
        o.e2e = int(e2e)
        o.serialize = int(serialize)
        o.payload_seed = payload_seed
        o.payload_text = payload.encode() if payload is not None else None
        o.keep_kv = int(keep_kv)
        res, jr = _out(), _out()
        st = N.rs_run_stats()
        c = cfg.to_c()
        N.check(N.lib.rs_engine_run(self.h, workload.encode(), C.byref(c), C.byref(o),
                                    C.byref(res), C.byref(jr), C.byref(st)))
        stats = {k: getattr(st, k) for k, _ in N.rs_run_stats._fields_}
        return N.take_string(res), N.take_string(jr), stats


# ---- EP disaggregation (include/rserve.h "EP disaggregation") -------------------------------
def ep_links(stages: int, encoders: int) -> List[Tuple[int, int]]:
    """Directed links (src, dst) of an EP topology, in creation order."""
    n = C.c_int32()
    N.check(N.lib.rs_ep_links(stages, encoders, C.byref(n), None))
    pairs = (C.c_int32 * (2 * n.value))()
    N.check(N.lib.rs_ep_links(stages, encoders, C.byref(n), pairs))
    return [(pairs[2 * i], pairs[2 * i + 1]) for i in range(n.value)]


def ep_role(rank: int, stages: int, encoders: int) -> Tuple[str, int]:
    """("prefill", s) for P_s = rank s; ("encoder", w) for E_w = rank stages + w."""
    if not 0 <= rank < stages + encoders:
        raise N.ConfigError(f"rank {rank} outside an EP world of {stages + encoders}")
    return ("prefill", rank) if rank < stages else ("encoder", rank - stages)


def ep_stage_layers(stage: int, stages: int, layers: int) -> Tuple[int, int]:
    """LLM layers [begin, end) of prefill stage `stage` (even split)."""
    return layers * stage // stages, layers * (stage + 1) // stages


def ep_context(model: N.rs_model_config, rank: int, stages: int, encoders: int, device: int = 0,
               **opts) -> "Pipeline":
    """The device context of EP rank `rank`: ViT only on encoder ranks; the
    stage's LLM layers on prefill ranks (LM head on the last one)."""
    role, idx = ep_role(rank, stages, encoders)
    L = model.llm_layers
    if role == "encoder":
        o = dict(opts, with_vit=True, with_lm_head=False, layer_begin=L, layer_end=L,
                 kv_tokens=0, slot_tokens=0, max_chunk_tokens=64)
        return Pipeline(model, device=device, **o)
    lb, le = ep_stage_layers(idx, stages, L)
    o = dict(opts, with_vit=False, with_lm_head=(idx == stages - 1), layer_begin=lb, layer_end=le)
    if idx > 0:
        o["slot_tokens"] = 0
    return Pipeline(model, device=device, **o)


def ep_ctrl_pack(text: str) -> bytes:
    """Text form of a control message -> its 32 KB wire bytes."""
    buf = C.create_string_buffer(N.EP_CTRL_BYTES)
    N.check(N.lib.rs_ep_ctrl_pack(text.encode(), buf, N.EP_CTRL_BYTES))
    return buf.raw


def ep_ctrl_unpack(msg: bytes) -> str:
    out = _out()
    N.check(N.lib.rs_ep_ctrl_unpack(msg, len(msg), C.byref(out)))
    return N.take_string(out)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    N.check(N.lib.rs_nccl_unique_id(buf))
    return buf.raw


def ep_slot_bytes(model: N.rs_model_config, max_chunk_tokens: int = 2048,
                  max_encode_tokens: int = 2048) -> int:
    """Largest EP message: a chunk residual, an encode batch's embeddings, a
    logits row or a control message."""
    d = model.llm_dim
    return max(max_chunk_tokens * d * 2, max_encode_tokens * d * 2, model.vocab * 4, N.EP_CTRL_BYTES)


class EpGroup:
    """EP endpoints of one rank (or of all ranks, for loopback).

    transport: "loopback" — every rank a thread of this process (one GPU is
    enough); "ipc" — one process per rank, CUDA-IPC mailboxes in each
    receiver's HBM written over NVLink (call connect() with all ranks' export()
    blobs); "nccl" — one process per GPU, one 2-rank communicator per link
    (`nccl_ids`: rank 0's ncclUniqueIds, one per ep_links() entry)."""

    def __init__(self, stages: int, encoders: int, transport: str = "loopback", rank: int = 0,
                 device: int = 0, nccl_ids: Optional[bytes] = None, slot_bytes: int = 0,
                 shm_name: Optional[str] = None):
        self.stages, self.encoders, self.transport = stages, encoders, transport
        o = N.rs_ep_options()
        o.stages, o.encoders = stages, encoders
        o.transport = {"loopback": 0, "nccl": 1, "ipc": 2}[transport]
        o.rank, o.device = rank, device
        self._ids = C.create_string_buffer(nccl_ids, len(nccl_ids)) if nccl_ids else None
        o.nccl_ids = C.cast(self._ids, C.c_void_p) if self._ids is not None else None
        o.slot_bytes = slot_bytes
        o.shm_name = shm_name.encode() if shm_name else None
        h = C.c_void_p()
        N.check(N.lib.rs_ep_create(C.byref(o), C.byref(h)))
        self.h = h

    def export(self) -> bytes:
        """IPC: this rank's receive handles."""
        n = C.c_uint64()
        N.check(N.lib.rs_ep_ipc_export(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(max(1, n.value))
        N.check(N.lib.rs_ep_ipc_export(self.h, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    def connect(self, blobs: Sequence[bytes]):
        """IPC: map the peers' mailboxes (blobs of all ranks, rank order)."""
        sizes = (C.c_uint64 * len(blobs))(*[len(b) for b in blobs])
        joined = b"".join(blobs)
        N.check(N.lib.rs_ep_ipc_connect(self.h, joined, sizes, len(blobs)))

    def close(self):
        if self.h:
            N.check(N.lib.rs_ep_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, p0: "Pipeline", workers: Optional[Sequence["Pipeline"]], workload: str,
            cfg: SimConfig, clock: str = "lockstep", e2e: bool = False, payload_seed: int = 7):
        """Engine run on P0 (rank 0) -> (decision log, journal, stats).
        Loopback: `workers` are the contexts of ranks 1..world-1."""
        o = N.rs_run_options()
        o.clock = 1 if clock == "real" else 0
        o.e2e = int(e2e)
        o.payload_seed = payload_seed
        arr = None
        if workers is not None:
            arr = (C.c_void_p * len(workers))(*[w.h.value for w in workers])
        res, jr = _out(), _out()
        st = N.rs_run_stats()
        c = cfg.to_c()
        N.check(N.lib.rs_ep_engine_run(self.h, p0.h, arr, workload.encode(), C.byref(c), C.byref(o),
                                       C.byref(res), C.byref(jr), C.byref(st)))
        p0._ep_logits = True
        stats = {k: getattr(st, k) for k, _ in N.rs_run_stats._fields_}
        return N.take_string(res), N.take_string(jr), stats

    def worker_prepare(self, ctx: "Pipeline", workload: str, payload_seed: int = 7, e2e: bool = False):
        N.check(N.lib.rs_ep_worker_prepare(self.h, ctx.h, workload.encode(), payload_seed, int(e2e)))

    def worker_run(self, ctx: "Pipeline"):
        N.check(N.lib.rs_ep_worker_run(self.h, ctx.h))


def engine_cell(ctx: "Pipeline", wcfg: WorkloadConfig, cfg: SimConfig, slo_ttft_ms: Optional[float] = None,
                clock: str = "real", payload_seed: int = 7, ep: Optional[EpGroup] = None,
                workers: Optional[Sequence["Pipeline"]] = None) -> Tuple[str, str, Dict]:
    """One experiment cell on the device engine: the report CSV
    row of experiment_cell() and the Chrome trace, from measured completions
    (clock="real") or the cost model's event order (clock="lockstep")."""
    o = N.rs_run_options()
    o.clock = 1 if clock == "real" else 0
    o.payload_seed = payload_seed
    arr = (C.c_void_p * len(workers))(*[w.h.value for w in workers]) if workers else None
    row, trace = _out(), _out()
    st = N.rs_run_stats()
    (wc, _keep), c = wcfg.to_c(), cfg.to_c()
    N.check(N.lib.rs_engine_cell(ctx.h, ep.h if ep is not None else None, arr, C.byref(wc), C.byref(c),
                                 -1.0 if slo_ttft_ms is None else slo_ttft_ms, C.byref(o),
                                 C.byref(row), C.byref(trace), C.byref(st)))
    return N.take_string(row), N.take_string(trace), {k: getattr(st, k) for k, _ in N.rs_run_stats._fields_}
