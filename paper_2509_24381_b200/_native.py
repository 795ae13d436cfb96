"""ctypes binding of the rserve-b200 C-ABI (include/rserve.h, include/rserve_ops.h).

The native library is built in-tree (``paper_2509_24381_b200/_lib/``) by
``__graft_entry__.build()`` / ``make -C paper_2509_24381_b200/csrc``. There is
no Python or CPU fallback for any product path: if the library is missing,
importing this module raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "librserve_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"rserve-b200 native library not built: {LIB_PATH} missing "
        "(run `python -c 'import __graft_entry__ as g; g.build()'`)")

lib = C.CDLL(LIB_PATH)

# ---- status -----------------------------------------------------------------
RS_OK = 0
STATUS_NAMES = {
    1: "ConfigError", 2: "RegistryError", 3: "DoubleEncodeError", 4: "AlignmentError",
    5: "DependencyViolation", 6: "InputError", 7: "DataError", 8: "IoError",
    9: "InternalError", 10: "SimError", 20: "CudaError", 21: "NcclError", 99: "UnknownError",
}


class SimError(RuntimeError):
    """Root of the mirrored reference exception hierarchy (errors.hpp:23-80)."""


def _mk(name):
    return type(name, (SimError,), {})


ConfigError = _mk("ConfigError")
RegistryError = _mk("RegistryError")
DoubleEncodeError = _mk("DoubleEncodeError")
AlignmentError = _mk("AlignmentError")
DependencyViolation = _mk("DependencyViolation")
InputError = _mk("InputError")
DataError = _mk("DataError")
IoError = _mk("IoError")
InternalError = _mk("InternalError")


class DeviceError(RuntimeError):
    """CUDA / NCCL failure inside the native library."""


_EXC = {1: ConfigError, 2: RegistryError, 3: DoubleEncodeError, 4: AlignmentError,
        5: DependencyViolation, 6: InputError, 7: DataError, 8: IoError, 9: InternalError,
        10: SimError, 20: DeviceError, 21: DeviceError}

lib.rs_last_error.restype = C.c_char_p
lib.rs_version.restype = C.c_char_p
lib.rs_free.argtypes = [C.c_void_p]


def check(status: int) -> None:
    if status != RS_OK:
        msg = lib.rs_last_error().decode()
        raise _EXC.get(status, RuntimeError)(msg)


def take_string(p: C.c_char_p) -> str:
    """Copy a malloc'd char* returned by the library and free it."""
    if not p:
        return ""
    s = C.cast(p, C.c_char_p).value.decode()
    lib.rs_free(p)
    return s


# ---- POD structs (mirror include/rserve.h) ------------------------------------------
class rs_cost_model(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "alpha_enc_ms", "beta_enc_ms_per_token", "eps_tx_ms", "zeta_tx_ms_per_token",
        "gamma_stage_ms", "delta_stage_ms_per_token", "kappa_attn_ms", "tp_speedup")]


class rs_sim_config(C.Structure):
    _fields_ = [("policy", C.c_int32), ("pipeline_mode", C.c_int32), ("stages", C.c_int32),
                ("encoder_workers", C.c_int32), ("token_budget", C.c_uint64),
                ("embedding_batch_tokens", C.c_uint64), ("release_at", C.c_int32),
                ("hidden_size", C.c_uint32), ("cost", rs_cost_model)]


class rs_int_dist(C.Structure):
    _fields_ = [("uniform", C.c_int32), ("lo", C.c_uint64), ("hi", C.c_uint64)]


class rs_template(C.Structure):
    _fields_ = [("pattern", C.c_int32), ("num_mm_items", rs_int_dist),
                ("mm_item_tokens", rs_int_dist), ("text_segment_tokens", rs_int_dist),
                ("probability", C.c_double)]


class rs_workload_config(C.Structure):
    _fields_ = [("arrival_rate", C.c_double), ("duration_s", C.c_double), ("seed", C.c_uint64),
                ("templates", C.POINTER(rs_template)), ("n_templates", C.c_int32),
                ("has_slo", C.c_int32), ("slo_ttft_ms", C.c_double)]


class rs_model_config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "vit_dim", "vit_layers", "vit_heads", "vit_ff", "vit_window", "vit_fullatt_every",
        "patch_dim", "llm_dim", "llm_layers", "llm_q_heads", "llm_kv_heads", "llm_head_dim",
        "llm_ff", "vocab")] + [("rope_theta_llm", C.c_float), ("rope_theta_vit", C.c_float),
                               ("rms_eps", C.c_float), ("weight_seed", C.c_uint64)]


class rs_ctx_options(C.Structure):
    _fields_ = [("device", C.c_int32), ("max_prompt_tokens", C.c_uint64),
                ("slot_tokens", C.c_uint64), ("kv_tokens", C.c_uint64),
                ("max_chunk_tokens", C.c_uint64), ("max_encode_tokens", C.c_uint64),
                ("layer_begin", C.c_int32), ("layer_end", C.c_int32), ("with_vit", C.c_int32),
                ("with_lm_head", C.c_int32), ("tp_size", C.c_int32), ("tp_rank", C.c_int32),
                ("tp_group", C.c_int32)]


class rs_run_options(C.Structure):
    _fields_ = [("clock", C.c_int32), ("e2e", C.c_int32), ("serialize", C.c_int32),
                ("payload_seed", C.c_uint64), ("payload_text", C.c_char_p), ("keep_kv", C.c_int32)]


class rs_run_stats(C.Structure):
    _fields_ = [("wall_ms", C.c_double), ("gpu_ms", C.c_double), ("h2d_bytes", C.c_uint64),
                ("d2h_bytes", C.c_uint64), ("kernel_launches", C.c_uint64),
                ("encode_gpu_ms", C.c_double), ("prefill_gpu_ms", C.c_double),
                ("host_max_gap_ms", C.c_double), ("host_last_seen_ms", C.c_double),
                ("host_max_call_ms", C.c_double), ("host_max_call_kind", C.c_int32),
                ("reserved0", C.c_int32), ("host_max_launch_ms", C.c_double),
                ("host_finish_sync_ms", C.c_double)]


def _sig(name, argtypes, restype=C.c_int):
    fn = getattr(lib, name, None)
    if fn is None:
        return None
    fn.argtypes = argtypes
    fn.restype = restype
    return fn


PCHAR = C.POINTER(C.c_char_p)
_sig("rs_generate_workload", [C.POINTER(rs_workload_config), PCHAR])
_sig("rs_simulate", [C.c_char_p, C.POINTER(rs_sim_config), PCHAR, PCHAR])
_sig("rs_experiment_cell", [C.POINTER(rs_workload_config), C.POINTER(rs_sim_config),
                            C.c_double, PCHAR])
_sig("rs_plan_batches", [C.c_char_p, C.c_uint64, C.c_uint64, PCHAR])
_sig("rs_model_preset", [C.c_int32, C.POINTER(rs_model_config)])
_sig("rs_ctx_create", [C.POINTER(rs_model_config), C.POINTER(rs_ctx_options),
                       C.POINTER(C.c_void_p)])
_sig("rs_ctx_destroy", [C.c_void_p])
_sig("rs_request_create", [C.c_void_p, C.c_uint64, C.c_char_p, C.c_void_p])
_sig("rs_mark_encoded", [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p])
_sig("rs_schedulable", [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)])
_sig("rs_advance_prefill", [C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64),
                            C.POINTER(C.c_uint64)])
_sig("rs_release", [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64])
_sig("rs_request_erase", [C.c_void_p, C.c_uint64])
_sig("rs_read_bitmap", [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64])
_sig("rs_read_slots", [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p])
_sig("rs_tracker_stats", [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)])
_sig("rs_encode", [C.c_void_p, C.POINTER(C.c_uint64), C.c_int32, C.c_void_p, C.c_int32,
                   C.POINTER(C.c_void_p)])
_sig("rs_prefill_chunk", [C.c_void_p, C.POINTER(C.c_uint64), C.c_int32])
_sig("rs_logits", [C.c_void_p, C.c_uint64, C.c_void_p, C.POINTER(C.c_int32)])
_sig("rs_synchronize", [C.c_void_p])
_sig("rs_engine_run", [C.c_void_p, C.c_char_p, C.POINTER(rs_sim_config),
                       C.POINTER(rs_run_options), PCHAR, PCHAR, C.POINTER(rs_run_stats)])
_sig("rs_weight_info", [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                        C.POINTER(C.c_int64), C.POINTER(C.c_int64)])
_sig("rs_debug_buffer", [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)])

# asynchronous seam (caller-owned event loop)
class rs_segment(C.Structure):
    _fields_ = [("kind", C.c_int32), ("tokens", C.c_uint64)]


class rs_event(C.Structure):
    _fields_ = [("kind", C.c_int32), ("stage", C.c_int32), ("tag", C.c_uint64), ("time_ms", C.c_double)]


EV_ENCODE_DONE, EV_TRANSFER_DONE, EV_STAGE_DONE, EV_CHUNK_COMPLETE = 1, 2, 3, 4
_sig("rs_request_create_segments", [C.c_void_p, C.c_uint64, C.POINTER(rs_segment), C.c_int32, C.c_void_p])
_sig("rs_encode_batch_async", [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.c_int32, C.c_void_p,
                               C.c_int32, C.c_void_p, C.c_uint64])
_sig("rs_embeddings_ready", [C.c_void_p, C.c_uint64])
_sig("rs_prefill_chunk_async", [C.c_void_p, C.POINTER(C.c_uint64), C.c_int32, C.c_void_p, C.c_uint64])
_sig("rs_release_async", [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64])
_sig("rs_request_erase_async", [C.c_void_p, C.c_uint64, C.c_uint64])
_sig("rs_poll", [C.c_void_p, C.POINTER(rs_event), C.c_int32, C.c_int32, C.POINTER(C.c_int32)])


# EP disaggregation
class rs_ep_options(C.Structure):
    _fields_ = [("stages", C.c_int32), ("encoders", C.c_int32), ("transport", C.c_int32),
                ("rank", C.c_int32), ("device", C.c_int32), ("nccl_ids", C.c_void_p),
                ("slot_bytes", C.c_uint64), ("shm_name", C.c_char_p)]


_sig("rs_ep_links", [C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)])
_sig("rs_nccl_unique_id", [C.c_void_p])
_sig("rs_ep_create", [C.POINTER(rs_ep_options), C.POINTER(C.c_void_p)])
_sig("rs_ep_destroy", [C.c_void_p])
_sig("rs_ep_ipc_export", [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)])
_sig("rs_ep_ipc_connect", [C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_int32])
_sig("rs_ep_worker_prepare", [C.c_void_p, C.c_void_p, C.c_char_p, C.c_uint64, C.c_int32])
_sig("rs_ep_worker_run", [C.c_void_p, C.c_void_p])
_sig("rs_ep_engine_run", [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p), C.c_char_p,
                          C.POINTER(rs_sim_config), C.POINTER(rs_run_options), PCHAR, PCHAR,
                          C.POINTER(rs_run_stats)])
_sig("rs_engine_cell", [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(rs_workload_config),
                        C.POINTER(rs_sim_config), C.c_double, C.POINTER(rs_run_options), PCHAR, PCHAR,
                        C.POINTER(rs_run_stats)])
_sig("rs_ep_ctrl_pack", [C.c_char_p, C.c_void_p, C.c_uint64])
_sig("rs_ep_ctrl_unpack", [C.c_void_p, C.c_uint64, PCHAR])
EP_CTRL_BYTES = 4096 * 8

# op-level ABI (include/rserve_ops.h)
VP, I = C.c_void_p, C.c_int
_sig("rs_op_gemm", [VP, I, VP, I, VP, I, VP, VP, I, VP, I, I, I, I, I, VP])
_sig("rs_op_rmsnorm", [VP, I, VP, VP, I, I, I, C.c_float, VP])
_sig("rs_op_attention_varlen", [VP, I, VP, I, VP, I, I, I, I, I, C.c_float, VP])
_sig("rs_op_attention_varlen_tc", [VP, I, VP, I, VP, I, I, I, I, C.c_float, VP])
_sig("rs_op_attention_window_tc", [VP, I, VP, I, VP, I, I, I, I, C.c_float, VP, C.c_float, VP])
_sig("rs_op_attention_prefill", [VP, I, I, VP, I, I, I, VP, VP, C.c_longlong, VP, I, I, I,
                                  C.c_float, VP])
_sig("rs_op_attention_decode", [VP, I, VP, I, I, C.POINTER(C.c_int), C.POINTER(C.c_void_p), VP, VP, I, I, I,
                                 C.c_float, VP])
_sig("rs_kernel_launches", [], C.c_ulonglong)
_sig("rs_profile_enable", [C.c_int])
_sig("rs_payload_generate", [C.c_char_p, C.c_uint64, PCHAR])
_sig("rs_payload_validate", [C.c_char_p, C.c_char_p, C.c_int32, PCHAR])
_sig("rs_decode", [C.c_void_p, C.POINTER(C.c_uint64), C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                  C.POINTER(C.c_float), C.POINTER(C.c_double)])
_sig("rs_decode_release", [C.c_void_p, C.c_uint64])


class rs_kv_meta(C.Structure):
    _fields_ = [("tokens", C.c_uint64), ("image_bytes", C.c_uint64), ("next_rope", C.c_int32),
                ("layer_begin", C.c_int32), ("layer_end", C.c_int32), ("kv_heads", C.c_int32),
                ("head_dim", C.c_int32), ("page_tokens", C.c_int32), ("tp_size", C.c_int32)]


_sig("rs_tp_buffer", [C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p])
_sig("rs_tp_connect", [C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p])
_sig("rs_kv_request_create", [C.c_void_p, C.c_uint64, C.c_char_p])
_sig("rs_tp_prefill", [C.c_void_p, C.POINTER(C.c_uint64), C.c_int32, C.c_void_p, C.c_void_p])
_sig("rs_tp_logits", [C.c_void_p, C.c_uint64, C.POINTER(C.c_float), C.POINTER(C.c_int32)])
_sig("rs_kv_image_bytes", [C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64)])
_sig("rs_kv_export", [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.POINTER(rs_kv_meta), C.c_void_p])
_sig("rs_kv_import", [C.c_void_p, C.c_uint64, C.POINTER(rs_kv_meta), C.c_void_p, C.c_void_p])
_sig("rs_profile_drain", [PCHAR])


def profile_drain():
    """{class: dict(launches, ms, flops, bytes)} accumulated since enable."""
    out = C.c_char_p()
    check(lib.rs_profile_drain(C.byref(out)))
    res = {}
    for line in take_string(out).splitlines():
        k, n, ms, fl, by = line.split()
        res[k] = dict(launches=int(n), ms=float(ms), flops=float(fl), bytes=float(by))
    return res


def version() -> str:
    return lib.rs_version().decode()


def exported_symbols():
    """Names of the C-ABI functions declared in include/*.h and found in the .so."""
    return [n for n in dir(lib) if n.startswith("rs_")]
