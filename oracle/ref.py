"""ORACLE — test infrastructure only. ctypes wrapper of oracle/_ref/liblmmsim_ref.so,
the C-ABI over the UNMODIFIED reference headers (oracle/ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's reference / cpu_baseline
legs use this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "liblmmsim_ref.so")
REFERENCE = "/root/reference/proj"


def build(quiet: bool = True) -> bool:
    """Builds oracle/_ref from /root/reference when present. False if absent."""
    if not os.path.isdir(REFERENCE):
        return os.path.exists(LIB)
    out = subprocess.run(["make", "-C", HERE, "-j8", "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    return True


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise FileNotFoundError(f"{LIB} missing (run oracle.ref.build() where /root/reference exists)")
        _lib = C.CDLL(LIB)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_free.argtypes = [C.c_void_p]
    return _lib


def _take(p):
    s = C.cast(p, C.c_char_p).value.decode() if p else ""
    lib().ref_free(p)
    return s


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {lib().ref_last_error().decode()}")


def simulate(workload: str, sim_c) -> str:
    out = C.c_char_p()
    _check(lib().ref_simulate(workload.encode(), C.byref(sim_c), C.byref(out)))
    return _take(out)


def generate_workload(w_c) -> str:
    out = C.c_char_p()
    _check(lib().ref_generate_workload(C.byref(w_c), C.byref(out)))
    return _take(out)


def experiment_cell(w_c, sim_c, slo) -> str:
    out = C.c_char_p()
    _check(lib().ref_experiment_cell(C.byref(w_c), C.byref(sim_c),
                                     C.c_double(-1.0 if slo is None else float(slo)), C.byref(out)))
    return _take(out)


def plan_batches(layout: str, rid: int, c: int) -> str:
    out = C.c_char_p()
    _check(lib().ref_plan_batches(layout.encode(), C.c_uint64(rid), C.c_uint64(c), C.byref(out)))
    return _take(out)


def replay(workload: str, sim_c, journal: str) -> str:
    out = C.c_char_p()
    _check(lib().ref_replay(workload.encode(), C.byref(sim_c), journal.encode(), C.byref(out)))
    return _take(out)


def time_simulate(workload: str, sim_c, reps: int) -> float:
    """Nanoseconds per run_simulation call (single thread, as the reference)."""
    ns = C.c_double()
    _check(lib().ref_time_simulate(workload.encode(), C.byref(sim_c), C.c_int(reps), C.byref(ns)))
    return ns.value


# ---- standalone config structs --------------------------------------------------------------
# Layout mirrors of include/rserve.h rs_sim_config / rs_workload_config (what
# ref_shim.cpp reads), so the CPU reference arm never loads the product
# library (bench.py --impl reference).
POLICIES = {"vanilla_pp": 0, "epd_baseline": 1, "intra_only": 2, "rserve": 3}
PATTERNS = {"alternating": 0, "consecutive_mm": 1, "text_first": 2}


class CostModel(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "alpha_enc_ms", "beta_enc_ms_per_token", "eps_tx_ms", "zeta_tx_ms_per_token",
        "gamma_stage_ms", "delta_stage_ms_per_token", "kappa_attn_ms", "tp_speedup")]


class SimConfigC(C.Structure):
    _fields_ = [("policy", C.c_int32), ("pipeline_mode", C.c_int32), ("stages", C.c_int32),
                ("encoder_workers", C.c_int32), ("token_budget", C.c_uint64),
                ("embedding_batch_tokens", C.c_uint64), ("release_at", C.c_int32),
                ("hidden_size", C.c_uint32), ("cost", CostModel)]


class IntDist(C.Structure):
    _fields_ = [("uniform", C.c_int32), ("lo", C.c_uint64), ("hi", C.c_uint64)]


class Template(C.Structure):
    _fields_ = [("pattern", C.c_int32), ("num_mm_items", IntDist), ("mm_item_tokens", IntDist),
                ("text_segment_tokens", IntDist), ("probability", C.c_double)]


class WorkloadConfigC(C.Structure):
    _fields_ = [("arrival_rate", C.c_double), ("duration_s", C.c_double), ("seed", C.c_uint64),
                ("templates", C.POINTER(Template)), ("n_templates", C.c_int32),
                ("has_slo", C.c_int32), ("slo_ttft_ms", C.c_double)]


def sim_config(policy="rserve", stages=1, token_budget=2048, c_tokens=1024, encoder_workers=1,
               hidden_size=3584, **cost) -> SimConfigC:
    s = SimConfigC()
    s.policy = POLICIES[policy]
    s.pipeline_mode = -1
    s.stages = stages
    s.encoder_workers = encoder_workers
    s.token_budget = token_budget
    s.embedding_batch_tokens = c_tokens
    s.release_at = 1
    s.hidden_size = hidden_size
    s.cost.tp_speedup = 1.0
    for k, v in cost.items():
        setattr(s.cost, k, v)
    return s


def workload_config(seed: int, rate: float, duration_s: float, pattern="alternating",
                    mm_items=(4, 16), mm_tokens=1024, text_tokens=(32, 256)):
    """One-template WorkloadConfig (workload.hpp:109-136); returns (struct, keep-alive)."""
    def dist(v):
        d = IntDist()
        lo, hi = (v, v) if isinstance(v, int) else v
        d.uniform, d.lo, d.hi = int(lo != hi), lo, hi
        return d
    arr = (Template * 1)()
    arr[0].pattern = PATTERNS[pattern]
    arr[0].num_mm_items = dist(mm_items)
    arr[0].mm_item_tokens = dist(mm_tokens)
    arr[0].text_segment_tokens = dist(text_tokens)
    arr[0].probability = 1.0
    w = WorkloadConfigC()
    w.arrival_rate, w.duration_s, w.seed = rate, duration_s, seed
    w.templates = C.cast(arr, C.POINTER(Template))
    w.n_templates = 1
    return w, arr
