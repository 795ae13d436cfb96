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
