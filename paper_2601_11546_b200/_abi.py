"""ctypes mirror of include/relserve.h (structs, enums, status codes)."""

from __future__ import annotations

import ctypes as C

import numpy as np

RS_OK = 0
RS_EINVAL = 1
RS_EINFEASIBLE = 2
RS_EABORT_LIMIT = 3
RS_EABORT_IDLE = 4
RS_ECACHE_PINNED = 5
RS_ECUDA = 6
RS_ENOMEM = 7
RS_EUNSUPPORTED = 8
RS_RUNNING = 100

# parity-mode snapshot flags (include/relserve.h RS_SNAP_*)
SNAP_ESTIMATED, SNAP_OVERRIDE, SNAP_LIVE, SNAP_WAITING = 1, 2, 4, 8

POLICY_IDS = {"fcfs": 0, "sp": 1, "relserve": 2, "relserve-pp": 3, "relserve-dp": 4}
ACTIONS = ("prefill", "decode", "idle")
CASES = ("preempt", "internal", "transitional", "forced")


class CostModel(C.Structure):
    _fields_ = [("alpha_p", C.c_double), ("beta_p", C.c_double),
                ("alpha_d", C.c_double), ("beta_d", C.c_double)]


class Config(C.Structure):
    _fields_ = [
        ("cap", C.c_int64), ("max_num_seqs", C.c_int64), ("max_num_batched_tokens", C.c_int64),
        ("sample_size", C.c_int64), ("tau", C.c_double), ("noise_sigma", C.c_double),
        ("block_size", C.c_int64), ("capacity_blocks", C.c_int64), ("iteration_limit", C.c_int64),
        ("log_decisions", C.c_int32), ("policy", C.c_int32), ("record_order", C.c_int32), ("reserved", C.c_int32),
    ]


class Pcg64State(C.Structure):
    _fields_ = [("state_hi", C.c_uint64), ("state_lo", C.c_uint64),
                ("inc_hi", C.c_uint64), ("inc_lo", C.c_uint64),
                ("has_uint32", C.c_uint32), ("uinteger", C.c_uint32)]

    @classmethod
    def from_numpy(cls, state: dict) -> "Pcg64State":
        s = int(state["state"]["state"])
        inc = int(state["state"]["inc"])
        m = (1 << 64) - 1
        return cls(s >> 64, s & m, inc >> 64, inc & m, int(state["has_uint32"]), int(state["uinteger"]))

    def to_numpy(self) -> dict:
        return {
            "bit_generator": "PCG64",
            "state": {"state": (self.state_hi << 64) | self.state_lo,
                      "inc": (self.inc_hi << 64) | self.inc_lo},
            "has_uint32": int(self.has_uint32),
            "uinteger": int(self.uinteger),
        }


class TraceView(C.Structure):
    _fields_ = [
        ("num_relqueries", C.c_int64), ("num_requests", C.c_int64),
        ("rel_id", C.c_void_p), ("arrival", C.c_void_p), ("output_limit", C.c_void_p),
        ("row_off", C.c_void_p), ("tok", C.c_void_p), ("out", C.c_void_p),
        ("chain_blocks", C.c_void_p), ("static_prio", C.c_void_p),
    ]


ITER_RECORD_DTYPE = np.dtype([
    ("iteration", np.int64), ("clock", np.float64), ("m_plus", np.float64), ("m_minus", np.float64),
    ("delta_plus", np.float64), ("delta_minus", np.float64), ("delta_total", np.float64),
    ("kv_reserved", np.int64), ("action", np.int32), ("kase", np.int32), ("head", np.int32),
    ("n_waiting", np.int32), ("batch_rq", np.int32), ("batch_first", np.int32),
    ("batch_n", np.int32), ("n_reestimated", np.int32),
])
assert ITER_RECORD_DTYPE.itemsize == 96


class IterRecord(C.Structure):
    _fields_ = [(n, {np.dtype(np.int64): C.c_int64, np.dtype(np.float64): C.c_double,
                     np.dtype(np.int32): C.c_int32}[ITER_RECORD_DTYPE.fields[n][0]])
                for n in ITER_RECORD_DTYPE.names]


class TraceStatus(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64), ("clock", C.c_double), ("cache_hit_tokens", C.c_int64),
        ("cache_miss_tokens", C.c_int64), ("kv_reserved", C.c_int64), ("n_log", C.c_int64),
        ("live_relqueries", C.c_int64), ("admitted", C.c_int64), ("status", C.c_int32),
        ("error_detail", C.c_int32), ("rng", Pcg64State), ("phase_cycles", C.c_int64 * 23), ("alg_bytes", C.c_int64),
        ("batches", C.c_int64),
    ]


def ptr(a: np.ndarray | None) -> int | None:
    """Raw data pointer of a contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data
