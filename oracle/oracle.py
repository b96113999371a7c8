"""ctypes wrapper of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may use
this module, and only as the checker / baseline -- never as the product path.
"""

from __future__ import annotations

import ctypes as C
import math
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from paper_2601_11546_b200 import _abi, _marshal
from paper_2601_11546_b200.engine import EngineConfig, POLICIES

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "lib" / "librelsim_oracle.so"

OR_REC_DPU, OR_REC_WAITING, OR_REC_RNG = 1, 2, 4


class _DpuRec(C.Structure):
    _fields_ = [("rq", C.c_int32), ("reused", C.c_int32), ("overridden", C.c_int32),
                ("pad", C.c_int32), ("value", C.c_double)]


class _Result(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("pad", C.c_int32), ("iterations", C.c_int64), ("clock", C.c_double),
        ("cache_hit_tokens", C.c_int64), ("cache_miss_tokens", C.c_int64), ("kv_reserved", C.c_int64),
        ("dpu_wall_s", C.c_double), ("aba_wall_s", C.c_double), ("total_wall_s", C.c_double),
        ("first_sight_wall_s", C.c_double), ("first_sight_iter", C.c_int64),
        ("n_log", C.c_int64), ("log", C.c_void_p),
        ("num_relqueries", C.c_int64), ("num_requests", C.c_int64),
        ("first_prefill_start", C.POINTER(C.c_double)), ("last_prefill_end", C.POINTER(C.c_double)),
        ("last_decode_end", C.POINTER(C.c_double)),
        ("generated", C.POINTER(C.c_int32)), ("prefilled", C.POINTER(C.c_uint8)),
        ("completion_iter", C.POINTER(C.c_int64)), ("priority", C.POINTER(C.c_double)),
        ("n_dpu", C.c_int64), ("dpu_off", C.POINTER(C.c_int64)), ("dpu", C.POINTER(_DpuRec)),
        ("n_wait", C.c_int64), ("wait_off", C.POINTER(C.c_int64)), ("wait", C.POINTER(C.c_int32)),
        ("rng_trace", C.POINTER(C.c_uint64)), ("rng", _abi.Pcg64State),
        ("iter_wall", C.POINTER(C.c_double)), ("message", C.c_char * 256),
    ]


def build(quiet: bool = True) -> Path:
    subprocess.run(["make", "-C", str(HERE)], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = C.CDLL(str(LIB_PATH))
        L.or_run.restype = C.POINTER(_Result)
        L.or_run.argtypes = [C.POINTER(_abi.TraceView), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                             C.POINTER(_abi.Config), C.POINTER(_abi.CostModel), C.POINTER(_abi.CostModel),
                             C.POINTER(_abi.Pcg64State), C.c_int32]
        L.or_run_noise.restype = C.POINTER(_Result)
        L.or_run_noise.argtypes = L.or_run.argtypes + [C.c_void_p, C.c_int64]
        L.or_free.argtypes = [C.POINTER(_Result)]
        L.or_pem.restype = C.c_int
        L.or_pem.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                             C.c_int64, C.POINTER(_abi.CostModel), C.POINTER(C.c_double)]
        L.or_choice.restype = C.c_int
        L.or_choice.argtypes = [C.POINTER(_abi.Pcg64State), C.c_int64, C.c_int64, C.c_void_p]
        L.or_next64.restype = C.c_uint64
        L.or_next64.argtypes = [C.POINTER(_abi.Pcg64State)]
        L.or_next32.restype = C.c_uint32
        L.or_next32.argtypes = [C.POINTER(_abi.Pcg64State)]
        _lib = L
    return _lib


@dataclass
class OracleResult:
    status: int
    message: str
    iterations: int
    clock: float
    cache_hit_tokens: int
    cache_miss_tokens: int
    kv_reserved: int
    log: np.ndarray              # ITER_RECORD_DTYPE[n_log]
    first_prefill_start: np.ndarray
    last_prefill_end: np.ndarray
    last_decode_end: np.ndarray
    generated: np.ndarray
    prefilled: np.ndarray
    completion_iter: np.ndarray
    priority: np.ndarray
    dpu_off: np.ndarray | None
    dpu: np.ndarray | None
    wait_off: np.ndarray | None
    wait: np.ndarray | None
    rng_trace: np.ndarray | None
    rng: dict
    dpu_wall_s: float
    aba_wall_s: float
    total_wall_s: float
    first_sight_wall_s: float
    first_sight_iter: int
    iter_wall: np.ndarray


def _arr(p, n, dt):
    if not p or n == 0:
        return np.zeros(0, dt)
    return np.ctypeslib.as_array(p, shape=(n,)).copy().astype(dt)


def run(trace, policy: str, world_model, config: EngineConfig | None = None, policy_model=None,
        seed: int = 0, record: int = 0, explicit_trie: bool | None = None) -> OracleResult:
    """Run the CPU restatement of relsim's Engine on a trace (mirror types)."""
    if policy not in POLICIES:
        raise ValueError(policy)
    cfg = config or EngineConfig()
    pm = policy_model if policy_model is not None else world_model
    m = _marshal.marshal_trace(trace, cfg.block_size, policy, pm,
                               cfg.sp_priority_fns, check_forest=False)
    trie = m.trie
    if explicit_trie is False:
        trie = None
    c_cfg = _marshal.make_config(cfg, policy)
    world = _marshal.make_model(world_model)
    pol = _marshal.make_model(pm)
    rng = _marshal.dpu_rng_state(seed)
    L = lib()
    args = (None, None, None, 0)
    if trie is not None:
        args = (_abi.ptr(trie.path_off), _abi.ptr(trie.path_node), _abi.ptr(trie.node_parent),
                int(trie.node_parent.shape[0]))
    noise = np.zeros(0)
    if cfg.noise_sigma > 0:  # the reference's draws (engine.py:198): one per executed batch, at most one per iteration
        n = min(int(cfg.iteration_limit), 1 << 22)
        noise = np.random.default_rng(np.random.SeedSequence([seed, 0xE7])).standard_normal(n)
    rp = L.or_run_noise(C.byref(m.view), *args, C.byref(c_cfg), C.byref(world), C.byref(pol), C.byref(rng),
                        record, noise.ctypes.data if len(noise) else None, len(noise))
    try:
        r = rp.contents
        R, N, nl = r.num_relqueries, r.num_requests, r.n_log
        log = np.zeros(nl, _abi.ITER_RECORD_DTYPE)
        if nl:
            C.memmove(log.ctypes.data, r.log, nl * _abi.ITER_RECORD_DTYPE.itemsize)
        res = OracleResult(
            status=r.status, message=r.message.decode(), iterations=r.iterations, clock=r.clock,
            cache_hit_tokens=r.cache_hit_tokens, cache_miss_tokens=r.cache_miss_tokens,
            kv_reserved=r.kv_reserved, log=log,
            first_prefill_start=_arr(r.first_prefill_start, R, np.float64),
            last_prefill_end=_arr(r.last_prefill_end, R, np.float64),
            last_decode_end=_arr(r.last_decode_end, R, np.float64),
            generated=_arr(r.generated, N, np.int32), prefilled=_arr(r.prefilled, N, np.uint8),
            completion_iter=_arr(r.completion_iter, N, np.int64), priority=_arr(r.priority, N, np.float64),
            dpu_off=_arr(r.dpu_off, nl + 1, np.int64) if record & OR_REC_DPU else None,
            dpu=(np.ctypeslib.as_array(C.cast(r.dpu, C.POINTER(C.c_uint8)), shape=(r.n_dpu * 24,)).copy()
                 .view(np.dtype([("rq", np.int32), ("reused", np.int32), ("overridden", np.int32),
                                 ("pad", np.int32), ("value", np.float64)]))
                 if record & OR_REC_DPU and r.n_dpu else None),
            wait_off=_arr(r.wait_off, nl + 1, np.int64) if record & OR_REC_WAITING else None,
            wait=_arr(r.wait, r.n_wait, np.int32) if record & OR_REC_WAITING else None,
            rng_trace=(_arr(r.rng_trace, 4 * nl, np.uint64).reshape(nl, 4) if record & OR_REC_RNG else None),
            rng=r.rng.to_numpy(), dpu_wall_s=r.dpu_wall_s, aba_wall_s=r.aba_wall_s,
            total_wall_s=r.total_wall_s, first_sight_wall_s=r.first_sight_wall_s,
            first_sight_iter=r.first_sight_iter, iter_wall=_arr(r.iter_wall, nl, np.float64),
        )
    finally:
        L.or_free(rp)
    return res


def pem(utok, remaining, prefilled, constraints, model) -> float:
    u = np.ascontiguousarray(utok, np.int64)
    r = np.ascontiguousarray(remaining, np.int32)
    p = np.ascontiguousarray(prefilled, np.uint8)
    out = C.c_double()
    cm = _marshal.make_model(model)
    rc = lib().or_pem(len(u), _abi.ptr(u), _abi.ptr(r), _abi.ptr(p), constraints.cap,
                      constraints.max_num_seqs, constraints.max_num_batched_tokens, C.byref(cm),
                      C.byref(out))
    if rc == _abi.RS_EINFEASIBLE:
        from paper_2601_11546_b200.priority import InfeasibleRequestError
        raise InfeasibleRequestError("uncached tokens exceed cap")
    assert rc == 0
    return out.value


def choice(state: _abi.Pcg64State, n: int, k: int) -> np.ndarray:
    idx = np.zeros(max(k, 1), np.int64)
    rc = lib().or_choice(C.byref(state), n, k, _abi.ptr(idx))
    if rc:
        raise ValueError(f"or_choice rc={rc}")
    return idx[:k]
