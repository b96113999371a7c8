"""ctypes binding of the CUDA library (lib/librelserve_b200.so, include/relserve.h).

Loading fails loudly when the library is missing or no CUDA device is visible:
the scheduler has no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from . import _abi

HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ["RS_LIB"]) if os.environ.get("RS_LIB") else HERE / "lib" / "librelserve_b200.so"

_lib = None


class NativeLibraryMissing(ImportError):
    pass


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryMissing(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the scheduler hot path)")
    L = C.CDLL(str(LIB_PATH))
    L.rs_last_error.restype = C.c_char_p
    L.rs_build_info.restype = C.c_char_p
    L.rs_engine_create.restype = C.c_int
    L.rs_engine_create.argtypes = [C.POINTER(_abi.TraceView), C.c_int32, C.POINTER(_abi.Config),
                                   C.POINTER(_abi.CostModel), C.POINTER(_abi.CostModel),
                                   C.POINTER(_abi.Pcg64State), C.c_int32, C.c_int64, C.POINTER(C.c_void_p)]
    L.rs_engine_step.restype = C.c_int
    L.rs_engine_step.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
    L.rs_engine_status.restype = C.c_int
    L.rs_engine_status.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(_abi.TraceStatus)]
    L.rs_engine_read_log.restype = C.c_int
    L.rs_engine_read_log.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_void_p]
    L.rs_engine_read_ledgers.restype = C.c_int
    L.rs_engine_read_ledgers.argtypes = [C.c_void_p, C.c_int32] + [C.c_void_p] * 4
    L.rs_engine_read_requests.restype = C.c_int
    L.rs_engine_read_requests.argtypes = [C.c_void_p, C.c_int32] + [C.c_void_p] * 4
    L.rs_waiting_argmin.restype = C.c_int
    L.rs_waiting_argmin.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
    L.rs_engine_read_running.restype = C.c_int
    L.rs_engine_read_running.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]
    L.rs_engine_read_completion.restype = C.c_int
    L.rs_engine_read_completion.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
    L.rs_engine_destroy.restype = None
    L.rs_engine_destroy.argtypes = [C.c_void_p]
    L.rs_engine_device_bytes.restype = C.c_int64
    L.rs_engine_device_bytes.argtypes = [C.c_void_p]
    L.rs_pem_batch.restype = C.c_int
    L.rs_pem_batch.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                               C.c_int64, C.c_int64, C.POINTER(_abi.CostModel), C.c_void_p, C.c_int32]
    L.rs_device_clock_khz.restype = C.c_int
    L.rs_device_clock_khz.argtypes = [C.c_int32]
    L.rs_choice_sequence.restype = C.c_int
    L.rs_choice_sequence.argtypes = [C.POINTER(_abi.Pcg64State), C.c_int64, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_int32]
    L.rs_engine_create_sharded.restype = C.c_int
    L.rs_engine_create_sharded.argtypes = [C.POINTER(_abi.TraceView), C.POINTER(_abi.Config),
                                           C.POINTER(_abi.CostModel), C.POINTER(_abi.CostModel),
                                           C.POINTER(_abi.Pcg64State), C.c_int32, C.c_int64, C.c_int32,
                                           C.c_int32, C.POINTER(C.c_void_p)]
    L.rs_engine_mailbox.restype = C.c_int
    L.rs_engine_mailbox.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]
    L.rs_engine_connect.restype = C.c_int
    L.rs_engine_connect.argtypes = [C.c_void_p, C.c_void_p]
    L.rs_ipc_get_handle.restype = C.c_int
    L.rs_ipc_get_handle.argtypes = [C.c_void_p, C.c_void_p]
    L.rs_ipc_open_handle.restype = C.c_int
    L.rs_ipc_open_handle.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p)]
    L.rs_trace_v1_load.restype = C.c_int
    L.rs_trace_v1_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
    L.rs_trace_v1_info.restype = C.c_int
    L.rs_trace_v1_info.argtypes = [C.c_void_p] + [C.c_void_p] * 4
    L.rs_trace_v1_columns.restype = C.c_int
    L.rs_trace_v1_columns.argtypes = [C.c_void_p] + [C.c_void_p] * 7
    L.rs_trace_v1_free.restype = None
    L.rs_trace_v1_free.argtypes = [C.c_void_p]
    L.rs_trace_v1_error.restype = C.c_char_p
    L.rs_engine_read_order.restype = C.c_int
    L.rs_engine_read_order.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_void_p]
    L.rs_arrange.restype = C.c_int
    L.rs_arrange.argtypes = [C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int64, C.c_int64,
                             C.c_int64, C.c_double, C.c_double, C.c_int64, C.c_int32, C.POINTER(_abi.CostModel),
                             C.c_int32, C.c_void_p]
    L.rs_engine_set_noise.restype = C.c_int
    L.rs_engine_set_noise.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int64]
    L.rs_ipc_close.restype = C.c_int
    L.rs_ipc_close.argtypes = [C.c_void_p]
    L.rs_engine_read_dpu.restype = C.c_int
    L.rs_engine_read_dpu.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                     C.c_void_p]
    L.rs_engine_read_results.restype = C.c_int
    L.rs_engine_read_results.argtypes = [C.c_void_p, C.c_void_p] + [C.c_void_p] * 4
    L.rs_sort_pairs.restype = C.c_int
    L.rs_sort_pairs.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int32]
    _lib = L
    return L


#: every symbol include/relserve.h declares
EXPORTED_SYMBOLS = (
    "rs_last_error", "rs_build_info", "rs_engine_create", "rs_engine_step", "rs_engine_status",
    "rs_engine_read_log", "rs_engine_read_ledgers", "rs_engine_read_requests", "rs_engine_read_completion",
    "rs_engine_read_running",
    "rs_engine_destroy", "rs_engine_device_bytes", "rs_pem_batch", "rs_choice_sequence", "rs_device_clock_khz",
    "rs_engine_create_sharded", "rs_engine_mailbox", "rs_engine_connect", "rs_ipc_get_handle",
    "rs_ipc_open_handle", "rs_ipc_close", "rs_engine_set_noise", "rs_arrange", "rs_waiting_argmin",
    "rs_engine_read_order", "rs_engine_read_dpu", "rs_sort_pairs", "rs_engine_read_results", "rs_trace_v1_load", "rs_trace_v1_info", "rs_trace_v1_columns", "rs_trace_v1_free",
    "rs_trace_v1_error",
)


_clock_khz: dict[int, int] = {}


def device_clock_khz(device: int = 0) -> int:
    if device not in _clock_khz:  # the attribute query costs milliseconds
        _clock_khz[device] = int(lib().rs_device_clock_khz(device))
    return _clock_khz[device]


def _check(rc: int):
    if rc != _abi.RS_OK:
        from .engine import raise_for

        msg = lib().rs_last_error().decode()
        raise_for(rc, msg)
        raise RuntimeError(f"rc={rc}: {msg}")


def _stream_ptr(stream) -> int | None:
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):  # torch.cuda.Stream
        return int(stream.cuda_stream)
    return int(stream)


class NativeEngine:
    """Owns an rs_engine handle (device SoA for one or more traces)."""

    def __init__(self, views, cfg: _abi.Config, world: _abi.CostModel, pol: _abi.CostModel, rngs,
                 device: int, log_capacity: int, shards: int = 1, rank: int = -1):
        """shards > 1: `views` is one trace, sharded (rank -1: every shard here, one CTA each;
        rank >= 0: this process's shard, see connect())."""
        L = lib()
        h = C.c_void_p()
        self._cfg, self._world, self._pol = cfg, world, pol
        if shards > 1:
            assert len(views) == 1 and len(rngs) == 1
            _check(L.rs_engine_create_sharded(C.byref(views[0]), C.byref(cfg), C.byref(world), C.byref(pol),
                                              C.byref(rngs[0]), device, log_capacity, shards, rank,
                                              C.byref(h)))
            n = shards if rank < 0 else 1
        else:
            n = len(views)
            arr_v = (_abi.TraceView * n)(*views)
            arr_r = (_abi.Pcg64State * n)(*rngs)
            _check(L.rs_engine_create(arr_v, n, C.byref(cfg), C.byref(world), C.byref(pol), arr_r, device,
                                      log_capacity, C.byref(h)))
        self.h = h
        self.n = n
        self.shards, self.rank = shards, rank
        self.device = device
        self.log_capacity = log_capacity
        self._opened: list[int] = []

    # -- sharded pool, one shard per process (include/relserve.h) ----------
    def mailbox_handle(self) -> bytes:
        """CUDA IPC handle (64 bytes) of this shard's mailbox."""
        p, nb = C.c_void_p(), C.c_int64()
        _check(lib().rs_engine_mailbox(self.h, C.byref(p), C.byref(nb)))
        buf = (C.c_uint8 * 64)()
        _check(lib().rs_ipc_get_handle(p, buf))
        return bytes(buf)

    def connect(self, handles: list[bytes]):
        """Map every peer's mailbox (handles[rank] is this shard's own) and connect."""
        ptrs = (C.c_void_p * self.shards)()
        for d, hd in enumerate(handles):
            if d == self.rank:
                continue
            p = C.c_void_p()
            buf = (C.c_uint8 * 64).from_buffer_copy(hd)
            _check(lib().rs_ipc_open_handle(buf, self.device, C.byref(p)))
            self._opened.append(p.value)
            ptrs[d] = p
        _check(lib().rs_engine_connect(self.h, ptrs))

    def set_noise(self, t: int, z: np.ndarray):
        """World-model noise draws for trace t (-1: all), include/relserve.h rs_engine_set_noise."""
        z = np.ascontiguousarray(z, np.float64)
        _check(lib().rs_engine_set_noise(self.h, t, z.ctypes.data if len(z) else None, len(z)))

    def step(self, max_iters: int, stream=None):
        _check(lib().rs_engine_step(self.h, int(max_iters), _stream_ptr(stream)))

    def status(self, stream=None) -> list[_abi.TraceStatus]:
        st = (_abi.TraceStatus * self.n)()
        _check(lib().rs_engine_status(self.h, _stream_ptr(stream), st))
        return list(st)

    def read_log(self, t: int, first: int, count: int) -> np.ndarray:
        out = np.zeros(count, _abi.ITER_RECORD_DTYPE)
        if count:
            _check(lib().rs_engine_read_log(self.h, t, first, count, out.ctypes.data))
        return out

    def read_order(self, t: int, first: int, count: int, R: int) -> np.ndarray:
        """Parity mode: the waiting queue of logged iterations [first, first+count), trace-order
        relQuery indices, one row of R per iteration (-1 past the queue's length)."""
        out = np.full((count, max(R, 1)), -1, np.int32)
        if count:
            _check(lib().rs_engine_read_order(self.h, t, first, count, out.ctypes.data))
        return out[:, :R]

    def read_dpu(self, t: int, first: int, count: int, R: int):
        """Parity mode: the priority update of logged iterations [first, first+count): per
        iteration and relQuery (trace order) the value and RS_SNAP_* flags, and the DPU
        generator state after the update (include/relserve.h rs_engine_read_dpu)."""
        vals = np.full((count, max(R, 1)), np.nan, np.float64)
        flags = np.zeros((count, max(R, 1)), np.uint8)
        rng = (_abi.Pcg64State * max(count, 1))()
        if count:
            _check(lib().rs_engine_read_dpu(self.h, t, first, count, vals.ctypes.data, flags.ctypes.data, rng))
        return vals[:, :R], flags[:, :R], [rng[i] for i in range(count)]

    def read_results(self, R_total: int, N_total: int, stream=None):
        """Every trace's ledgers (first_prefill_start, last_prefill_end, last_decode_end) and
        completion iterations, traces concatenated (include/relserve.h rs_engine_read_results)."""
        b, c, d = (np.zeros(R_total, np.float64) for _ in range(3))
        comp = np.zeros(N_total, np.int32)
        _check(lib().rs_engine_read_results(self.h, _stream_ptr(stream), b.ctypes.data, c.ctypes.data,
                                            d.ctypes.data, comp.ctypes.data))
        return b, c, d, comp

    def read_ledgers(self, t: int, R: int):
        a, b, c, d = (np.zeros(R, np.float64) for _ in range(4))
        _check(lib().rs_engine_read_ledgers(self.h, t, a.ctypes.data, b.ctypes.data, c.ctypes.data,
                                            d.ctypes.data))
        return a, b, c, d

    def read_requests(self, t: int, N: int):
        gen = np.zeros(N, np.int32)
        pre = np.zeros(N, np.uint8)
        comp = np.zeros(N, np.int64)
        prio = np.zeros(N, np.float64)
        _check(lib().rs_engine_read_requests(self.h, t, gen.ctypes.data, pre.ctypes.data,
                                             comp.ctypes.data, prio.ctypes.data))
        return gen, pre, comp, prio

    def read_running(self, t: int) -> np.ndarray:
        """Trace-order rows of the running requests, in execution order."""
        n = C.c_int32(0)
        rows = np.zeros(1024, np.int32)
        _check(lib().rs_engine_read_running(self.h, t, rows.ctypes.data, len(rows), C.byref(n)))
        if n.value > len(rows):
            rows = np.zeros(n.value, np.int32)
            _check(lib().rs_engine_read_running(self.h, t, rows.ctypes.data, len(rows), C.byref(n)))
        return rows[: n.value].copy()

    def read_completion(self, t: int, N: int) -> np.ndarray:
        """int32 completion iterations, trace order, in page-locked memory from torch's caching
        host allocator (one DMA; the block returns to the cache when the array is dropped)."""
        import torch

        comp = torch.empty(N, dtype=torch.int32, pin_memory=True).numpy()
        _check(lib().rs_engine_read_completion(self.h, t, comp.ctypes.data))
        return comp

    def device_bytes(self) -> int:
        return int(lib().rs_engine_device_bytes(self.h))

    def close(self):
        if self.h:
            lib().rs_engine_destroy(self.h)
            self.h = None
        for p in self._opened:
            lib().rs_ipc_close(C.c_void_p(p))
        self._opened = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pem_batch(item_off, utok, rem, pre, constraints, model, device=0) -> np.ndarray:
    n_sets = len(item_off) - 1
    out = np.zeros(max(n_sets, 0), np.float64)
    if n_sets <= 0:
        return out
    cm = _abi.CostModel(model.alpha_p, model.beta_p, model.alpha_d, model.beta_d)
    keep = [np.ascontiguousarray(x) for x in (item_off, utok, rem, pre)]
    _check(lib().rs_pem_batch(n_sets, *(k.ctypes.data for k in keep), constraints.cap,
                              constraints.max_num_seqs, constraints.max_num_batched_tokens, C.byref(cm),
                              out.ctypes.data, device))
    return out


def choice_sequence(state: _abi.Pcg64State, ns, ks, device=0) -> np.ndarray:
    ns = np.ascontiguousarray(ns, np.int64)
    ks = np.ascontiguousarray(ks, np.int64)
    out = np.zeros(max(int(ks.sum()), 1), np.int64)
    _check(lib().rs_choice_sequence(C.byref(state), len(ns), ns.ctypes.data, ks.ctypes.data,
                                    out.ctypes.data, device))
    return out[: int(ks.sum())]


def arrange(running, d_min_rel_id, prefill_n, prefill_utok, prefill_rel_id, prefill_output_limit, m_plus, m_minus,
            n_waiting, policy, model, device=0) -> np.ndarray:
    """The device arranger (include/relserve.h rs_arrange).  running: [(rel_id, output_limit)] of the
    decode candidate's distinct relQueries.  Returns one rs_iter_record (NaN = None)."""
    rel = np.ascontiguousarray([r for r, _ in running], np.int64)
    ol = np.ascontiguousarray([o for _, o in running], np.int64)
    out = np.zeros(1, _abi.ITER_RECORD_DTYPE)
    cm = _abi.CostModel(model.alpha_p, model.beta_p, model.alpha_d, model.beta_d)
    nan = float("nan")
    _check(lib().rs_arrange(len(rel), rel.ctypes.data if len(rel) else None, ol.ctypes.data if len(ol) else None,
                            int(d_min_rel_id), int(prefill_n), int(prefill_utok), int(prefill_rel_id),
                            int(prefill_output_limit), nan if m_plus is None else float(m_plus),
                            nan if m_minus is None else float(m_minus), int(n_waiting), _abi.POLICY_IDS[policy],
                            C.byref(cm), device, out.ctypes.data))
    return out[0]


def waiting_argmin(priority, waiting, device=0):
    """The device waiting-queue head (include/relserve.h rs_waiting_argmin): entries in admission
    order; returns (head index or -1, number waiting)."""
    p = np.ascontiguousarray(priority, np.float64)
    w = np.ascontiguousarray(waiting, np.uint8)
    if p.shape != w.shape:
        raise ValueError("priority and waiting differ in length")
    head, count = C.c_int64(), C.c_int64()
    _check(lib().rs_waiting_argmin(p.ctypes.data if len(p) else None, w.ctypes.data if len(w) else None, len(p),
                                   device, C.byref(head), C.byref(count)))
    return head.value, count.value


def sort_pairs(keys, values, device=0):
    """Stable device radix sort of (uint64 key, int32 value) pairs by key (include/relserve.h
    rs_sort_pairs, north-star kernel 2)."""
    k = np.ascontiguousarray(keys, np.uint64)
    v = np.ascontiguousarray(values, np.int32)
    if k.shape != v.shape:
        raise ValueError("keys and values differ in length")
    ko, vo = np.empty_like(k), np.empty_like(v)
    _check(lib().rs_sort_pairs(k.ctypes.data if len(k) else None, v.ctypes.data if len(v) else None, len(k),
                               ko.ctypes.data if len(k) else None, vo.ctypes.data if len(v) else None, device))
    return ko, vo


def priority_keys(prio) -> np.ndarray:
    """okey() of include/relserve.h's waiting order: uint64 keys whose unsigned order is the
    numeric order of the priorities (any sign)."""
    b = np.ascontiguousarray(prio, np.float64).view(np.uint64)
    neg = (b >> np.uint64(63)).astype(bool)
    return np.where(neg, ~b, b | np.uint64(1 << 63))


def read_trace_v1(path):
    """relsim-trace-v1 counts via the native reader: (rel_id, arrival, output_limit, prefix_len,
    row_off, tok, out, rate, seed); ValueError on a malformed file."""
    L = lib()
    h = C.c_void_p()
    if L.rs_trace_v1_load(str(path).encode(), C.byref(h)) != _abi.RS_OK:
        raise ValueError(L.rs_trace_v1_error().decode())
    try:
        R, N, seed = C.c_int64(), C.c_int64(), C.c_int64()
        rate = C.c_double()
        L.rs_trace_v1_info(h, C.byref(R), C.byref(N), C.byref(rate), C.byref(seed))
        R, N = R.value, N.value
        cols = (np.zeros(R, np.int64), np.zeros(R, np.float64), np.zeros(R, np.int32), np.zeros(R, np.int32),
                np.zeros(R + 1, np.int64), np.zeros(N, np.int32), np.zeros(N, np.int32))
        L.rs_trace_v1_columns(h, *(c.ctypes.data for c in cols))
    finally:
        L.rs_trace_v1_free(h)
    return (*cols, rate.value, seed.value)
