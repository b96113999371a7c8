"""relQuery / request state types and synthetic arrival traces (host side).

Mirrors the reference data model (`pkg/src/relsim/workload.py:105-167`) so that
code written against `relsim.workload` runs unchanged, but stores a trace
column-wise (numpy structure-of-arrays) from the start: the device engine
uploads these columns as-is, and per-request Python objects are only built
when a caller asks for `trace.entries`.

Token IDs are opaque.  Traces built by `generate_trace` / `load_trace` keep
only counts and rebuild token IDs on demand from the same count-keyed PCG64
streams the reference uses (`workload.py:248-262`), so `Request.tokens` is
identical to the reference's when it is read.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from enum import Enum
from pathlib import Path
from typing import Sequence

import numpy as np

VOCAB_SIZE = 2**31


class QueryType(Enum):
    FILTERING = "filtering"
    CLASSIFICATION = "classification"
    RATING = "rating"
    SUMMARIZATION = "summarization"
    OPEN = "open"


#: Output-token limit per query type (`workload.py:33-40`).
OUTPUT_LIMITS = {
    QueryType.FILTERING: 5,
    QueryType.CLASSIFICATION: 10,
    QueryType.RATING: 5,
    QueryType.SUMMARIZATION: 50,
    QueryType.OPEN: 100,
}


class SchemaError(ValueError):
    """A trace record or template is malformed."""


def token_stream(seed: int, rel_id: int, stream: int, n: int) -> list[int]:
    """Count-keyed token IDs: PCG64(SeedSequence([seed, rel_id, stream])).

    Same stream definition as the reference (`workload.py:248-250`).
    """
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, rel_id, stream])))
    return rng.integers(0, VOCAB_SIZE, size=n).tolist()


def materialize_tokens(seed: int, rel_id: int, req_id: int, tok: int, prefix_len: int) -> list[int]:
    """Shared prefix from stream 0 + unique suffix from stream req_id+1 (`workload.py:253-262`)."""
    return token_stream(seed, rel_id, 0, prefix_len) + token_stream(
        seed, rel_id, req_id + 1, tok - prefix_len
    )


class Request:
    """One prompt of a relQuery (`workload.py:105-136`).

    ``tokens`` may be given explicitly (as in the reference) or left to be
    rebuilt from the count-keyed streams (``token_seed``/``prefix_len``).
    ``generated``, ``priority`` and ``prefilled`` are engine-mutated state.
    """

    __slots__ = (
        "rel_id", "req_id", "_tokens", "_tok", "_token_seed", "_prefix_len",
        "output_limit", "actual_output_len", "arrival", "generated", "priority",
        "prefilled",
    )

    def __init__(
        self,
        rel_id: int,
        req_id: int,
        tokens: Sequence[int] | None,
        output_limit: int,
        actual_output_len: int,
        arrival: float = 0.0,
        generated: int = 0,
        priority: float = 0.0,
        prefilled: bool = False,
        *,
        tok: int | None = None,
        token_seed: int | None = None,
        prefix_len: int = 0,
    ):
        if tokens is not None:
            tokens = list(tokens)
            if not tokens:
                raise ValueError("request tokens must be non-empty")
            tok = len(tokens)
        elif tok is None or token_seed is None or tok <= 0:
            raise ValueError("request needs tokens or (tok, token_seed)")
        if not (1 <= actual_output_len <= output_limit):
            raise ValueError("actual_output_len out of range")
        self.rel_id = rel_id
        self.req_id = req_id
        self._tokens = tokens
        self._tok = int(tok)
        self._token_seed = token_seed
        self._prefix_len = int(prefix_len)
        self.output_limit = output_limit
        self.actual_output_len = actual_output_len
        self.arrival = arrival
        self.generated = generated
        self.priority = priority
        self.prefilled = prefilled

    @property
    def tokens(self) -> list[int]:
        if self._tokens is None:
            self._tokens = materialize_tokens(
                self._token_seed, self.rel_id, self.req_id, self._tok, self._prefix_len
            )
        return self._tokens

    @property
    def has_explicit_tokens(self) -> bool:
        return self._token_seed is None

    @property
    def tok(self) -> int:
        return self._tok

    @property
    def done(self) -> bool:
        return self.generated >= self.actual_output_len

    def __repr__(self) -> str:
        return (f"Request(rel_id={self.rel_id}, req_id={self.req_id}, tok={self.tok}, "
                f"output_limit={self.output_limit}, actual_output_len={self.actual_output_len})")


class RelQuery:
    """A templated batch of requests, one per table row (`workload.py:139-151`)."""

    __slots__ = ("rel_id", "requests", "output_limit", "arrival", "prefix_len")

    def __init__(self, rel_id: int, requests: list[Request], output_limit: int,
                 arrival: float, prefix_len: int = 0):
        self.rel_id = rel_id
        self.requests = requests
        self.output_limit = output_limit
        self.arrival = arrival
        self.prefix_len = prefix_len

    @property
    def size(self) -> int:
        return len(self.requests)


@dataclass
class TraceColumns:
    """Column-wise trace: the host-side image of the device SoA.

    relQueries are in trace order (sorted by arrival); rows of relQuery i are
    ``row_off[i]:row_off[i+1]`` in req_id order.
    """

    rel_id: np.ndarray        # int64[R]
    arrival: np.ndarray       # float64[R]
    output_limit: np.ndarray  # int32[R]
    prefix_len: np.ndarray    # int32[R]
    row_off: np.ndarray       # int64[R+1]
    tok: np.ndarray           # int32[N]
    out: np.ndarray           # int32[N]  (actual_output_len: simulated EOS point)
    token_seed: int | None    # count-keyed token streams, or None (explicit tokens)

    @property
    def num_relqueries(self) -> int:
        return int(self.rel_id.shape[0])

    @property
    def num_requests(self) -> int:
        return int(self.tok.shape[0])

    @property
    def size(self) -> np.ndarray:
        return np.diff(self.row_off).astype(np.int64)


class ArrivalTrace:
    """Timed relQuery trace (`workload.py:154-167`), column-backed.

    Constructed either from RelQuery entries (reference signature) or from
    `TraceColumns` (what `generate_trace`/`load_trace` produce).  ``entries``
    is materialised lazily from the columns on first access.
    """

    def __init__(self, entries: list[RelQuery] | None = None, rate: float = 1.0,
                 seed: int = 0, *, columns: TraceColumns | None = None):
        if entries is None and columns is None:
            raise ValueError("ArrivalTrace needs entries or columns")
        self.rate = rate
        self.seed = seed
        self._entries = list(entries) if entries is not None else None
        self._columns = columns
        if self._entries is not None:
            times = [q.arrival for q in self._entries]
            if times != sorted(times):
                raise ValueError("trace entries must be sorted by arrival")
        else:
            arr = columns.arrival
            if arr.shape[0] > 1 and np.any(arr[1:] < arr[:-1]):
                raise ValueError("trace entries must be sorted by arrival")

    @property
    def entries(self) -> list[RelQuery]:
        if self._entries is None:
            self._entries = _entries_from_columns(self._columns)
        return self._entries

    @property
    def materialized(self) -> bool:
        return self._entries is not None

    def columns(self) -> TraceColumns:
        """Column view of the trace (built from entries when needed)."""
        if self._columns is None or self._entries is not None and self._columns_stale():
            self._columns = _columns_from_entries(self._entries)
        return self._columns

    def pin_memory(self) -> "ArrivalTrace":
        """Move the column arrays into page-locked host memory (torch's pinned host
        allocator), so engine creation uploads them by DMA instead of through the
        driver's pageable staging.  Returns self; values are unchanged."""
        import dataclasses

        import torch

        c = self.columns()

        def pin(a):
            return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

        self._columns = dataclasses.replace(
            c, **{f: pin(getattr(c, f)) for f in ("rel_id", "arrival", "output_limit", "prefix_len", "row_off",
                                                   "tok", "out")})
        return self

    def _columns_stale(self) -> bool:
        c = self._columns
        if c.num_relqueries != len(self._entries):
            return True
        return False

    @property
    def num_requests(self) -> int:
        if self._entries is not None:
            return sum(q.size for q in self._entries)
        return self._columns.num_requests


def _entries_from_columns(c: TraceColumns) -> list[RelQuery]:
    if c.token_seed is None:
        raise SchemaError("explicit-token traces must carry their entries")
    entries = []
    tok = c.tok.tolist()
    out = c.out.tolist()
    off = c.row_off.tolist()
    for i in range(c.num_relqueries):
        rel_id = int(c.rel_id[i])
        arrival = float(c.arrival[i])
        limit = int(c.output_limit[i])
        plen = int(c.prefix_len[i])
        reqs = [
            Request(rel_id, j, None, limit, out[k], arrival,
                    tok=tok[k], token_seed=c.token_seed, prefix_len=plen)
            for j, k in enumerate(range(off[i], off[i + 1]))
        ]
        entries.append(RelQuery(rel_id, reqs, limit, arrival, plen))
    return entries


def _columns_from_entries(entries: list[RelQuery]) -> TraceColumns:
    r = len(entries)
    sizes = np.fromiter((q.size for q in entries), dtype=np.int64, count=r)
    row_off = np.zeros(r + 1, dtype=np.int64)
    np.cumsum(sizes, out=row_off[1:])
    n = int(row_off[-1])
    tok = np.empty(n, dtype=np.int32)
    out = np.empty(n, dtype=np.int32)
    seeds = set()
    k = 0
    for q in entries:
        for rq in q.requests:
            tok[k] = rq.tok
            out[k] = rq.actual_output_len
            seeds.add(None if rq.has_explicit_tokens else rq._token_seed)
            k += 1
    token_seed = None
    if len(seeds) == 1:
        (token_seed,) = seeds
    elif len(seeds) > 1:
        token_seed = None
    return TraceColumns(
        rel_id=np.fromiter((q.rel_id for q in entries), dtype=np.int64, count=r),
        arrival=np.fromiter((q.arrival for q in entries), dtype=np.float64, count=r),
        output_limit=np.fromiter((q.output_limit for q in entries), dtype=np.int32, count=r),
        prefix_len=np.fromiter((q.prefix_len for q in entries), dtype=np.int32, count=r),
        row_off=row_off,
        tok=tok,
        out=out,
        token_seed=token_seed,
    )


@dataclass
class TraceConfig:
    """Synthetic trace parameters (`workload.py:224-245`)."""

    num_relqueries: int = 100
    size_range: tuple[int, int] = (1, 100)
    rate: float = 1.0
    mean_input_len: int = 200
    output_limit: int | None = None
    shared_fraction: float = 0.40
    seed: int = 0

    def validate(self):
        if self.rate <= 0:
            raise ValueError("rate must be positive")
        lo, hi = self.size_range
        if not (1 <= lo <= hi):
            raise ValueError("size_range must be a non-empty positive range")
        if self.num_relqueries <= 0:
            raise ValueError("num_relqueries must be positive")
        if not (0.0 <= self.shared_fraction < 1.0):
            raise ValueError("shared_fraction must be in [0, 1)")


def _pack(rel_ids, arrivals, limits, prefix_lens, sizes, toks, outs, seed) -> TraceColumns:
    row_off = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(np.asarray(sizes, dtype=np.int64), out=row_off[1:])
    return TraceColumns(
        rel_id=np.asarray(rel_ids, dtype=np.int64),
        arrival=np.asarray(arrivals, dtype=np.float64),
        output_limit=np.asarray(limits, dtype=np.int32),
        prefix_len=np.asarray(prefix_lens, dtype=np.int32),
        row_off=row_off,
        tok=np.concatenate(toks).astype(np.int32) if toks else np.zeros(0, np.int32),
        out=np.concatenate(outs).astype(np.int32) if outs else np.zeros(0, np.int32),
        token_seed=seed,
    )


def generate_trace(config: TraceConfig) -> ArrivalTrace:
    """Poisson-arrival trace, count-identical to the reference generator.

    The main PCG64 stream is consumed in the same order as
    `workload.py:273-288` (exponential gap, size, query type, suffix lengths,
    EOS points per relQuery), so counts and arrivals match bit for bit; token
    IDs come from the count-keyed streams when read.
    """
    config.validate()
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([config.seed])))
    qtypes = list(QueryType)
    lo, hi = config.size_range
    prefix_len = max(1, round(config.shared_fraction * config.mean_input_len))
    suffix_mean = max(1, config.mean_input_len - prefix_len)
    s_lo, s_hi = max(1, suffix_mean // 2), suffix_mean + suffix_mean // 2 + 1
    clock = 0.0
    arrivals, limits, sizes, toks, outs = [], [], [], [], []
    for _ in range(config.num_relqueries):
        clock += rng.exponential(1.0 / config.rate)
        size = int(rng.integers(lo, hi + 1))
        qt = qtypes[rng.integers(0, len(qtypes))]
        limit = config.output_limit if config.output_limit is not None else OUTPUT_LIMITS[qt]
        suffix = rng.integers(s_lo, s_hi, size=size)
        out = rng.integers(max(1, limit // 2), limit + 1, size=size)
        arrivals.append(clock)
        limits.append(limit)
        sizes.append(size)
        toks.append(suffix + prefix_len)
        outs.append(out)
    n = config.num_relqueries
    cols = _pack(np.arange(n), arrivals, limits, [prefix_len] * n, sizes, toks, outs, config.seed)
    return ArrivalTrace(rate=config.rate, seed=config.seed, columns=cols)


def generate_heavy_tail_trace(
    num_relqueries: int = 5000,
    size_range: tuple[int, int] = (1, 399),
    rate: float = 1e6,
    mean_input_len: int = 200,
    shared_fraction: float = 0.40,
    seed: int = 0,
    pareto_alpha: float = 1.5,
    pareto_xm: float = 8.0,
    max_output_limit: int = 2048,
) -> ArrivalTrace:
    """Config-3 workload: heavy-tailed per-relQuery output limits.

    The reference has no heavy-tailed generator; this
    one draws ``output_limit = min(max_limit, floor(xm * V**(-1/alpha)))``
    with V = 1 - U uniform in (0, 1] (Pareto alpha=1.5, x_m=8) and per-row EOS
    points uniform in [max(1, L//2), L].  Tokens use the standard count-keyed
    streams, so `save_trace` output is loadable by the reference's
    `load_trace` and both sides see identical inputs.
    """
    cfg = TraceConfig(num_relqueries, size_range, rate, mean_input_len, None, shared_fraction, seed)
    cfg.validate()
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 0x7A11])))
    lo, hi = size_range
    prefix_len = max(1, round(shared_fraction * mean_input_len))
    suffix_mean = max(1, mean_input_len - prefix_len)
    s_lo, s_hi = max(1, suffix_mean // 2), suffix_mean + suffix_mean // 2 + 1
    clock = 0.0
    arrivals, limits, sizes, toks, outs = [], [], [], [], []
    for _ in range(num_relqueries):
        clock += rng.exponential(1.0 / rate)
        size = int(rng.integers(lo, hi + 1))
        v = 1.0 - rng.random()
        limit = int(min(max_output_limit, max(1, math.floor(pareto_xm * v ** (-1.0 / pareto_alpha)))))
        suffix = rng.integers(s_lo, s_hi, size=size)
        out = rng.integers(max(1, limit // 2), limit + 1, size=size)
        arrivals.append(clock)
        limits.append(limit)
        sizes.append(size)
        toks.append(suffix + prefix_len)
        outs.append(out)
    n = num_relqueries
    cols = _pack(np.arange(n), arrivals, limits, [prefix_len] * n, sizes, toks, outs, seed)
    return ArrivalTrace(rate=rate, seed=seed, columns=cols)


# ---------------------------------------------------------------------------
# relsim-trace-v1 files (pkg/docs/trace-schema.md; writer/loader semantics of
# workload.py:326-384)
# ---------------------------------------------------------------------------

def save_trace(trace: ArrivalTrace, path: str | Path) -> None:
    c = trace.columns()
    path = Path(path)
    with path.open("w") as f:
        f.write(json.dumps({"schema": "relsim-trace-v1", "rate": trace.rate, "seed": trace.seed}) + "\n")
        off = c.row_off.tolist()
        tok = c.tok.tolist()
        out = c.out.tolist()
        for i in range(c.num_relqueries):
            plen = int(c.prefix_len[i])
            rec = {
                "rel_id": int(c.rel_id[i]),
                "arrival_s": float(c.arrival[i]),
                "size": off[i + 1] - off[i],
                "output_limit": int(c.output_limit[i]),
                "prefix_len": plen,
                "requests": [
                    {"tok": tok[k], "prefix_len": plen, "out": out[k]}
                    for k in range(off[i], off[i + 1])
                ],
            }
            f.write(json.dumps(rec) + "\n")


def load_trace(path: str | Path) -> ArrivalTrace:
    """Read a relsim-trace-v1 file (workload.py:349-384).  The counts come from the native
    reader (csrc/trace_v1.cpp) when the library is built, else from the json module."""
    from . import _native

    path = Path(path)
    if _native.LIB_PATH.exists():
        try:
            rel_id, arrival, limit, plen, row_off, tok, out, rate, seed = _native.read_trace_v1(path)
        except ValueError as e:
            raise SchemaError(str(e)) from None
        cols = TraceColumns(rel_id=rel_id, arrival=arrival, output_limit=limit, prefix_len=plen, row_off=row_off,
                            tok=tok, out=out, token_seed=int(seed))
        return ArrivalTrace(rate=rate, seed=int(seed), columns=cols)
    return load_trace_json(path)


def load_trace_json(path: str | Path) -> ArrivalTrace:
    """load_trace with the json module (the reference's reader, restated on columns)."""
    path = Path(path)
    with path.open() as f:
        header = json.loads(f.readline())
        if header.get("schema") != "relsim-trace-v1":
            raise ValueError(f"unrecognized trace file {path}")
        seed = header["seed"]
        rel_ids, arrivals, limits, plens, sizes, toks, outs = [], [], [], [], [], [], []
        for line in f:
            rec = json.loads(line)
            reqs = rec["requests"]
            if rec.get("size", len(reqs)) != len(reqs):
                raise SchemaError(f"relQuery {rec['rel_id']}: size != len(requests)")
            for rr in reqs:
                if rr["prefix_len"] != rec["prefix_len"]:
                    raise SchemaError(f"relQuery {rec['rel_id']}: per-request prefix_len differs")
            rel_ids.append(rec["rel_id"])
            arrivals.append(rec["arrival_s"])
            limits.append(rec["output_limit"])
            plens.append(rec["prefix_len"])
            sizes.append(len(reqs))
            toks.append(np.fromiter((rr["tok"] for rr in reqs), dtype=np.int32, count=len(reqs)))
            outs.append(np.fromiter((rr["out"] for rr in reqs), dtype=np.int32, count=len(reqs)))
    cols = _pack(rel_ids, arrivals, limits, plens, sizes, toks, outs, seed)
    return ArrivalTrace(rate=header["rate"], seed=seed, columns=cols)
