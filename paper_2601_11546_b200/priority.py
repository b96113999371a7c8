"""Scheduler constraints, priority records and the GPU priority estimator.

Mirrors the public types of `pkg/src/relsim/priority.py` (SchedulerConstraints
30-40, PriorityRecord 62-68, RemainderItem 71-78, InfeasibleRequestError 26-27,
static_req_prio/static_relquery_prio 221-235).  `pem_batch` evaluates the
reference's `pem()` (priority.py:163-218) for many remainders at once on the
device -- the same device routine the engine's priority updater runs.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from .cost_model import LinearCostModel


class InfeasibleRequestError(ValueError):
    """A single request cannot fit the accelerator capacity."""


@dataclass(frozen=True)
class SchedulerConstraints:
    cap: int
    max_num_seqs: int
    max_num_batched_tokens: int

    def __post_init__(self):
        if min(self.cap, self.max_num_seqs, self.max_num_batched_tokens) <= 0:
            raise ValueError("constraints must be positive")
        if self.max_num_batched_tokens > self.cap:
            raise ValueError("max_num_batched_tokens must not exceed cap")


@dataclass
class PriorityRecord:
    rel_id: int
    value: float
    iteration_computed: int
    reused: bool = False
    starvation_override: bool = False


@dataclass(frozen=True)
class RemainderItem:
    request: object
    utok: int
    remaining: int
    prefilled: bool


def remainder_items(relquery, utok_of: Callable) -> list[RemainderItem]:
    """Live requests with the utok values the estimator uses (priority.py:81-98)."""
    items = []
    for r in relquery.requests:
        remaining = r.output_limit - r.generated
        if r.done or (r.prefilled and remaining <= 0):
            continue
        items.append(RemainderItem(r, 0 if r.prefilled else utok_of(r), remaining, r.prefilled))
    return items


def static_req_prio(request, l1: Callable[[int], float], l2: Callable[[int], float]) -> float:
    return l1(request.tok) + l2(request.output_limit)


def static_relquery_prio(relquery, l1, l2) -> float:
    return sum(static_req_prio(r, l1, l2) for r in relquery.requests)


def pem_batch(remainders: Sequence[Sequence[RemainderItem]] | Sequence[tuple],
              constraints: SchedulerConstraints, model: LinearCostModel,
              device: int = 0) -> np.ndarray:
    """pem() of every remainder, computed on the GPU.

    Each remainder is a sequence of RemainderItem, or a tuple of arrays
    ``(utok, remaining, prefilled)``.  Raises InfeasibleRequestError like the
    reference when an item's utok exceeds cap.
    """
    from . import _native

    offs = [0]
    utok, rem, pre = [], [], []
    for items in remainders:
        if isinstance(items, tuple):
            u, r, p = (np.asarray(x) for x in items)
        else:
            u = np.fromiter((it.utok for it in items), dtype=np.int64, count=len(items))
            r = np.fromiter((it.remaining for it in items), dtype=np.int32, count=len(items))
            p = np.fromiter((it.prefilled for it in items), dtype=np.uint8, count=len(items))
        if np.any(u > constraints.cap):
            raise InfeasibleRequestError(f"{int(u.max())} uncached tokens exceed cap {constraints.cap}")
        utok.append(u.astype(np.int64))
        rem.append(r.astype(np.int32))
        pre.append(p.astype(np.uint8))
        offs.append(offs[-1] + len(u))
    cat = (lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt))
    return _native.pem_batch(np.asarray(offs, np.int64), cat(utok, np.int64), cat(rem, np.int32),
                             cat(pre, np.uint8), constraints, model, device)


def pem(items: Sequence[RemainderItem], constraints: SchedulerConstraints, model: LinearCostModel,
        device: int = 0) -> float:
    """relsim's `pem(items, constraints, model)` (priority.py:163-218): the estimated
    remaining duration of one remainder, by the engine's device PEM (rs_pem_batch)."""
    return float(pem_batch([items], constraints, model, device)[0])



# -- the finer-grained priority API (relsim/__init__.py:3-12) ------------------


@dataclass
class CacheMissRatio:
    """A relQuery remainder's sampled uncached-token ratio (prefix_cache.py:20-29)."""

    rel_id: int
    ratio: float
    computed_at_iteration: int

    def __post_init__(self):
        if not (0.0 <= self.ratio <= 1.0):
            raise ValueError("ratio must be in [0, 1]")


def sample_cache_miss_ratio(cache, relquery_requests, sample_size: int, rng: np.random.Generator,
                            iteration: int = 0) -> CacheMissRatio:
    """relsim's sampler (prefix_cache.py:141-169): k = min(sample_size, n) rows drawn
    without replacement by ``rng.choice`` only when k < n (else every row, no draw);
    ratio = Σ cache.match_uncached(row, refresh=False) / Σ tok, an exact integer sum
    divided once.  ``cache`` is any object with relsim's ``match_uncached``."""
    if not relquery_requests:
        raise ValueError("relquery has no unfinished requests")
    n = len(relquery_requests)
    k = min(sample_size, n)
    picks = rng.choice(n, size=k, replace=False).tolist() if k < n else range(n)
    utok = tok = 0
    for i in picks:
        r = relquery_requests[int(i)]
        utok += cache.match_uncached(r, refresh=False)
        tok += r.tok
    return CacheMissRatio(relquery_requests[0].rel_id, utok / tok, iteration)


def utok_approx(request, ratio: float) -> int:
    """min(tok, ⌊tok·ratio + 0.5⌋), one rounded multiply and one rounded add
    (prefix_cache.py:172-176)."""
    if not (0.0 <= ratio <= 1.0):
        raise ValueError("ratio must be in [0, 1]")
    return min(request.tok, math.floor(request.tok * ratio + 0.5))


def apply_starvation_override(waiting_relqueries, records: dict, tau: float, clock: float) -> set:
    """Zero the record (and member priorities) of every wholly-waiting relQuery whose
    waiting time per original request exceeds tau, strictly (priority.py:318-339)."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    hit = set()
    if math.isinf(tau):
        return hit
    for rq in waiting_relqueries:
        if (clock - rq.arrival) / rq.size > tau:
            rec = records[rq.rel_id]
            rec.value, rec.starvation_override = 0.0, True
            for r in rq.requests:
                r.priority = 0.0
            hit.add(rq.rel_id)
    return hit


class DynamicPriorityUpdater:
    """relsim's Dynamic Priority Updater (priority.py:238-315) with the estimates of one
    update evaluated together on the GPU.

    The reuse rule, the cache-miss sampling (the caller's numpy Generator and prefix
    cache, consumed in the reference's visit order, so the generator stream advances
    exactly as relsim's does) and ``utok*`` stay on the host; every relQuery the update
    re-estimates contributes one remainder to a single ``rs_pem_batch`` launch -- the
    engine's own device PEM -- instead of one Python ``pem()`` loop per relQuery.
    Records, reuse, the starvation override and the per-request ``priority`` writes
    follow the reference.  (The engine itself never calls this class: its priority
    update runs inside the persistent kernel.)
    """

    def __init__(self, constraints: SchedulerConstraints, model: LinearCostModel, cache, sample_size: int = 8,
                 tau: float = math.inf, rng: np.random.Generator | None = None, *, device: int = 0):
        if tau <= 0:
            raise ValueError("tau must be positive")
        self.constraints = constraints
        self.model = model
        self.cache = cache
        self.sample_size = sample_size
        self.tau = tau
        self.rng = rng if rng is not None else np.random.default_rng(0)
        self.device = device
        self._records: dict[int, PriorityRecord] = {}
        self._seen_last_iteration: set[int] = set()

    def _can_reuse(self, rq) -> bool:
        if rq.rel_id not in self._records or rq.rel_id not in self._seen_last_iteration:
            return False
        return not any(r.prefilled or r.done for r in rq.requests)

    def _remainder(self, rq, iteration: int):
        """The remainder columns estimate() prices (priority.py:268-285), or None when
        no request is live (value 0.0, no draw)."""
        live = [r for r in rq.requests if not r.done]
        if not live:
            return None
        unpre = [r for r in live if not r.prefilled]
        ratio = (sample_cache_miss_ratio(self.cache, unpre, self.sample_size, self.rng, iteration).ratio
                 if unpre else 0.0)
        items = remainder_items(rq, lambda r: utok_approx(r, ratio))
        return (np.fromiter((it.utok for it in items), np.int64, len(items)),
                np.fromiter((it.remaining for it in items), np.int32, len(items)),
                np.fromiter((it.prefilled for it in items), np.uint8, len(items)))

    def estimate(self, rq, iteration: int) -> float:
        rem = self._remainder(rq, iteration)
        return 0.0 if rem is None else float(pem_batch([rem], self.constraints, self.model, self.device)[0])

    def update(self, relqueries, iteration: int, clock: float) -> dict[int, PriorityRecord]:
        relqueries = list(relqueries)
        records: dict[int, PriorityRecord] = {}
        todo, rems = [], []
        for rq in relqueries:  # visit order = the generator's consumption order
            if self._can_reuse(rq):
                prev = self._records[rq.rel_id]
                records[rq.rel_id] = PriorityRecord(rq.rel_id, prev.value, prev.iteration_computed, reused=True)
                continue
            rec = PriorityRecord(rq.rel_id, 0.0, iteration)
            records[rq.rel_id] = rec
            rem = self._remainder(rq, iteration)
            if rem is not None:
                todo.append(rec)
                rems.append(rem)
        if rems:  # one device launch for every estimate of this update
            for rec, v in zip(todo, pem_batch(rems, self.constraints, self.model, self.device).tolist()):
                rec.value = v
        waiting = [rq for rq in relqueries if not any(r.prefilled for r in rq.requests)]
        apply_starvation_override(waiting, records, self.tau, clock)
        for rq in relqueries:
            v = records[rq.rel_id].value
            for r in rq.requests:
                r.priority = v
        self._records = records
        self._seen_last_iteration = {rq.rel_id for rq in relqueries}
        return records
