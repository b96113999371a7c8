"""Scheduler constraints, priority records and the GPU priority estimator.

Mirrors the public types of `pkg/src/relsim/priority.py` (SchedulerConstraints
30-40, PriorityRecord 62-68, RemainderItem 71-78, InfeasibleRequestError 26-27,
static_req_prio/static_relquery_prio 221-235).  `pem_batch` evaluates the
reference's `pem()` (priority.py:163-218) for many remainders at once on the
device -- the same device routine the engine's priority updater runs.
"""

from __future__ import annotations

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

