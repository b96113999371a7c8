"""Latency decomposition of a RunResult (mirror of `pkg/src/relsim/report.py:22-47`).

Host-side post-processing of the ledgers the device engine returns; used for
the "avg relQuery latency parity" half of the headline metric.
"""

from __future__ import annotations

from dataclasses import dataclass

from .engine import RunResult, TimestampLedger


class IncompleteLedgerError(ValueError):
    pass


@dataclass(frozen=True)
class LatencyBreakdown:
    rel_id: int
    waiting_s: float
    core_s: float
    tail_s: float

    @property
    def total_s(self) -> float:
        return self.waiting_s + self.core_s + self.tail_s


def decompose(rel_id: int, ledger: TimestampLedger) -> LatencyBreakdown:
    if (ledger.first_prefill_start is None or ledger.last_prefill_end is None
            or ledger.last_decode_end is None):
        raise IncompleteLedgerError(f"relQuery {rel_id}: missing timestamps")
    return LatencyBreakdown(
        rel_id=rel_id,
        waiting_s=ledger.first_prefill_start - ledger.arrival,
        core_s=ledger.last_prefill_end - ledger.first_prefill_start,
        tail_s=ledger.last_decode_end - ledger.last_prefill_end,
    )


def avg_latency(result: RunResult) -> float:
    """Mean total latency over completed relQueries (in rel_id order)."""
    vals = [decompose(r, led).total_s for r, led in sorted(result.ledgers.items()) if led.complete]
    return sum(vals) / len(vals) if vals else 0.0
