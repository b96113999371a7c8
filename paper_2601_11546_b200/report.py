"""Latency decomposition and cross-run summaries of device RunResults.

Mirror of the reference's reporting API (`pkg/src/relsim/report.py`): the
latency breakdown of one relQuery (report.py:22-47) and the (policy, rate)
summary table with speedups against a baseline policy (report.py:50-155),
so the "avg relQuery latency parity" half of the headline metric and the
reference's result tables come straight from GPU runs.  Host-side
post-processing of the ledgers the device engine returns.

The arithmetic follows the reference operation for operation (Python floats,
the builtin `sum` over values in the same order: groups by sorted key, runs in
input order, relQueries in ledger order, which is admission order), so the
tables -- and their CSV files -- are byte-identical to the reference's for the
same runs (tests/test_report_parity.py).
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass
from pathlib import Path

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
    """arrival -> first prefill start -> last prefill end -> last decode end (report.py:35-47)."""
    stamps = (ledger.first_prefill_start, ledger.last_prefill_end, ledger.last_decode_end)
    if any(t is None for t in stamps):
        raise IncompleteLedgerError(f"relQuery {rel_id}: missing timestamps")
    start, prefilled, decoded = stamps
    return LatencyBreakdown(rel_id, start - ledger.arrival, prefilled - start, decoded - prefilled)


def avg_latency(result: RunResult) -> float:
    """Mean total latency over completed relQueries (in rel_id order)."""
    vals = [decompose(r, led).total_s for r, led in sorted(result.ledgers.items()) if led.complete]
    return sum(vals) / len(vals) if vals else 0.0


#: SummaryRow's metric fields, in the reference's column order (report.py:73-77, 86-90)
METRICS = ("avg_latency_s", "max_latency_s", "avg_waiting_share", "avg_core_share", "avg_tail_share",
           "avg_unit_waiting_time", "speedup_vs_baseline")


@dataclass(frozen=True)
class SummaryRow:
    policy: str
    rate: float
    num_runs: int
    avg_latency_s: float
    max_latency_s: float
    avg_waiting_share: float
    avg_core_share: float
    avg_tail_share: float
    avg_unit_waiting_time: float
    speedup_vs_baseline: float


@dataclass
class SummaryTable:
    baseline: str
    rows: list[SummaryRow]

    def write_csv(self, path) -> None:
        """Wide table, one row per (policy, rate); floats as repr (report.py:69-83)."""
        header = ["policy", "rate", "num_runs", *METRICS[:-1], "speedup_vs_" + self.baseline]
        with Path(path).open("w", newline="") as f:
            w = csv.writer(f)
            w.writerow(header)
            w.writerows([r.policy, r.rate, r.num_runs, *(repr(getattr(r, m)) for m in METRICS)] for r in self.rows)

    def write_long_csv(self, path) -> None:
        """Plot-ready long format: policy, rate, metric, value (report.py:85-98)."""
        with Path(path).open("w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["policy", "rate", "metric", "value"])
            w.writerows([r.policy, r.rate, m, repr(getattr(r, m))] for r in self.rows for m in METRICS)


def _mean(xs: list[float]) -> float:
    return sum(xs) / len(xs) if xs else 0.0


def _group_stats(group: list[RunResult]) -> dict:
    """Per-(policy, rate) aggregates over every relQuery of every run of the group."""
    totals: list[float] = []
    shares: tuple[list[float], list[float], list[float]] = ([], [], [])
    unit_waiting: list[float] = []
    for run in group:
        for rel_id, led in run.ledgers.items():
            b = decompose(rel_id, led)
            t = b.total_s
            totals.append(t)
            if t > 0:
                for acc, part in zip(shares, (b.waiting_s, b.core_s, b.tail_s)):
                    acc.append(part / t)
            unit_waiting.append(b.waiting_s / run.relquery_sizes[rel_id])
    return {"num_runs": len(group), "avg": sum(totals) / len(totals), "max": max(totals),
            "shares": tuple(_mean(s) for s in shares), "uw": sum(unit_waiting) / len(unit_waiting)}


def summarize(runs: list[RunResult], baseline: str = "fcfs") -> SummaryTable:
    """Aggregate runs by (policy, rate); averages are over relQueries; speedup = the baseline
    policy's average latency at the same rate over this one's (NaN if the baseline did not
    run at that rate).  Runs must cover the same relQuery sets (report.py:101-155)."""
    if not runs:
        raise ValueError("need at least one run")
    if len({tuple(sorted(r.ledgers)) for r in runs}) > 1:
        raise ValueError("runs cover different relQuery sets; traces mismatch")
    groups: dict[tuple[str, float], list[RunResult]] = {}
    for run in runs:
        groups.setdefault((run.policy, run.rate), []).append(run)
    stats = {key: _group_stats(groups[key]) for key in sorted(groups)}
    rows = []
    for (policy, rate), st in stats.items():
        base = stats.get((baseline, rate))
        rows.append(SummaryRow(policy, rate, st["num_runs"], st["avg"], st["max"], *st["shares"], st["uw"],
                               base["avg"] / st["avg"] if base else math.nan))
    return SummaryTable(baseline, rows)
