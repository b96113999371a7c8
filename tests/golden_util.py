"""Helpers shared by the golden-fixture generator and the parity tests.

Test infrastructure only: nothing in the product package imports this.
"""

from __future__ import annotations

import gzip
import hashlib
import json
from pathlib import Path

import numpy as np

GOLDEN_DIR = Path(__file__).resolve().parent / "golden"


def digest_arrays(rel_id, arrival, output_limit, prefix_len, sizes, tok, out) -> str:
    h = hashlib.sha256()
    for a, dt in ((rel_id, np.int64), (arrival, np.float64), (output_limit, np.int64),
                  (prefix_len, np.int64), (sizes, np.int64), (tok, np.int64), (out, np.int64)):
        h.update(np.ascontiguousarray(np.asarray(a, dtype=dt)).tobytes())
    return h.hexdigest()


def digest_entries(entries) -> str:
    """Digest of a trace given RelQuery-like objects (reference or mirror types)."""
    return digest_arrays(
        [q.rel_id for q in entries],
        [q.arrival for q in entries],
        [q.output_limit for q in entries],
        [q.prefix_len for q in entries],
        [len(q.requests) for q in entries],
        [r.tok for q in entries for r in q.requests],
        [r.actual_output_len for q in entries for r in q.requests],
    )


def digest_columns(c) -> str:
    return digest_arrays(c.rel_id, c.arrival, c.output_limit, c.prefix_len,
                         np.diff(c.row_off), c.tok, c.out)


#: named `EngineConfig.sp_priority_fns` pairs (golden configs say {"sp_fns": name}):
#: static priorities of either sign, so the waiting order is checked below zero too
SP_FNS = {
    "neg_mixed": (lambda tok: -0.001 * tok, lambda ol: 0.3 - 0.02 * ol),
    "neg_only": (lambda tok: -1.0 - 0.0005 * tok, lambda ol: -0.01 * ol),
}


def load_golden(name: str) -> dict:
    p = GOLDEN_DIR / f"{name}.json.gz"
    with gzip.open(p, "rt") as f:
        return json.load(f)


def golden_names() -> list[str]:
    return sorted(p.name[: -len(".json.gz")] for p in GOLDEN_DIR.glob("*.json.gz"))
