"""A scripted sequence of DynamicPriorityUpdater.update calls (test infrastructure).

The same script drives relsim's updater (tests/golden/make_dpu_golden.py, in the
build container) and this package's device-backed one (tests/test_gpu_dpu_api.py):
relQueries arrive, rows are prefilled as a leading run of the lowest-priority
relQuery (A-inv1), prefilled rows decode, finished relQueries leave; the prefix
cache is a stub whose uncached count of a row is ``tok - 16 * m[rel_id]`` with the
resident chain lengths ``m`` changing between updates.  Every quantity the script
derives comes from integer arithmetic and the updater's own outputs, so both runs
see identical inputs iff the updaters agree.
"""

from __future__ import annotations

import numpy as np


class StubCache:
    """Duck-typed prefix cache: relsim's ``match_uncached(request, refresh=False)``."""

    def __init__(self):
        self.m: dict[int, int] = {}

    def match_uncached(self, request, refresh: bool = True) -> int:
        return max(0, request.tok - 16 * self.m.get(request.rel_id, 0))


SCENARIOS = {
    # name: (seed, relQueries, iterations, tau, sample_size)
    "dpu_api_inf": (11, 40, 60, float("inf"), 8),
    "dpu_api_tau": (12, 30, 60, 0.0004, 8),
    "dpu_api_k3": (13, 24, 40, float("inf"), 3),
}


def build(seed: int, n_rq: int, Request, RelQuery):
    rs = np.random.default_rng(seed)
    rqs = []
    for i in range(n_rq):
        size = int(rs.integers(1, 60))
        ol = int(rs.choice([5, 10, 50, 100]))
        arrival = float(i) * 0.0005
        reqs = []
        for j in range(size):
            tok = int(rs.integers(17, 300))
            out = int(rs.integers(max(1, ol // 2), ol + 1))
            reqs.append(Request(1000 + i, j, list(range(tok)), ol, out, arrival))
        rqs.append(RelQuery(1000 + i, reqs, ol, arrival))
    return rqs


def drive(dpu, cache: StubCache, rqs, iterations: int, seed: int):
    """Run the script; returns per-update [(rel_id, value, iteration_computed, reused, override)]
    plus the generator state after each update."""
    rs = np.random.default_rng(seed + 1000)
    live: list = []
    nxt = 0
    clock = 0.0
    out, states = [], []
    for it in range(iterations):
        while nxt < len(rqs) and rqs[nxt].arrival <= clock:
            live.append(rqs[nxt])
            nxt += 1
        recs = dpu.update(live, it, clock)
        out.append([(r.rel_id, r.value, r.iteration_computed, r.reused, r.starvation_override)
                     for r in recs.values()])
        st = dpu.rng.bit_generator.state
        states.append((int(st["state"]["state"]), int(st["has_uint32"]), int(st["uinteger"])))
        # decode one token on every prefilled, unfinished row
        for q in live:
            for r in q.requests:
                if r.prefilled and not r.done:
                    r.generated += 1
        # prefill a leading run of the pending rows of the min-(priority, arrival, rel_id) waiting relQuery
        waiting = [q for q in live if any(not r.prefilled for r in q.requests)]
        if waiting and it % 3 != 2:
            head = min(waiting, key=lambda q: (recs[q.rel_id].value, q.arrival, q.rel_id))
            pend = [r for r in head.requests if not r.prefilled]
            for r in pend[: int(rs.integers(1, 12))]:
                r.prefilled = True
        live = [q for q in live if not all(r.done for r in q.requests)]
        for q in live:  # the resident chains drift
            if rs.random() < 0.3:
                cache.m[q.rel_id] = int(rs.integers(0, 8))
        clock += 0.0007
    return out, states
