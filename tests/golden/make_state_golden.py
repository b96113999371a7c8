"""Goldens of relsim's Engine state between iterations (test infrastructure; runs in
the build container where the reference is mounted):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_state_golden.py

For each case the reference Engine runs with EngineConfig(iteration_limit=k) for
several k; when it stops (SimulationAborted, engine.py:376-379) its `running` list
(engine.py:205, execution order) and `waiting` queue (engine.py:160-176, 277-281)
are the state after k iterations.  Recorded: running as (rel_id, req_id), waiting as
(rel_id, pending req_ids' first and count, priority.hex()), the live relQueries (dict
order), the ledgers (engine.py:52-61) and the decision log so far.
"""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, "/root/reference/pkg/src")

from relsim.cost_model import world_preset  # noqa: E402
from relsim.engine import Engine, EngineConfig, SimulationAborted  # noqa: E402
from relsim.priority import SchedulerConstraints  # noqa: E402
from relsim.workload import TraceConfig, generate_trace  # noqa: E402

CASES = {
    # name: (trace config kwargs, policy, constraints, checkpoints)
    "state_relserve": (dict(num_relqueries=12, size_range=(5, 60), rate=40.0, seed=3), "relserve",
                       (4000, 24, 600), (1, 2, 5, 9, 17, 33, 60, 100)),
    "state_fcfs": (dict(num_relqueries=10, size_range=(5, 50), rate=40.0, seed=4), "fcfs",
                   (4000, 24, 600), (1, 3, 8, 20, 45, 90)),
}


def snapshot(trace_kw, policy, cons, k):
    trace = generate_trace(TraceConfig(**trace_kw))
    cfg = EngineConfig(constraints=SchedulerConstraints(*cons), iteration_limit=k)
    eng = Engine(trace, policy, world_preset("opt-13b-like"), cfg)
    try:
        eng.run()
        done = True
    except SimulationAborted:
        done = False
    return {"k": k, "finished": done, "iteration": eng.iteration, "clock": eng.clock.hex(),
            "kv_reserved": eng.kv_reserved,
            "running": [[r.rel_id, r.req_id] for r in eng.running],
            "waiting": [[w.relquery.rel_id, w.pending[0].req_id, len(w.pending), w.priority.hex()]
                        for w in eng.waiting],
            "live": list(eng.live_relqueries),
            "ledgers": [[k, v.arrival, v.first_prefill_start, v.last_prefill_end, v.last_decode_end]
                        for k, v in eng.ledgers.items()],
            "log": [[e.iteration, e.case, e.action] for e in eng.decision_log],
            "next_arrival": eng.next_arrival, "kv_resident_tokens": eng.kv_resident_tokens}


def main():
    out = ROOT / "tests" / "golden" / "state"
    out.mkdir(parents=True, exist_ok=True)
    for name, (kw, policy, cons, ks) in CASES.items():
        doc = {"name": name, "trace": kw, "policy": policy, "constraints": cons, "world": "opt-13b-like",
               "snapshots": [snapshot(kw, policy, cons, k) for k in ks]}
        with gzip.open(out / f"{name}.json.gz", "wt") as f:
            json.dump(doc, f)
        print(name, [(s["k"], len(s["running"]), len(s["waiting"])) for s in doc["snapshots"]])


if __name__ == "__main__":
    main()
