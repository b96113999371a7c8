"""Reference outcomes of edge-case traces (test infrastructure; run in the build
container where the reference is mounted):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_edge_golden.py

Each case is a hand-built trace (explicit token lists) run through relsim's
`run` under every policy; recorded: the exception type and message, or the
iteration count, the final clock (hex), the decision log's (iteration, case,
action) triples and the ledgers.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT / "tests"))

from relsim.cost_model import world_preset  # noqa: E402
from relsim.engine import EngineConfig, run  # noqa: E402
from relsim.priority import SchedulerConstraints  # noqa: E402
from relsim.workload import ArrivalTrace, RelQuery, Request  # noqa: E402

import edge_cases  # noqa: E402

POLICIES = ("fcfs", "sp", "relserve", "relserve-pp", "relserve-dp")


def main():
    out = {}
    for name, spec in edge_cases.CASES.items():
        for pol in POLICIES:
            trace = edge_cases.build(spec, ArrivalTrace, RelQuery, Request)
            cfg = EngineConfig(constraints=SchedulerConstraints(*spec["constraints"]))
            try:
                r = run(trace, pol, world_preset("opt-13b-like"), cfg)
                rec = {"iterations": r.iterations, "clock": r.sim_duration.hex(),
                       "log": [[e.iteration, e.case, e.action] for e in r.decision_log],
                       "ledgers": {str(k): [v.arrival, v.first_prefill_start, v.last_prefill_end, v.last_decode_end]
                                   for k, v in sorted(r.ledgers.items())}}
            except Exception as e:  # noqa: BLE001 -- the reference's exception is the expected outcome
                rec = {"raises": type(e).__name__, "message": str(e)}
            out[f"{name}/{pol}"] = rec
            print(name, pol, rec.get("raises") or (rec["iterations"], rec["clock"]))
    _write(out)


def _write(out):
    import gzip

    with gzip.open(ROOT / "tests" / "golden" / "edge" / "edge_cases.json.gz", "wt") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
