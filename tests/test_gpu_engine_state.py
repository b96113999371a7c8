"""Engine state between steps equals relsim's (goldens: tests/golden/make_state_golden.py):
after k iterations, `Engine.running` (engine.py:205, execution order) and `Engine.waiting`
(engine.py:160-176, ordered by (priority, arrival, rel_id)) hold the same requests and
relQuery entries, `live_relqueries`, `ledgers` and `decision_log` agree, and the clock and
kv reservation agree bit for bit."""

import gzip
import json

import pytest

from golden_util import GOLDEN_DIR
from paper_2601_11546_b200 import SchedulerConstraints, TraceConfig, generate_trace, world_preset
from paper_2601_11546_b200.engine import Engine, EngineConfig

pytestmark = pytest.mark.gpu

NAMES = sorted(p.name[: -len(".json.gz")] for p in (GOLDEN_DIR / "state").glob("*.json.gz"))


@pytest.mark.parametrize("name", NAMES)
def test_running_and_waiting_between_steps(name):
    with gzip.open(GOLDEN_DIR / "state" / f"{name}.json.gz", "rt") as f:
        g = json.load(f)
    trace = generate_trace(TraceConfig(**{k: tuple(v) if isinstance(v, list) else v for k, v in g["trace"].items()}))
    cfg = EngineConfig(constraints=SchedulerConstraints(*g["constraints"]))
    eng = Engine(trace, g["policy"], world_preset(g["world"]), cfg, device=0)
    try:
        done = 0
        for snap in g["snapshots"]:
            eng.step(snap["k"] - done)
            done = snap["k"]
            assert eng.iteration == snap["iteration"]
            assert eng.clock.hex() == snap["clock"]
            assert eng.kv_reserved == snap["kv_reserved"]
            assert [[r.rel_id, r.req_id] for r in eng.running] == snap["running"], snap["k"]
            assert [[w.relquery.rel_id, w.pending[0].req_id, len(w.pending), w.priority.hex()]
                    for w in eng.waiting] == snap["waiting"], snap["k"]
            assert list(eng.live_relqueries) == snap["live"], snap["k"]
            assert [[k, v.arrival, v.first_prefill_start, v.last_prefill_end, v.last_decode_end]
                    for k, v in eng.ledgers.items()] == snap["ledgers"], snap["k"]
            assert [[e.iteration, e.case, e.action] for e in eng.decision_log] == snap["log"], snap["k"]
            assert eng.next_arrival == snap["next_arrival"], snap["k"]
            assert eng.kv_resident_tokens == snap["kv_resident_tokens"], snap["k"]
    finally:
        eng.close()
